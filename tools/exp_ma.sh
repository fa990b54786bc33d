# max-active early cutoff (WB_MA_EARLY=<min live tokens>, 0 = off): parity + timing
set -u
o=gpurun_out/exp_ma; mkdir -p $o
WB_MA_EARLY=1 timeout 900 python -m pytest tests -x -q -m gpu > $o/tests_ma1.log 2>&1; echo "tests ma=1: $(tail -1 $o/tests_ma1.log)"
WB_MA_EARLY=1 timeout 300 python tools/stress.py 150 7 > $o/stress_ma1.log 2>&1; echo "stress ma=1: $(tail -2 $o/stress_ma1.log | tr '\n' ' ')"
run() { name=$1; shift; timeout 900 env "$@" > $o/$name.json 2> $o/$name.err; echo "$name: $(python -c "import json,sys; d=json.load(open('$o/$name.json')); print(round(d['value']), d['ms_per_step'], d['roofline']['frac'], d['counters_per_step']['n_cand'], d['counters_per_step']['n_surv'], d.get('e2e',{}).get('value'))" 2>&1 | tail -1)"; }
run c2_ma0 WB_MA_EARLY=0 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e
run c2_ma1024 WB_MA_EARLY=1024 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e
run c2_ma1 WB_MA_EARLY=1 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e
run c2_ma4096 WB_MA_EARLY=4096 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e
run c5_ma1024 WB_MA_EARLY=1024 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu --no-e2e
