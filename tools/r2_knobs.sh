# config-2 timings (K = 2) under tuning knobs; one line each
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
run() { env "$@" timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/knob.json 2>/dev/null;
        python -c "import json,sys;d=json.load(open('gpurun_out/knob.json'));print(sys.argv[1:], round(d['ms_per_step'],2))" "$@"; }
run WB_CLUSTER=2
run WB_CLUSTER=2 WB_XCHG_GATHER=1
run WB_CLUSTER=2 WB_XCHG_GATHER=0
run WB_CLUSTER=2 WB_SMEM_KB=80
run WB_CLUSTER=2 WB_SMEM_KB=128
run WB_CLUSTER=2 WB_ROW_PREFETCH=0
run WB_CLUSTER=2 WB_PREFETCH=0
run WB_CLUSTER=2 WB_EXACT_MIN=0
