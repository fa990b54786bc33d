# perf-only iteration: config-2 timings at the listed cluster sizes (no tests)
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
for K in ${KS:-1 2}; do
  WB_CLUSTER=$K timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu ${BENCH_ARGS} > gpurun_out/q_K$K.json 2> gpurun_out/q_K$K.err
  echo "K=$K rc=$?"; python -c "import json;d=json.load(open('gpurun_out/q_K$K.json'));print(round(d['value']), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['phase_share'])"
done
