python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
timeout 1500 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_checks.py tests/test_gpu_scale_parity.py tests/test_gpu_robustness.py -x -q -m gpu > gpurun_out/iter_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/iter_tests.log
for K in ${KS:-1 2}; do
  WB_CLUSTER=$K timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/iter_K$K.json 2> gpurun_out/iter_K$K.err
  echo "K=$K rc=$?"; python -c "import json;d=json.load(open('gpurun_out/iter_K$K.json'));print(round(d['value']), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['phase_share'])"
done
