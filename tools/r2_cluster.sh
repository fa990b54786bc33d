python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_cluster.py -x -q -m gpu > gpurun_out/r2_cluster_tests.log 2>&1; echo "cluster tests rc=$?"
tail -25 gpurun_out/r2_cluster_tests.log
for K in 1 2 4; do
  WB_CLUSTER=$K timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2_c2_K$K.json 2> gpurun_out/r2_c2_K$K.err
  echo "K=$K rc=$?"; python -c "import json;d=json.load(open('gpurun_out/r2_c2_K$K.json'));print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['phase_share'])"
done
