set -x
nproc; free -g | head -2
python -c "import __graft_entry__; __graft_entry__.build()"
timeout 1800 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_robustness.py -x -q -m gpu -rA > gpurun_out/r2_scale_tests.log 2>&1; echo "scale rc=$?"
tail -30 gpurun_out/r2_scale_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_c2.json 2> gpurun_out/r2_bench_c2.err; echo "bench rc=$?"
cat gpurun_out/r2_bench_c2.json; tail -5 gpurun_out/r2_bench_c2.err
