mkdir -p gpurun_out/r01m
python -m pytest tests/test_gpu_lattice.py -x -q > gpurun_out/r01m/tests.log 2>&1; tail -1 gpurun_out/r01m/tests.log
python bench.py --config 3 --steps 3 --warmup 3 --no-cpu > gpurun_out/r01m/c3.json 2>&1
