mkdir -p gpurun_out/r01r
python -m pytest tests -x -q -m gpu > gpurun_out/r01r/tests.log 2>&1; tail -3 gpurun_out/r01r/tests.log
python bench.py --config 3 --steps 2 --warmup 3 --no-cpu > gpurun_out/r01r/c3.json 2>&1
python bench.py --steps 3 --warmup 3 > gpurun_out/r01r/c2.json 2>&1
