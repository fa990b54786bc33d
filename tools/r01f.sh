mkdir -p gpurun_out/r01f
python -m pytest tests -x -q -m gpu > gpurun_out/r01f/tests.log 2>&1; tail -1 gpurun_out/r01f/tests.log
python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r01f/c2.json 2>&1
python bench.py --config 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/r01f/c4.json 2>&1
python bench.py --config 3 --steps 2 --warmup 3 --no-cpu > gpurun_out/r01f/c3.json 2>&1
