mkdir -p gpurun_out/r01s
timeout 900 python -m pytest tests -x -q -m gpu -o faulthandler_timeout=120 > gpurun_out/r01s/tests.log 2>&1; tail -3 gpurun_out/r01s/tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r01s/c2.json 2>&1
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/r01s/c4.json 2>&1
timeout 900 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu > gpurun_out/r01s/c3.json 2>&1
