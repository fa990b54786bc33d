mkdir -p gpurun_out/r01n
python -m pytest tests -x -q -m gpu > gpurun_out/r01n/tests.log 2>&1; tail -1 gpurun_out/r01n/tests.log
python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01n/c2_pf.json 2>&1
WB_PREFETCH=0 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01n/c2_nopf.json 2>&1
python bench.py --config 4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01n/c4_pf.json 2>&1
python bench.py --utts 148 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01n/c2u148_pf.json 2>&1
