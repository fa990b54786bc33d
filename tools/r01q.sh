mkdir -p gpurun_out/r01q
python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01q/c2.json 2>&1
WB_PREFETCH_SLOTS=1 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01q/c2_ps.json 2>&1
WB_PREFETCH_SLOTS=1 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01q/c4_ps.json 2>&1
WB_PREFETCH_SLOTS=1 python bench.py --utts 148 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01q/c2u148_ps.json 2>&1
