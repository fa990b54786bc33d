mkdir -p gpurun_out/r01i
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01i/base.json 2>&1
WB_LIB=$PWD/paper_1808_00687_b200/_lib/var/ef.so python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01i/ef.json 2>&1
WB_SMEM_KB=0 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01i/smemfull.json 2>&1
WB_SMEM_KB=160 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01i/smem160.json 2>&1
WB_LIB=$PWD/paper_1808_00687_b200/_lib/var/ef.so python bench.py --config 5 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01i/ef_c5.json 2>&1
