mkdir -p gpurun_out/r01e
for v in u2g4 u1g4 u2g2 u1g2; do
 WB_LIB=$PWD/paper_1808_00687_b200/_lib/var/$v.so python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01e/c2_$v.json 2>&1
 WB_LIB=$PWD/paper_1808_00687_b200/_lib/var/$v.so python bench.py --config 4 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01e/c4_$v.json 2>&1
done
