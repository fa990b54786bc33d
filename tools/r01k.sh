mkdir -p gpurun_out/r01k
for u in 32 64 148; do python bench.py --utts $u --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01k/c2_u$u.json 2>&1; done
python bench.py --config 3 --utts 148 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01k/c3_u148.json 2>&1
