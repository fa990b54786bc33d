mkdir -p gpurun_out/r01l
for ma in 7000 3500 1750; do python bench.py --utts 32 --max-active $ma --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01l/u32_ma$ma.json 2>&1; done
