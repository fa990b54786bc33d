mkdir -p gpurun_out/r01c
for kb in 48 100 160 0; do for b in 1024 512; do
 WB_SMEM_KB=$kb python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --block $b > gpurun_out/r01c/c2_${kb}_${b}.json 2>&1
done; done
