o=gpurun_out/smem; mkdir -p $o
for kb in 100 64 80 120 100; do
WB_SMEM_KB=$kb timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $o/c2_$kb.json 2>/dev/null
python -c "import json; d=json.load(open('$o/c2_$kb.json')); print('$kb', round(d['value']), round(d['ms_per_step'],1))"
done
