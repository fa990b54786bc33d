# lanes-per-SM sweep on config 5 (experiment)
set -u
o=gpurun_out/exp2; mkdir -p $o
M=paper_1808_00687_b200/_lib/libwfstb200_m2.so
run() { name=$1; shift; timeout 900 env "$@" --no-cpu --no-e2e > $o/$name.json 2> $o/$name.err; echo "$name: $(python -c "import json,sys; d=json.load(open('$o/$name.json')); print(round(d['value']), d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1)"; }
C5="python bench.py --config 5 --steps 2 --warmup 3"
run c5_1024s64 WB_SMEM_KB=64 $C5
run c5_512x2s48 WB_SMEM_KB=48 WB_LIB=$M $C5 --block 512 --lanes 296
run c5_512x2s40 WB_SMEM_KB=40 WB_LIB=$M $C5 --block 512 --lanes 296
run c5_512x2s80 WB_SMEM_KB=80 WB_LIB=$M $C5 --block 512 --lanes 296
run c5_256x4s40 WB_SMEM_KB=40 WB_LIB=$M $C5 --block 256 --lanes 592
run c5_256x4s32 WB_SMEM_KB=32 WB_LIB=$M $C5 --block 256 --lanes 592
run c5_512x2s64 WB_SMEM_KB=64 WB_LIB=$M $C5 --block 512 --lanes 296
