# ncu --set full of the config-2 decode kernel (200-frame utterances to bound replay time)
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
CMD="python bench.py --steps 1 --warmup 1 --frames 200 --profile"
WB_CLUSTER=${K:-2} $CMD > gpurun_out/prof_plain.log 2>&1 &&
WB_CLUSTER=${K:-2} ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 1 -c 1 \
    -o gpurun_out/prof_c2_K${K:-2} $CMD > gpurun_out/prof_ncu.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/prof_ncu.log
