# A/B of variant libraries on config 2: VARS="base inl" (base = the product library)
for v in ${VARS:-base}; do
  for K in ${KS:-2}; do
    if [ "$v" = base ]; then L=$PWD/paper_1808_00687_b200/_lib/libwfstb200.so; else L=$PWD/paper_1808_00687_b200/_lib/libwfstb200_$v.so; fi
    WB_LIB=$L WB_CLUSTER=$K timeout 600 python bench.py --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu ${BENCH_ARGS} > gpurun_out/ab_${v}_K$K.json 2> gpurun_out/ab_${v}_K$K.err
    echo "$v K=$K rc=$?"; python -c "import json;d=json.load(open('gpurun_out/ab_${v}_K$K.json'));print(round(d['value']), round(d['ms_per_step'],2), d.get('parity'), d['phase_share'])"
  done
done
