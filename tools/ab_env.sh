# A/B over environment settings on config 2: ENVS="A=1,B=2 A=0" (comma-separated per run; "-" = none)
L=${LIB:-$PWD/paper_1808_00687_b200/_lib/libwfstb200.so}
for e in ${ENVS:--}; do
  for K in ${KS:-2}; do
    envs=$(echo "$e" | tr ',' ' '); [ "$e" = "-" ] && envs=""
    env $envs WB_LIB=$L WB_CLUSTER=$K timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu ${BENCH_ARGS} > gpurun_out/abe.json 2> gpurun_out/abe.err
    echo "[$e] K=$K rc=$? $(python -c "import json;d=json.load(open('gpurun_out/abe.json'));print(round(d['value']), round(d['ms_per_step'],2), {k:round(v,3) for k,v in d['phase_share'].items()})" 2>&1 | tail -1)"
  done
done
