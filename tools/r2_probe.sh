# spin probe: thread 0's lane-barrier wait per phase (probe build), config 2 at K = ${K:-2}
for K in ${KS:-2}; do
WB_LIB=$PWD/paper_1808_00687_b200/_lib/libwfstb200_probe.so WB_CLUSTER=$K timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu ${BENCH_ARGS} > gpurun_out/probe_K$K.json 2> gpurun_out/probe_K$K.err
echo "K=$K rc=$?"; python - $K <<'PY'
import json,sys
d=json.load(open('gpurun_out/probe_K%s.json'%sys.argv[1])); ps=d['phase_share']; t=ps['other']
print(round(d['ms_per_step'],2), {k: round(v/t,4) for k,v in ps.items() if k!='other'}, 'total spin', round(sum(v for k,v in ps.items() if k!='other')/t,4))
PY
done
