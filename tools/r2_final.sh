# final evidence for the committed kernel: ncu traffic + atomics of the config-2 decode kernel
# (default K), launch list of the default bench command, then the benches of configs 2-5
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex_op_atom_dot_cas.sum,lts__t_requests_srcunit_tex_op_atom_dot_alu.sum,lts__t_sectors_srcunit_tex_op_atom.sum,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum,lts__t_sector_hit_rate.pct,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum
P="python bench.py --steps 1 --warmup 1 --profile"
$P > gpurun_out/fin_p.log 2>&1 &&
ncu --metrics $M --clock-control none -k regex:decode_kernel -s 1 -c 1 --csv --log-file gpurun_out/fin_metrics_c2.csv $P > gpurun_out/fin_ncu.log 2>&1
echo "metrics rc=$?"
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/fin_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches.csv $CMD > gpurun_out/fin_launch_run.log 2>&1
echo "launches rc=$?"
python tools/update_traffic.py gpurun_out/fin_metrics_c2.csv 2 "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum of one config-2 decode_kernel launch (profiles/r02_fin_metrics_c2.csv)"
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/fin_c2.json 2> gpurun_out/fin_c2.err; echo "c2 rc=$?"
for c in 4 3 5; do
  timeout 1500 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/fin_c$c.json 2> gpurun_out/fin_c$c.err; echo "c$c rc=$?"
done
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin_ref_c2.json 2> gpurun_out/fin_ref.err; echo "ref rc=$?"
for f in gpurun_out/fin_c*.json gpurun_out/fin_ref_c2.json; do python - "$f" <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
e=d.get('e2e') or {}; p=d.get('e2e_from_posteriors') or {}; r=d.get('roofline') or {}
print(sys.argv[1], round(d['value']), 'ms', round(d['ms_per_step'],1), 'e2e', round(e.get('value',0)), 'post', round(p.get('value',0)), 'frac', r.get('frac'), 'traffic', r.get('traffic'), 'parity', d.get('parity'))
PY
done
