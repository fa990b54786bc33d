# ncu evidence for the current kernel: launch list of the default bench command, and per-launch
# DRAM traffic + L2 atomic counts of the config-2 decode kernel (full 1000-frame batch) at the
# automatic cluster size (K=2) and at K=1
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/nf_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/nf_launches.csv $CMD > gpurun_out/nf_launch_run.log 2>&1
echo "launches rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex_op_atom_dot_cas.sum,lts__t_requests_srcunit_tex_op_atom_dot_alu.sum,lts__t_sectors_srcunit_tex_op_atom.sum,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum,lts__t_sector_hit_rate.pct,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
for K in 2 1; do
  P="python bench.py --steps 1 --warmup 1 --profile"
  WB_CLUSTER=$K $P > gpurun_out/nf_p$K.log 2>&1 &&
  WB_CLUSTER=$K ncu --metrics $M --clock-control none -k regex:decode_kernel -s 1 -c 1 --csv --log-file gpurun_out/nf_metrics_K$K.csv $P > gpurun_out/nf_ncu_K$K.log 2>&1
  echo "metrics K=$K rc=$?"
done
