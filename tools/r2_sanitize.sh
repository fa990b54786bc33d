# compute-sanitizer memcheck / racecheck / synccheck / initcheck on smoke() (one small decode
# batch: FSD + LSD streaming through decode_batch, and a lattice decode with device pruning)
python -c "import __graft_entry__; __graft_entry__.build()"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python -c "import __graft_entry__; __graft_entry__.smoke()" > gpurun_out/r2_sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/r2_sanitize_$tool.log
done
