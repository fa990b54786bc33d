#!/usr/bin/env bash
# The measurement recipe behind profiles/ (run on the B200 box through gpurun):
#   gpurun --timeout 3000 -- 'bash tools/gpu_measure.sh r02'
# Tests first; ncu only after the same command has exited 0 without it.
set -u
tag=${1:-rXX}
out=gpurun_out/$tag
mkdir -p "$out"
timeout 900 python -m pytest tests -x -q -m gpu > "$out/tests.log" 2>&1; tail -1 "$out/tests.log"
timeout 900 python bench.py --steps 5 --warmup 3 > "$out/bench_c2.json" 2> "$out/bench_c2.err"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > "$out/ref_c2.json" 2> "$out/ref_c2.err"
for c in 3 4 5; do
  timeout 1200 python bench.py --config $c --steps 2 --warmup 3 --no-cpu > "$out/bench_c$c.json" 2> "$out/bench_c$c.err"
done
timeout 600 python bench.py --profile --steps 1 --warmup 3 > "$out/plain_profile.json" 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$out/launches_c2.csv" python bench.py --profile --steps 2 --warmup 3 > "$out/ncu_launch.log" 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 \
    -o "$out/decode_c2_full" python bench.py --profile --steps 1 --warmup 3 > "$out/ncu_full.log" 2>&1
ls -la "$out"
