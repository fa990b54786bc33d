mkdir -p gpurun_out/r01b
python -m pytest tests -x -q -m gpu > gpurun_out/r01b/tests.log 2>&1; tail -2 gpurun_out/r01b/tests.log
python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01b/bench_c2.json 2> gpurun_out/r01b/bench_c2.err
python bench.py --config 4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01b/bench_c4.json 2> gpurun_out/r01b/bench_c4.err
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 -o gpurun_out/r01b/decode_c2_full python bench.py --profile --steps 1 --warmup 3 > gpurun_out/r01b/ncu_full.log 2>&1
