mkdir -p gpurun_out/r01d
python bench.py --config 3 --steps 2 --warmup 3 > gpurun_out/r01d/bench_c3.json 2> gpurun_out/r01d/bench_c3.err
tail -3 gpurun_out/r01d/bench_c3.err
