set -x
mkdir -p gpurun_out/r01
python bench.py --steps 5 --warmup 3 > gpurun_out/r01/bench_c2.json 2> gpurun_out/r01/bench_c2.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r01/ref_c2.json 2> gpurun_out/r01/ref_c2.err
python bench.py --config 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/r01/bench_c4.json 2> gpurun_out/r01/bench_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01/launches_c2.csv python bench.py --profile --steps 2 --warmup 3 > gpurun_out/r01/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 -o gpurun_out/r01/decode_c2_full python bench.py --profile --steps 1 --warmup 3 > gpurun_out/r01/ncu_full.log 2>&1
ls -la gpurun_out/r01
