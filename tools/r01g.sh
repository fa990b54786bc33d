mkdir -p gpurun_out/r01g
python bench.py --config 5 --steps 2 --warmup 3 --no-cpu > gpurun_out/r01g/c5.json 2> gpurun_out/r01g/c5.err
tail -2 gpurun_out/r01g/c5.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01g/launches_c2.csv python bench.py --profile --steps 2 --warmup 3 > gpurun_out/r01g/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 -o gpurun_out/r01g/decode_c2_full python bench.py --profile --steps 1 --warmup 3 > gpurun_out/r01g/ncu_full.log 2>&1
