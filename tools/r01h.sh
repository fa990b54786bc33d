mkdir -p gpurun_out/r01h
python -m pytest tests -x -q -m gpu > gpurun_out/r01h/tests.log 2>&1; tail -1 gpurun_out/r01h/tests.log
python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r01h/c2.json 2>&1
python bench.py --config 5 --steps 2 --warmup 3 --no-cpu > gpurun_out/r01h/c5.json 2> gpurun_out/r01h/c5.err
tail -2 gpurun_out/r01h/c5.err
python bench.py --profile --steps 1 --warmup 3 > gpurun_out/r01h/plain_profile.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01h/launches_c2.csv python bench.py --profile --steps 2 --warmup 3 > gpurun_out/r01h/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 -o gpurun_out/r01h/decode_c2_full python bench.py --profile --steps 1 --warmup 3 > gpurun_out/r01h/ncu_full.log 2>&1
