mkdir -p gpurun_out/fin
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/fin/tests.log 2>&1; tail -1 gpurun_out/fin/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; tail -1 gpurun_out/fin/smoke.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/fin/ref2.json 2> gpurun_out/fin/ref2.err; echo "ref2 rc=$?"; cut -c1-200 gpurun_out/fin/ref2.json
WB_BENCH_SAME_DEVICE=1 WB_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 3 --utts 16 --frames 200 --no-cpu > gpurun_out/fin/b2.json 2> gpurun_out/fin/b2.err; echo "b2 rc=$?"; cut -c1-300 gpurun_out/fin/b2.json
