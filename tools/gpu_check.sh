# Round-end check on one B200: GPU tests, smoke, config-2 bench, two-rank reference + plumbing runs
o=gpurun_out/fin; mkdir -p $o
timeout 900 python -m pytest tests -x -q -m gpu > $o/tests.log 2>&1; tail -1 $o/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; tail -1 $o/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > $o/bench_c2.json 2> $o/bench_c2.err; echo "bench rc=$?"; cut -c1-160 $o/bench_c2.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > $o/ref2.json 2> $o/ref2.err; echo "ref2 rc=$?"
WB_BENCH_SAME_DEVICE=1 WB_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 3 --utts 16 --frames 200 --no-cpu > $o/b2.json 2> $o/b2.err; echo "b2 rc=$?"
