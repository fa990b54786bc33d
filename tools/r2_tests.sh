# the full -m gpu suite (what the driver runs at round end) + smoke
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
timeout 2400 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"
tail -15 gpurun_out/gpu_tests.log
timeout 600 python -c "import __graft_entry__; __graft_entry__.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
