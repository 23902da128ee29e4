# dense path (f1) bring-up: dense tests first (bounded), then the whole gpu suite, then cfg3 bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 420 python -m pytest tests/test_gpu_dense.py -x -q --timeout 200 > gpurun_out/dense_tests.log 2>&1; echo "dense tests rc=$?"
tail -40 gpurun_out/dense_tests.log
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu3.log 2>&1; echo "gpu suite rc=$?"
tail -15 gpurun_out/pytest_gpu3.log
timeout 400 python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench3_cfg3.log 2>&1; echo "bench cfg3 rc=$?"; tail -c 2500 gpurun_out/bench3_cfg3.log
