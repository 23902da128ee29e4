mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py -x -q --timeout 120 > gpurun_out/pytest24a.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest24a.log
timeout 600 python -m pytest tests -m gpu -x -q --timeout 200 > gpurun_out/pytest_gpu24.log 2>&1; echo "gpu suite rc=$?"; tail -2 gpurun_out/pytest_gpu24.log
timeout 300 python tools/trace_knn.py cfg2 > gpurun_out/trace24_cfg2.log 2>&1; head -14 gpurun_out/trace24_cfg2.log
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench24_cfg2.log 2>&1; echo "bench cfg2 rc=$?"; tail -c 400 gpurun_out/bench24_cfg2.log
timeout 400 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench24_cfg3.log 2>&1; echo "bench cfg3 rc=$?"; tail -c 300 gpurun_out/bench24_cfg3.log
