mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/trace_knn.py cfg2 > gpurun_out/trace8_cfg2.log 2>&1; echo "trace rc=$?"; tail -25 gpurun_out/trace8_cfg2.log
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu8.log 2>&1; echo "gpu suite rc=$?"; tail -5 gpurun_out/pytest_gpu8.log
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench8_cfg2.log 2>&1; echo "bench cfg2 rc=$?"; tail -c 300 gpurun_out/bench8_cfg2.log
