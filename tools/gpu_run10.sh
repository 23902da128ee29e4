mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 -k "scan_pool or knn_parity" > gpurun_out/pytest10a.log 2>&1; echo "sharing tests rc=$?"; tail -15 gpurun_out/pytest9a.log
timeout 600 python -m pytest tests -m gpu -x -q --timeout 200 > gpurun_out/pytest_gpu10.log 2>&1; echo "gpu suite rc=$?"; tail -5 gpurun_out/pytest_gpu10.log
timeout 300 python tools/trace_knn.py cfg2 > gpurun_out/trace10_cfg2.log 2>&1; echo "trace rc=$?"; head -20 gpurun_out/trace10_cfg2.log
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench10_cfg2.log 2>&1; echo "bench cfg2 rc=$?"; tail -c 1500 gpurun_out/bench10_cfg2.log
timeout 400 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench10_cfg3.log 2>&1; echo "bench cfg3 rc=$?"; tail -c 300 gpurun_out/bench10_cfg3.log
