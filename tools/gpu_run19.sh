mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/cfg2_probe.py 0 > gpurun_out/probe19.log 2>&1; tail -2 gpurun_out/probe19.log
timeout 300 python tools/cfg2_probe.py -1 > gpurun_out/probe19b.log 2>&1; tail -1 gpurun_out/probe19b.log
timeout 300 python tools/trace_knn.py cfg2 > gpurun_out/trace19_cfg2.log 2>&1; head -12 gpurun_out/trace19_cfg2.log
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py -x -q --timeout 120 > gpurun_out/pytest19a.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest19a.log
