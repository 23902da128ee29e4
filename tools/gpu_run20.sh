mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/cfg2_probe.py 0 > gpurun_out/probe20.log 2>&1; tail -2 gpurun_out/probe20.log
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py -x -q --timeout 120 > gpurun_out/pytest20a.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest20a.log
