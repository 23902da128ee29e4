mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1800 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py::test_cfg2_full_size_sampled -v --timeout 900 -x > gpurun_out/fullsize.log 2>&1; echo "fullsize rc=$?"; grep -E "PASS|FAIL|Error|assert|passed|failed" gpurun_out/fullsize.log | tail -20
