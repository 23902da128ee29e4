mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x --timeout 200 -k "index_invariants or model_parity" > gpurun_out/f3_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/f3_tests.log
timeout 1500 python tools/build_sweeps.py > gpurun_out/build_sweeps.md 2> gpurun_out/build_sweeps.err; echo "sweeps rc=$?"; head -40 gpurun_out/build_sweeps.md; tail -5 gpurun_out/build_sweeps.err
