mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/cfg2_probe.py 0 > gpurun_out/probe22.log 2>&1; tail -2 gpurun_out/probe22.log
timeout 300 python tools/cfg2_probe.py -1 > gpurun_out/probe22b.log 2>&1; tail -1 gpurun_out/probe22b.log
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py -x -q --timeout 120 > gpurun_out/pytest22a.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest22a.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_query|k_dense" --csv --log-file gpurun_out/launches22.csv python tools/cfg2_probe.py 0 > gpurun_out/ncu22.log 2>&1; echo "ncu list rc=$?"
