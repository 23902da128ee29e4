mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/dense_probe.py cfg2 > gpurun_out/probe14.log 2>&1; echo "probe rc=$?"; cat gpurun_out/probe14.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_query" --csv --log-file gpurun_out/launches14_cfg2.csv python tools/dense_probe.py cfg2 > gpurun_out/ncu14a.log 2>&1; echo "ncu list rc=$?"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 -k "scan_pool or knn_parity" > gpurun_out/pytest14a.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest14a.log
