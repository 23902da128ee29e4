mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/dense_probe.py cfg3 2000000 1000 > gpurun_out/probe4.log 2>&1; echo "probe rc=$?"; cat gpurun_out/probe4.log
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu4.log 2>&1; echo "gpu suite rc=$?"; tail -5 gpurun_out/pytest_gpu4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_query|k_dense|k_merge" --csv --log-file gpurun_out/launches4_cfg3.csv python tools/dense_probe.py cfg3 2000000 1000 > gpurun_out/ncu4a.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_screen -s 1 -c 1 -o gpurun_out/prof4_dense python tools/dense_probe.py cfg3 2000000 1000 > gpurun_out/ncu4b.log 2>&1; echo "ncu full rc=$?"
