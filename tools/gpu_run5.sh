mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/dense_probe.py cfg3 2000000 1000 > gpurun_out/probe6.log 2>&1; echo "probe rc=$?"; cat gpurun_out/probe5.log
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu6.log 2>&1; echo "gpu suite rc=$?"; tail -5 gpurun_out/pytest_gpu5.log
timeout 400 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench6_cfg3.log 2>&1; echo "bench cfg3 rc=$?"; tail -c 1800 gpurun_out/bench6_cfg3.log
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench6_cfg2.log 2>&1; echo "bench cfg2 rc=$?"; tail -c 600 gpurun_out/bench6_cfg2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_query|k_dense|k_merge" --csv --log-file gpurun_out/launches6_cfg3.csv python tools/dense_probe.py cfg3 2000000 1000 > gpurun_out/ncu6a.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_screen -s 1 -c 1 -o gpurun_out/prof6_dense python tools/dense_probe.py cfg3 2000000 1000 > gpurun_out/ncu6b.log 2>&1; echo "ncu full rc=$?"
