mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/dense_probe.py cfg2 > gpurun_out/probe13.log 2>&1; echo "probe rc=$?"; cat gpurun_out/probe13.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|Radix" --csv --log-file gpurun_out/launches13_cfg2.csv python tools/dense_probe.py cfg2 > gpurun_out/ncu13a.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_query -s 4 -c 2 -o gpurun_out/prof13_cfg2 python tools/dense_probe.py cfg2 > gpurun_out/ncu13b.log 2>&1; echo "ncu full rc=$?"
