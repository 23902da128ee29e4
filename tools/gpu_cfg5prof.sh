mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/dense_probe.py cfg5 4000000 1000 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_query|k_dense" --csv --log-file gpurun_out/c5_list.csv python tools/dense_probe.py cfg5 4000000 1000 > /dev/null 2>&1; echo "list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_query -s 3 -c 2 -o gpurun_out/c5_prof python tools/dense_probe.py cfg5 4000000 1000 > gpurun_out/c5_ncu.log 2>&1; echo "ncu rc=$?"
