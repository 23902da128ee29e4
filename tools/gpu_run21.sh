mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for dp in 0 -1; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_query|k_dense" --csv --log-file gpurun_out/launches21_$dp.csv python tools/cfg2_probe.py $dp > gpurun_out/ncu21_$dp.log 2>&1; echo "ncu list rc=$?"
done
