mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
SOFA_FRONT_BATCHES=64 timeout 300 python tools/cfg2_probe.py -1 > gpurun_out/probe17.log 2>&1; tail -2 gpurun_out/probe17.log
SOFA_FRONT_BATCHES=64 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_query" --csv --log-file gpurun_out/launches17.csv python tools/cfg2_probe.py -1 > gpurun_out/ncu17a.log 2>&1; echo "ncu list rc=$?"
