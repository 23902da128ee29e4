mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python tools/build_sweeps.py > gpurun_out/build_sweeps.md 2> gpurun_out/build_sweeps.err; echo "sweeps rc=$?"; tail -3 gpurun_out/build_sweeps.err
CMD="python tools/dense_probe.py cfg3 10000000 1000"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_transform -c 1 -o gpurun_out/prof_transform $CMD > gpurun_out/ncu_tr.log 2>&1; echo "ncu rc=$?"
