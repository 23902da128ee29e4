mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for fb in 1000000 64 16; do
SOFA_FRONT_BATCHES=$fb timeout 300 python tools/dense_probe.py cfg2 > gpurun_out/probe15_$fb.log 2>&1; echo "probe fb=$fb rc=$?"; tail -2 gpurun_out/probe15_$fb.log
done
