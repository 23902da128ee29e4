mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for dp in -1 0; do
for fb in 1000000 64; do
SOFA_FRONT_BATCHES=$fb timeout 300 python tools/cfg2_probe.py $dp > gpurun_out/probe16_${dp}_$fb.log 2>&1; echo "fb=$fb rc=$?"; tail -2 gpurun_out/probe16_${dp}_$fb.log
done; done
