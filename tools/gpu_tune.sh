# parameter sweep for the front budget (SOFA_FRONT_BATCHES) on configs[1]
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for fb in 4 8 16 32 64; do
SOFA_FRONT_BATCHES=$fb timeout 300 python tools/cfg2_probe.py 0 > gpurun_out/tune_fb$fb.log 2>&1; echo "fb=$fb"; tail -2 gpurun_out/tune_fb$fb.log | cut -c1-200
done
