mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_isax.py -q -x --timeout 200 > gpurun_out/f2_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/f2_tests.log
timeout 900 python tools/tlb_ablation.py > gpurun_out/tlb_ablation.md 2> gpurun_out/tlb_ablation.err; echo "ablation rc=$?"; head -30 gpurun_out/tlb_ablation.md; tail -5 gpurun_out/tlb_ablation.err
