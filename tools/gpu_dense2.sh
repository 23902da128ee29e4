mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_dense.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x --timeout 300 2>&1 | tail -1
for c in cfg2 cfg3 cfg4 cfg5; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d2_$c.log 2>&1
tail -1 gpurun_out/d2_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['workload'], round(d['value']), round(d['ms_per_step'],2), r['bound'], round(r['frac'],3), {k: round(v,2) for k,v in d['kernel_ms'].items()})"
done
