mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for i in 1 2 3; do
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab2_$i.log 2>&1
tail -1 gpurun_out/ab2_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['kernel_ms'].items()})"
done
timeout 300 python -m pytest tests/test_gpu_dense.py tests/test_gpu_parity.py -q -x --timeout 150 2>&1 | tail -1
