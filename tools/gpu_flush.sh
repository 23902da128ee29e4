mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for f in "" "--no-flush"; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $f > gpurun_out/flush$f.log 2>&1
tail -1 gpurun_out/flush$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['l2'], round(d['value']), round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['kernel_ms'].items()})"
done
