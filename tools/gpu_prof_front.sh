mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pf_bench.log 2>&1
tail -1 gpurun_out/pf_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['l2'], round(d['value']), round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['kernel_ms'].items()})"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_query -s 6 -c 1 -o gpurun_out/pf_front $CMD > gpurun_out/pf_ncu.log 2>&1; echo "ncu rc=$?"
