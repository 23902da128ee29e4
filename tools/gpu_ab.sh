# repeated bench runs (noise estimate) of the given configs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for c in "$@"; do for i in 1 2; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_$i.log 2>&1
tail -1 gpurun_out/ab_${c}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value']), round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['kernel_ms'].items()}, d['knn_stats']['dense_queries'])"
done; done
