# standard GPU check: build, dense + parity tests, then the bench configs given as arguments
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 400 python -m pytest tests/test_gpu_dense.py tests/test_gpu_parity.py -x -q --timeout 150 > gpurun_out/check_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/check_tests.log
for c in "$@"; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/check_$c.log 2>&1; echo "bench $c rc=$?"
  tail -1 gpurun_out/check_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['knn_stats']; print(d['config']['workload'], round(d['value'],1), 'q/s', round(d['ms_per_step'],3), 'ms', {k:s[k] for k in ('dense_queries','dense_candidates','dense_refined','refined','words_scanned','max_query_cycles')})"
done
