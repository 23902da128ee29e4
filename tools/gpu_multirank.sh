# multi-rank code path on a one-GPU box (gloo, 2 ranks on cuda:0): parity tests + a bench smoke
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -x --timeout 600 -k "two_ranks or seed or sharded" 2>&1 | tail -3
SOFA_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/mr_bench.log 2>&1; echo "bench 2 ranks rc=$?"
tail -1 gpurun_out/mr_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['value']), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms'].items()}, d['knn_stats']['refined'], d['knn_stats']['words_scanned'])"
