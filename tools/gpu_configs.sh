# every BASELINE config at full size on one GPU (exploratory: 2 steps, 3 warm-ups)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for c in cfg1 cfg5 cfg4; do
  timeout 1200 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_full_$c.log 2>&1; echo "bench $c rc=$?"; tail -c 700 gpurun_out/bench_full_$c.log; echo
done
