# round-1 evidence pass: per-query trace, ncu launch list + full capture of k_query (cfg2), other configs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python tools/trace_knn.py cfg2 > gpurun_out/trace_cfg2.log 2>&1; echo "trace rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_query -s 3 -c 1 -o gpurun_out/prof_cfg2 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
for c in cfg1 cfg3 cfg5 cfg4; do
  timeout 900 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?"; tail -c 1500 gpurun_out/bench_$c.log
done
