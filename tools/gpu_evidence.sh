# round evidence: default bench line (configs[1]) + every other config at full size on one GPU,
# the reference arm, an ncu launch list of the default command and full captures of the top kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python bench.py > gpurun_out/ev_bench_cfg2.log 2>&1; echo "bench cfg2 rc=$?"
for c in cfg1 cfg3 cfg5 cfg4; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/ev_bench_$c.log 2>&1; echo "bench $c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev_ref_cfg2.log 2>&1; echo "reference rc=$?"; tail -c 400 gpurun_out/ev_ref_cfg2.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/ev_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|Radix|DeviceRadix|Segmented" --csv --log-file gpurun_out/ev_launches_cfg2.csv $CMD > gpurun_out/ev_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_query -s 6 -c 2 -o gpurun_out/ev_prof_cfg2 $CMD > gpurun_out/ev_ncu_full.log 2>&1; echo "ncu full cfg2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dense_screen|k_transform" -c 2 -o gpurun_out/ev_prof_dense_cfg3 python tools/dense_probe.py cfg3 10000000 1000 > gpurun_out/ev_ncu_dense.log 2>&1; echo "ncu full dense rc=$?"
