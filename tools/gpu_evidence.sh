# round evidence: default bench line (configs[1]), configs[2] line, ncu launch list + full captures
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python bench.py > gpurun_out/ev_bench_cfg2.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/ev_bench_cfg2.log
timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_bench_cfg3.log 2>&1; echo "bench cfg3 rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/ev_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|Radix|DeviceRadix" --csv --log-file gpurun_out/ev_launches_cfg2.csv $CMD > gpurun_out/ev_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_query -s 6 -c 2 -o gpurun_out/ev_prof_cfg2 $CMD > gpurun_out/ev_ncu_full.log 2>&1; echo "ncu full cfg2 rc=$?"
CMD3="python tools/dense_probe.py cfg3 10000000 1000"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_screen -s 1 -c 1 -o gpurun_out/ev_prof_dense_cfg3 $CMD3 > gpurun_out/ev_ncu_dense.log 2>&1; echo "ncu full dense rc=$?"
