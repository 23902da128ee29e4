# A/B of two prebuilt libsofa.so (tools/ab/old.so, tools/ab/new.so) on the same box, alternating:
# gpu_ab_lib.sh "cfg..." reps steps
L=paper_2411_17483_b200/lib/libsofa.so
mkdir -p gpurun_out
for c in $1; do for i in $(seq ${2:-2}); do for v in old new; do
cp tools/ab/$v.so $L
timeout 900 python bench.py --config $c --steps ${3:-10} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ablib_${c}_${v}_$i.log 2>&1
echo -n "$v "; tail -1 gpurun_out/ablib_${c}_${v}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value']), round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['kernel_ms'].items()}, d['clocks']['sm_mhz'])"
done; done; done
cp tools/ab/new.so $L
