# bench a config under several values of one env knob: gpu_knob.sh VAR "v1 v2 ..." cfg...
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
var=$1; vals=$2; shift 2
for c in "$@"; do for v in $vals; do for i in ${REPS:-1 2}; do
env $var=$v timeout 900 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/knob_${c}_${v}_$i.log 2>&1
echo -n "$var=$v "; tail -1 gpurun_out/knob_${c}_${v}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value']), round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['kernel_ms'].items()}, d['knn_stats']['refined'])"
done; done; done
