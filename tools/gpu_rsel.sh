# front/scan refine-row variants: gpu_rsel.sh "cfg..." steps
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null || exit 1
for c in $1; do for fs in "2 2" "2 4" "4 4" "2 4" "2 2"; do set -- $fs
SOFA_R_FRONT=$1 SOFA_R_SCAN=$2 timeout 900 python bench.py --config $c --steps ${STEPS:-30} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rsel.log 2>&1
echo -n "front R=$1 scan R=$2 "; tail -1 gpurun_out/rsel.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value']), round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['kernel_ms'].items()})"
done; done
