mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x --timeout 200 -k "index_invariants or transform or knn_parity or block_size" 2>&1 | tail -2
timeout 300 python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2411_17483_b200 import datagen
from paper_2411_17483_b200.index import SofaIndex
for kind in ("cfg2", "cfg3"):
    w = datagen.WORKLOADS[kind]
    x = datagen.generate_rows(w, 0, w.n_series, device="cuda")
    best = None
    for _ in range(3):
        ix = SofaIndex(x, sample_size=datagen.default_sample_size(w))
        b = ix.info["build_ms"]
        best = b if best is None or sum(b.values()) < sum(best.values()) else best
        ix.close()
    print(kind, {k: round(v, 2) for k, v in best.items()}, "total", round(sum(best.values()), 2))
    del x
PY
