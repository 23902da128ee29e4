"""Per-query trace of one exact k-NN batch on a BASELINE workload (diagnostics, GPU box).
python tools/trace_knn.py [cfg2] [n_series]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17483_b200 import datagen, sofa as S  # noqa: E402
from paper_2411_17483_b200.index import SofaIndex  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
w = datagen.WORKLOADS[cfg]
if len(sys.argv) > 2:
    w = datagen.scaled(w, int(sys.argv[2]), w.n_queries)
x = datagen.generate_rows(w, 0, w.n_series, device="cuda")
q = datagen.generate_queries(w, device="cuda", data=x)
ix = SofaIndex(x, l=w.l, alphabet=w.alphabet, sample_size=datagen.default_sample_size(w))
for _ in range(2):
    ix.knn(q, w.k)
d, i, st = ix.knn(q, w.k, stats=True)
tr = S.sofa_knn_trace(ix.handle, w.n_queries)
tot = tr[:, :4].sum(1)
order = np.argsort(-tot)
np.set_printoptions(linewidth=250)
print("fields", S.TRACE_FIELDS)
print("mean", np.round(tr.mean(0)).astype(np.int64))
print("p50 ", np.percentile(tr, 50, axis=0).astype(np.int64))
print("p99 ", np.percentile(tr, 99, axis=0).astype(np.int64))
for r in order[:12]:
    print(r, tr[r])
src = datagen.query_sources(w) if w.query_kind == "noisy" else None
if src is not None:
    print("slowest queries found source:", [(int(r), int(i[r, 0]), int(src[r])) for r in order[:12]])
    print("dist of slowest:", d[order[:12], 0].cpu().numpy())
fl = np.nonzero(tr[:, 16] > 0)[0]
print("dense-flagged queries:", len(fl))
cand = np.nonzero(tr[:, 17] > 0)[0]
print("queries that reached the dense decision:", len(cand))
for r in cand[np.argsort(-tr[cand, 17])][:20]:
    print(r, "leaves", tr[r, 17], "pass", tr[r, 18], "/", tr[r, 19], "flag", tr[r, 16], "cycles", tr[r, :4].sum())
