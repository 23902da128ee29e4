"""Per-call timing distribution of configs[1] k-NN batches and the per-query trace of the fastest
and slowest stats calls (diagnostic)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17483_b200 import datagen, sofa as S  # noqa: E402
from paper_2411_17483_b200.index import SofaIndex  # noqa: E402

w = datagen.WORKLOADS["cfg2"]
x = datagen.generate_rows(w, 0, w.n_series, device="cuda")
q = datagen.generate_queries(w, device="cuda", data=x)
ix = SofaIndex(x, sample_size=datagen.default_sample_size(w))
for _ in range(3):
    ix.knn(q, 1)
ts = []
for _ in range(40):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ix.knn(q, 1)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("plain calls ms:", np.round(sorted(ts), 3))
runs = []
for _ in range(12):
    _, _, st = ix.knn(q, 1, stats=True)
    tr = S.sofa_knn_trace(ix.handle, w.n_queries)
    runs.append((st["kernel_ms"]["front"], st, tr))
runs.sort(key=lambda r: r[0])
for name, (f, st, tr) in (("fastest", runs[0]), ("slowest", runs[-1])):
    tot = tr[:, :4].sum(1)
    print(name, "front ms", round(f, 3), "max query cycles", tot.max(), "sum", tot.sum(), "words", st["words_scanned"],
          "refined", st["refined"], "tasks", st["scan_tasks"], "dense flagged", int((tr[:, 16] > 0).sum()))
    cta = tr[:, 14]
    per_cta = np.bincount(cta, weights=tot, minlength=444)
    print("   per-CTA busy cycles: max", per_cta.max(), "mean", per_cta.mean(), "CTAs used", (per_cta > 0).sum())
    print("   slowest queries", np.argsort(-tot)[:5], tot[np.argsort(-tot)[:5]])
    for qq in np.argsort(-tot)[:3]:
        print("     q", qq, "phases (prep, seed, tree, scan)", tr[qq, :4], "leaves", tr[qq, 4], "words", tr[qq, 5],
              "cand", tr[qq, 6], "refined", tr[qq, 7], "list", tr[qq, 10], "dense-inputs", tr[qq, 16:20])
