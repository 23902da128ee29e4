"""Dense-path probe (GPU box): one config, per-kernel CUDA-event breakdown is not available from
Python, so run under ncu for kernel times.  python tools/dense_probe.py [cfg3] [N] [Q]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17483_b200 import datagen  # noqa: E402
from paper_2411_17483_b200.index import SofaIndex  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
w = datagen.WORKLOADS[cfg]
N = int(sys.argv[2]) if len(sys.argv) > 2 else w.n_series
Q = int(sys.argv[3]) if len(sys.argv) > 3 else w.n_queries
w = datagen.scaled(w, N, Q)
x = datagen.generate_rows(w, 0, N, device="cuda")
q = datagen.generate_queries(w, device="cuda", data=x)
ix = SofaIndex(x, l=w.l, alphabet=w.alphabet, sample_size=datagen.default_sample_size(w))
torch.cuda.synchronize()
for it in range(3):
    t0 = time.perf_counter()
    d, i, st = ix.knn(q, w.k, stats=True)
    torch.cuda.synchronize()
    print(f"iter {it}: {1e3 * (time.perf_counter() - t0):.2f} ms", {k: st[k] for k in (
        "dense_queries", "dense_candidates", "dense_refined", "refined", "words_scanned")}, flush=True)
