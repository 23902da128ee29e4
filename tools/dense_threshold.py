"""Sweep of the dense-path stage-2 threshold (sofa_build_opts.dense_permille) on BASELINE workloads:
per setting, the batch time split (front / dense / scan), the dense queries and the sparse refines.
Results are identical for every setting (only the route of each query changes).

  python tools/dense_threshold.py cfg4:20000000 cfg2 ...
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17483_b200 import datagen  # noqa: E402
from paper_2411_17483_b200.index import SofaIndex  # noqa: E402

for arg in sys.argv[1:] or ["cfg2"]:
    name, _, n = arg.partition(":")
    w = datagen.WORKLOADS[name]
    if n:
        w = datagen.scaled(w, int(n), w.n_queries)
    x = datagen.generate_rows(w, 0, w.n_series, device="cuda")
    q = datagen.generate_queries(w, device="cuda", data=x)
    for pm in (2, 5, 10, 20, 50):
        ix = SofaIndex(x, l=w.l, alphabet=w.alphabet, sample_size=datagen.default_sample_size(w), dense_permille=pm)
        for _ in range(2):
            ix.knn(q, w.k)
        _, _, st = ix.knn(q, w.k, stats=True)
        torch.cuda.synchronize()
        ix.kernel_timing(1)
        for _ in range(5):
            ix.knn(q, w.k)
        km, _ = ix.kernel_timing(0)
        print(f"{name} N={w.n_series} permille {pm:3d}: front {km['front'] / 5:.3f} dense {km['dense'] / 5:.3f} "
              f"scan {km['scan'] / 5:.3f} ms | dense queries {st['dense_queries']} refined {st['refined']} "
              f"words {st['words_scanned']}", flush=True)
        ix.close()
    del x, q
    torch.cuda.empty_cache()
