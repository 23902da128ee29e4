"""Timing diagnostic of the dense screen's pipeline stages (sofa_tuning.dense_diag; results are wrong
while a diag bit is set, so nothing here checks them): the dense pass time with the full epilogue,
without its screening math, without TMEM loads, and with the producers ignoring their twins.

  python tools/dense_diag.py [cfg4] [n_series] [n_queries]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17483_b200 import datagen  # noqa: E402
from paper_2411_17483_b200.index import SofaIndex  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
w = datagen.WORKLOADS[cfg]
if len(sys.argv) > 2:
    w = datagen.scaled(w, int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else w.n_queries)
x = datagen.generate_rows(w, 0, w.n_series, device="cuda")
q = datagen.generate_queries(w, device="cuda", data=x)
ix = SofaIndex(x, l=w.l, alphabet=w.alphabet, sample_size=datagen.default_sample_size(w))
_, _, st = ix.knn(q, w.k, stats=True)
print(f"{cfg} N={w.n_series} dense queries {st['dense_queries']} candidates {st['dense_candidates']}", flush=True)
flops = 2.0 * st["dense_queries"] * w.n_series * w.length
MODES = [(1, 0, 0), (1, 0, 1), (1, 0, 2), (1, 0, 8), (1, 0, 16), (1, 0, 32), (1, 0, 48), (0, 0, 0), (0, 0, 2),
         (0, 0, 4), (0, 1, 0), (0, 1, 2), (1, 0, 0)]
if os.environ.get("DIAG_MODES"):
    MODES = [tuple(int(v) for v in m.split(",")) for m in os.environ["DIAG_MODES"].split(";")]
for mc, pair, diag in MODES:
    ix.set_tuning(dense_diag=diag, dense_pair=pair, dense_mcast=mc)
    for _ in range(2):
        ix.knn(q, w.k)
    torch.cuda.synchronize()
    ix.kernel_timing(1)
    for _ in range(5):
        ix.knn(q, w.k)
    km, groups = ix.kernel_timing(0)
    dense = km["dense"] / 5
    print(f"mcast {mc} pair {pair} diag {diag}: front {km['front'] / 5:.3f} ms  dense {dense:.3f} ms "
          f"({flops / dense / 1e9:.0f} TFLOP/s)  scan {km['scan'] / 5:.3f} ms", flush=True)
ix.set_tuning()
