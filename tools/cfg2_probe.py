"""cfg2 work-counter probe: python tools/cfg2_probe.py [dense_permille]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17483_b200 import datagen, sofa as S  # noqa: E402
from paper_2411_17483_b200.index import SofaIndex  # noqa: E402

dp = int(sys.argv[1]) if len(sys.argv) > 1 else 0
w = datagen.WORKLOADS["cfg2"]
x = datagen.generate_rows(w, 0, w.n_series, device="cuda")
q = datagen.generate_queries(w, device="cuda", data=x)
ix = SofaIndex(x, sample_size=datagen.default_sample_size(w), dense_permille=dp)
for it in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    d, i, st = ix.knn(q, 1, stats=True)
    e1.record()
    torch.cuda.synchronize()
    tr = S.sofa_knn_trace(ix.handle, w.n_queries)
    print(f"dp={dp} it={it} {e0.elapsed_time(e1):.2f} ms words {st['words_scanned']} cand {st['candidates']} "
          f"refined {st['refined']} front-refined {tr[:, 7].sum()} front-words {tr[:, 5].sum()} "
          f"tasks {st['scan_tasks']} maxq {st['max_query_cycles']} phases {st['phase_cycles']}", flush=True)
