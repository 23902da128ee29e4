"""Single-query latency (the paper's setting: queries answered one at a time) and small-batch
latency on a BASELINE workload: median / p90 GPU ms of knn over the first queries one by one.
python tools/latency_probe.py [cfg2] [n_queries_timed] [dense_batch_rows as a fraction of N, e.g. 0.25]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17483_b200 import datagen  # noqa: E402
from paper_2411_17483_b200.index import SofaIndex  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 50
w = datagen.WORKLOADS[cfg]
x = datagen.generate_rows(w, 0, w.n_series, device="cuda")
q = datagen.generate_queries(w, device="cuda", data=x)
ix = SofaIndex(x, l=w.l, alphabet=w.alphabet, sample_size=datagen.default_sample_size(w))
tag = ""
if len(sys.argv) > 3:  # the batch runs the dense pass once its flagged queries' estimated refines reach this
    ix.set_tuning(dense_batch_rows=max(1, int(float(sys.argv[3]) * w.n_series)))
    tag = f" [dense_batch_rows = {sys.argv[3]} N]"
for bs in (1, 8, 100):
    ts = []
    for s in range(0, min(m * bs, w.n_queries), bs):
        qq = q[s:s + bs].contiguous()
        ix.knn(qq, w.k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ix.knn(qq, w.k)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = np.array(ts)
    print(f"{w.name}{tag} batch {bs}: median {np.median(ts):.3f} ms  p90 {np.percentile(ts, 90):.3f} ms  "
          f"({len(ts)} batches; {bs / np.median(ts) * 1e3:,.0f} q/s)")
