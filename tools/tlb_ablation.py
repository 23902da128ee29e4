"""Synthetic analogs of the paper's TLB ablation (Tables 5/6) on the GPU:
mean TLB = mean sqrt(LB^2 / ED^2) over query x row pairs for SFA equi-depth / equi-width,
with variance-based selection (+VAR) or the first l real values (-VAR), and iSAX, at
alphabets 4..256 and l = 16; plus the mean selected coefficient index.  The paper's UCR
archive and datasets are not available; BASELINE.json's generators stand in (random walks for the
low-frequency sets, the 3-sinusoid recipe for the high-frequency ones).
python tools/tlb_ablation.py [N] [Q] [m] > profiles/r01_tlb_ablation.md"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17483_b200 import datagen  # noqa: E402
from paper_2411_17483_b200.index import SofaIndex  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
Q = int(sys.argv[2]) if len(sys.argv) > 2 else 50
M = int(sys.argv[3]) if len(sys.argv) > 3 else 20_000
L = 16
METHODS = [("SFA ED +VAR", "equi-depth", 0), ("SFA ED -VAR", "equi-depth", L // 2),
           ("SFA EW +VAR", "equi-width", 0), ("SFA EW -VAR", "equi-width", L // 2), ("iSAX", "isax", 0)]
ALPHABETS = [4, 8, 16, 32, 64, 128, 256]
out = {"N": N, "Q": Q, "pairs_per_query": M, "l": L, "rows": []}
print(f"# Mean TLB, synthetic stand-ins for Tables 5/6 (N={N:,} rows, {Q} queries x {M:,} rows, l={L})\n")
for kind in ("cfg1", "cfg3"):
    w = datagen.scaled(datagen.WORKLOADS[kind], N, Q)
    x = datagen.generate_rows(w, 0, N, device="cuda")
    q = datagen.generate_queries(w, device="cuda")
    name = "random walk (cfg recipe 0/1)" if kind == "cfg1" else "high frequency (cfg recipe 2)"
    print(f"## {name}\n")
    print("| method | " + " | ".join(f"a={a}" for a in ALPHABETS) + " | mean selected index |")
    print("|---|" + "---|" * (len(ALPHABETS) + 1))
    for label, binning, cl in METHODS:
        tl = []
        msi = None
        for a in ALPHABETS:
            ix = SofaIndex(x, l=L, alphabet=a, binning=binning, candidate_limit=cl,
                           sample_size=max(a, N // 100))
            lb2, ed2, _ = ix.lower_bounds(q, M)
            ok = ed2 > 0
            tl.append(float(torch.sqrt(lb2[ok].double() / ed2[ok].double()).mean()))
            if binning != "isax" and msi is None:
                msi = float(np.mean(np.asarray(ix.model["best_pos"]) >> 1))
            ix.close()
        out["rows"].append({"data": kind, "method": label, "tlb": dict(zip(ALPHABETS, tl)), "mean_selected_index": msi})
        print(f"| {label} | " + " | ".join(f"{t:.3f}" for t in tl) + f" | {msi if msi is None else f'{msi:.2f}'} |")
    print()
    del x, q
print("```json\n" + json.dumps(out) + "\n```")
