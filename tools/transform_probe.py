"""Transform (a1 + a3) throughput probe: builds the index of a config several times and prints the
build's transform phase (CUDA events on the build stream, sofa_get_info.build_ms) as GB/s of the
algorithmic bytes (rows read once; words, statistics, key, value and bf16 row copy written).

  python tools/transform_probe.py [cfg3] [n_series] [repeats]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17483_b200 import datagen  # noqa: E402
from paper_2411_17483_b200.index import SofaIndex  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
w = datagen.WORKLOADS[cfg]
if len(sys.argv) > 2:
    w = datagen.scaled(w, int(sys.argv[2]))
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
x = datagen.generate_rows(w, 0, w.n_series, device="cuda")
rows = w.n_series
nbytes = rows * w.length * 4 + rows * (16 * ((w.l + 15) // 16) + 8 + 8 + 2 * w.length)
best = None
for r in range(reps):
    ix = SofaIndex(x, l=w.l, alphabet=w.alphabet, sample_size=datagen.default_sample_size(w))
    torch.cuda.synchronize()
    ms = ix.info["build_ms"]["transform"]
    best = ms if best is None else min(best, ms)
    print(f"{cfg} N={rows} n={w.length} l={w.l}: transform {ms:.3f} ms = {nbytes / ms / 1e6:.0f} GB/s", flush=True)
    ix.close()
print(f"BEST {cfg} transform {best:.3f} ms = {nbytes / best / 1e6:.0f} GB/s")
