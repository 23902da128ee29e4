"""Small exact k-NN runs for compute-sanitizer (memcheck / racecheck / synccheck, one tool per call):
the front and scan modes of k_query (8-warp and 16-warp builds), the dense screen + post (forced),
the scan pool with range tasks (dense candidates whose batch skips the dense pass), the transform and
the model learning, all on configs[0]-sized inputs.  Checks the results against the oracle so a run
that "passes" the sanitizer also computed the right answer.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import sofa_oracle as O  # noqa: E402
from paper_2411_17483_b200 import datagen  # noqa: E402
from paper_2411_17483_b200.index import SofaIndex  # noqa: E402
from knn_check import assert_knn_parity  # noqa: E402


def run(name, x, q, k, **kw):
    ix = SofaIndex(x, **kw)
    d, i, st = ix.knn(q, k, stats=True)
    torch.cuda.synchronize()
    xn, qn = x.cpu().numpy(), q.cpu().numpy()
    do, io = O.knn_bruteforce(xn, qn, k)
    assert_knn_parity(d.cpu().numpy(), i.cpu().numpy(), do, io, xn, qn)
    print(f"{name}: ok (dense queries {st['dense_queries']}, scan tasks {st['scan_tasks']})", flush=True)
    ix.close()


def main():
    torch.cuda.set_device(0)
    w = datagen.scaled(datagen.WORKLOADS["cfg1"], 20_000, 16)
    x = datagen.generate_rows(w, 0, w.n_series, device="cuda")
    q = datagen.generate_queries(w, device="cuda")
    run("sparse, 16 queries (16-warp build)", x, q, 3, sample_size=2000, dense_permille=-1)
    q2 = datagen.generate_queries(datagen.scaled(w, w.n_series, 600), device="cuda")
    run("sparse, 600 queries (8-warp build, scan pool)", x, q2, 2, sample_size=2000, dense_permille=-1)
    run("dense forced", x, q, 4, sample_size=2000, dense_permille=1000)
    wh = datagen.scaled(datagen.WORKLOADS["cfg3"], 20_000, 1)
    xh = datagen.generate_rows(wh, 0, wh.n_series, device="cuda")
    qh = datagen.generate_queries(wh, device="cuda")
    # high-frequency rows: the probe flags the query, but one query's estimated refines (< N) do not add
    # up to a dense pass over the rows, so the scan pool finishes it from range tasks
    run("high-frequency, dense candidates scanned sparsely", xh, qh, 1, sample_size=2000)


if __name__ == "__main__":
    main()
