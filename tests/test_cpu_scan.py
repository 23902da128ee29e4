"""The CPU brute-force scan baseline (cpu_scan/) returns the oracle's exact k-NN (CPU test)."""
import numpy as np

import cpu_scan
from oracle import sofa_oracle as O
from paper_2411_17483_b200 import datagen

from knn_check import assert_knn_parity


def test_cpu_scan_equals_oracle():
    w = datagen.scaled(datagen.WORKLOADS["cfg1"], 20_000, 12, length=256)
    x = datagen.generate_rows(w, 0, w.n_series).numpy()
    q = datagen.generate_queries(w).numpy()
    x[7] = x[3]  # a duplicate: ties go to the smaller index
    st = cpu_scan.row_stats(x)
    d, i = cpu_scan.knn(x, st, q, 5, threads=4)
    do, io = O.knn_bruteforce(x, q, 5)
    assert_knn_parity(d, i, do, io, x, q)
    d1, i1 = cpu_scan.knn(x, st, x[[3]], 2, threads=3)
    assert list(i1[0]) == [3, 7] and d1[0, 0] == 0.0
