"""The k-NN acceptance check (BASELINE.json north_star), shared by the GPU tests and
__graft_entry__.smoke(): neighbour indices exact except ties within TIE_RTOL relative distance,
distances within DIST_RTOL relative, the k returned indices of a query distinct, padding (+inf, -1)
exactly where the oracle pads."""
import math

import numpy as np

from oracle import sofa_oracle as O

DIST_RTOL = 1e-4
TIE_RTOL = 1e-5


def assert_knn_parity(d_gpu, i_gpu, d_or, i_or, data_np=None, queries_np=None):
    """indices exact except ties within TIE_RTOL; distances within DIST_RTOL relative; no repeated
    index within a query's list.  A mismatched index is accepted only if its TRUE distance (oracle
    z-ED of that row, when the data are given) is within TIE_RTOL of the oracle's rank-r distance."""
    d_gpu = np.asarray(d_gpu, dtype=np.float64)
    i_gpu = np.asarray(i_gpu)
    assert d_gpu.shape == d_or.shape and i_gpu.shape == i_or.shape
    fin = np.isfinite(d_or)
    assert np.array_equal(np.isfinite(d_gpu), fin)
    assert np.array_equal(i_gpu >= 0, fin)
    np.testing.assert_allclose(d_gpu[fin], d_or[fin], rtol=DIST_RTOL, atol=1e-6)
    for q in range(i_gpu.shape[0]):
        got = i_gpu[q][i_gpu[q] >= 0]
        assert len(np.unique(got)) == len(got), (q, got)
    bad = (i_gpu != i_or) & fin
    for q, r in zip(*np.nonzero(bad)):
        ref = d_or[q, r]
        if data_np is not None:
            xh, _, _, _ = O.znorm(data_np[i_gpu[q, r]:i_gpu[q, r] + 1])
            qh, _, _, _ = O.znorm(queries_np[q:q + 1])
            true_d = math.sqrt(O.sq_dists_direct(xh, qh[0])[0])
        else:
            true_d = d_gpu[q, r]
        assert abs(true_d - ref) <= TIE_RTOL * max(ref, 1e-12) + 1e-7, (q, r, i_gpu[q, r], i_or[q, r], true_d, ref)
