"""GPU parity of the dense path (csrc/dense.cu): queries the SFA envelope filter
cannot prune are finished by a tcgen05 TF32 screen (a proven lower bound, approx - eps) plus the
exact refine.  Results must equal the oracle's brute force exactly as the sparse path's do, and
the two paths must return bit-identical (distance, index) lists on the same index."""
import numpy as np
import pytest
import torch

from oracle import sofa_oracle as O
from paper_2411_17483_b200 import datagen
from paper_2411_17483_b200.index import SofaIndex

from test_gpu_parity import _data, assert_knn_parity

pytestmark = pytest.mark.gpu


def _check(x, q, k, **kw):
    ix = SofaIndex(x, **kw)
    d, i, st = ix.knn(q, k, stats=True)
    torch.cuda.synchronize()
    do, io = O.knn_bruteforce(x.cpu().numpy(), q.cpu().numpy(), k)
    assert_knn_parity(d.cpu().numpy(), i.cpu().numpy(), do, io, x.cpu().numpy(), q.cpu().numpy())
    return ix, d, i, st


@pytest.mark.parametrize("kind,N,n,l,k,Q", [
    ("cfg3", 60_000, 256, 16, 1, 40),      # high frequency: every query goes dense by itself
    ("cfg3", 33_333, 256, 16, 7, 130),     # ragged N, 2 query tiles (130 > 128), k = 7
    ("cfg5", 40_000, 1024, 32, 10, 40),    # n = 1024 (32 K-chunks), l = 32, k = 10
    ("cfg3", 20_000, 100, 16, 3, 17),      # len not a multiple of 32 (TMA zero fill of the last chunk)
])
def test_dense_parity(kind, N, n, l, k, Q):
    w = datagen.scaled(datagen.WORKLOADS[kind], N, Q, length=n, l=l, k=k)
    x, q = _data(w)
    _, _, _, st = _check(x, q, k, l=l, sample_size=datagen.default_sample_size(w))
    if kind == "cfg3":
        assert st["dense_queries"] == Q
    # every dense query's k results were refined exactly from screened candidates (or its brute-force
    # fallback), so at least k candidates per dense query reached the refine
    assert st["dense_candidates"] >= st["dense_queries"] * k


@pytest.mark.parametrize("Q,k", [(1, 1), (1, 4), (3, 2), (300, 3)])
def test_dense_flagged_but_batch_sparse_scans_ranges(Q, k):
    """high-frequency queries are flagged by the probe before their tree descent, but the batch needs
    more estimated refines than they add up to (dense_batch_rows): the batch skips the dense pass and
    the scan pool finishes them from range tasks (every leaf in storage order, pruned by its envelope
    LB) — exact all the same"""
    w = datagen.scaled(datagen.WORKLOADS["cfg3"], 120_000 + 77, Q)
    x, q = _data(w)
    ix = SofaIndex(x, sample_size=datagen.default_sample_size(w))
    ix.set_tuning(dense_batch_rows=1 << 60)
    d, i, st = ix.knn(q, k, stats=True)
    do, io = O.knn_bruteforce(x.cpu().numpy(), q.cpu().numpy(), k)
    assert_knn_parity(d.cpu().numpy(), i.cpu().numpy(), do, io, x.cpu().numpy(), q.cpu().numpy())
    assert st["dense_queries"] == 0      # the dense pass did not run
    assert st["scan_queries"] == Q       # every query was handed to the scan pool
    assert st["words_scanned"] >= Q * w.n_series * 0.9  # (nearly) every word, no tree pruning


@pytest.mark.parametrize("kind,k", [("cfg1", 1), ("cfg4", 5), ("cfg2", 1)])
def test_forced_dense_equals_sparse(kind, k):
    """dense_permille=1000 forces every query through the dense path; -1 never: identical bits."""
    w = datagen.scaled(datagen.WORKLOADS[kind], 50_000 + 13, 70)
    x, q = _data(w)
    ixd, dd, idd, st = _check(x, q, k, sample_size=5000, dense_permille=1000)
    assert st["dense_queries"] > 0
    ixs = SofaIndex(x, sample_size=5000, dense_permille=-1)
    ds, is_, ss = ixs.knn(q, k, stats=True)
    assert ss["dense_queries"] == 0
    assert torch.equal(idd, is_) and torch.equal(dd, ds)


def test_dense_edge_rows_and_bsf_init():
    """constant rows, huge offsets/scales, exact duplicates and a caller bound through the dense path"""
    rng = np.random.default_rng(11)
    base = (np.sin(np.arange(64)[None, :] * rng.uniform(5, 25, size=(3000, 1)) + rng.uniform(0, 6, (3000, 1)))
            + 0.7 * rng.normal(size=(3000, 64))).astype(np.float32)
    base[10] = 3.0                           # constant -> zero vector
    base[11] = base[12] * 5000.0 + 1.0e4     # offset/scale: same z-normalised shape as row 12
    base[13] = base[14]                      # duplicate -> tie to the smaller index
    x = torch.from_numpy(base).cuda()
    qs = base[[10, 12, 14, 100, 2999]]
    q = torch.from_numpy(qs).cuda()
    ix, d, i, st = _check(x, q, 4, l=8, alphabet=64, sample_size=1000, block_size=32, dense_permille=1000)
    assert st["dense_queries"] >= 3
    assert i[2, 0].item() == 13 and i[2, 1].item() == 14 and d[2, 0].item() == 0.0
    d0 = d[:, 0] ** 2
    bound = (d0 * 0.5).contiguous()          # below every true NN: nothing may be returned
    d2, i2 = ix.knn(q, 4, bsf_init=bound)
    assert bool((i2[d0 > 0] == -1).all())


@pytest.mark.parametrize("N,k", [(37, 37), (37, 20), (300, 128), (513, 100)])
def test_dense_ragged_tile_with_unfilled_topk(N, k):
    """the dense screen's last row tile extends past N; while a query holds fewer than k results its
    threshold is +inf, and the rows past the end must still never become candidates (regression:
    they carried |x^|^2 = +inf, and +inf <= +inf emitted them)"""
    rng = np.random.default_rng(N + k)
    base = np.cumsum(rng.normal(size=(N, 32)), axis=1).astype(np.float32)
    x = torch.from_numpy(base).cuda()
    q = torch.from_numpy(base[[0, N // 2, N - 1]] + rng.normal(scale=0.1, size=(3, 32)).astype(np.float32)).cuda()
    ix, d, i, st = _check(x, q, k, l=4, alphabet=4, sample_size=N, block_size=32, dense_permille=1000)
    assert st["dense_queries"] == 3
    assert bool((i >= 0).all()) and bool((i < N).all())
    assert st["dense_candidates"] <= 3 * N


def test_dense_candidate_overflow_falls_back_exactly():
    """a 64-entry candidate buffer overflows; the per-query brute-force fallback keeps results exact"""
    w = datagen.scaled(datagen.WORKLOADS["cfg3"], 30_000, 20, k=3)
    x, q = _data(w)
    ix = SofaIndex(x, sample_size=3000)
    ix.set_tuning(dense_cand_cap=64)
    d, i, st = ix.knn(q, 3, stats=True)
    torch.cuda.synchronize()
    assert st["dense_queries"] == 20 and st["dense_candidates"] > 64, st
    assert st["dense_refined"] >= x.shape[0]   # at least one query was rescanned brute force
    do, io = O.knn_bruteforce(x.cpu().numpy(), q.cpu().numpy(), 3)
    assert_knn_parity(d.cpu().numpy(), i.cpu().numpy(), do, io, x.cpu().numpy(), q.cpu().numpy())
    ix.set_tuning()                            # default capacity: same bits
    d2, i2 = ix.knn(q, 3)
    assert torch.equal(d, d2) and torch.equal(i, i2)


def test_batch_decision_defers_few_flagged_queries():
    """noisy-member queries (cfg2 recipe): flagged queries, if any, are too few to justify a full
    tensor-core pass; the deferred sparse launch must finish them with identical results"""
    w = datagen.scaled(datagen.WORKLOADS["cfg2"], 120_000, 150)
    x, q = _data(w)
    ix, d, i, st = _check(x, q, 1, sample_size=datagen.default_sample_size(w))
    assert st["dense_queries"] == 0
    assert np.array_equal(i[:, 0].cpu().numpy(), datagen.query_sources(w))


@pytest.mark.parametrize("n,q,m", [(256, 200, 4096 + 77), (1024, 64, 1500), (100, 37, 999), (256, 256, 300)])
def test_dense_dots_within_bound(n, q, m):
    """the tensor cores' own accumulation (tcgen05.mma kind::f16, read back raw through
    sofa_dense_dots) against the bound the screen assumes: products of the bf16 operands
    exact, fp32 accumulation error <= n 2^-23 sum|x_t q_t|; and the total error against the float32
    inputs <= gamma |x| |q| (gamma = 2^-7 + 2^-15 + n 2^-23).  Adversarial rows: alternating large
    values that cancel, values on bf16 rounding midpoints, z-normalised walks, zeros"""
    from paper_2411_17483_b200 import sofa as S
    from test_dense_bound import bf16
    rng = np.random.default_rng(n * 7 + q)
    x = np.cumsum(rng.normal(size=(m, n)), axis=1)
    x = ((x - x.mean(1, keepdims=True)) / x.std(1, keepdims=True)).astype(np.float32)
    alt = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    x[:40] = (alt[None, :] * rng.uniform(1, 30, size=(40, 1)) + rng.normal(scale=1e-3, size=(40, n))).astype(np.float32)
    mid = (1.0 + (2 * rng.integers(0, 128, size=(40, n)) + 1) * 2.0 ** -8).astype(np.float32)  # bf16 ties
    x[40:80] = mid * rng.choice([-1.0, 1.0], size=(40, n))
    x[80:90] = 0.0
    qs = rng.normal(size=(q, n)).astype(np.float32)
    qs[0] = 1.0                       # against the alternating rows: heavy cancellation
    qs[1] = alt.astype(np.float32)    # ... or none
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(qs).cuda()
    out = torch.empty(m, q, dtype=torch.float32, device="cuda")
    S.sofa_dense_dots(xd, m, n, qd, q, out)
    hw = out.cpu().numpy().astype(np.float64)
    xb, qb = bf16(x).astype(np.float64), bf16(qs).astype(np.float64)
    exact = xb @ qb.T
    absprod = np.abs(xb) @ np.abs(qb).T
    acc_err = np.abs(hw - exact)
    assert np.all(acc_err <= n * 2.0 ** -23 * absprod), (acc_err / np.maximum(absprod, 1e-30)).max()
    gamma = 2.0 ** -7 + 2.0 ** -15 + n * 2.0 ** -23
    tot = np.abs(hw - x.astype(np.float64) @ qs.astype(np.float64).T)
    bound = gamma * np.linalg.norm(x.astype(np.float64), axis=1)[:, None] * np.linalg.norm(qs.astype(np.float64), axis=1)[None, :]
    assert np.all(tot <= bound + 1e-30), (tot / np.maximum(bound, 1e-30)).max()
    assert np.all(hw[80:90] == 0.0)


@pytest.mark.parametrize("kind,N,k,Q", [("cfg3", 30_000 + 5, 1, 300), ("cfg3", 20_000, 6, 70), ("cfg4", 60_000, 1, 90)])
def test_dense_pair_mode_identical(kind, N, k, Q):
    """the screen on CTA pairs (tcgen05 cta_group::2, M = 256, each CTA holding half of a query group)
    returns the same bits as the single-CTA screen, and both match the oracle"""
    w = datagen.scaled(datagen.WORKLOADS[kind], N, Q)
    x, q = _data(w)
    ix, d1, i1, st = _check(x, q, k, sample_size=datagen.default_sample_size(w), dense_permille=1000)
    assert st["dense_queries"] == Q
    ix.set_tuning(dense_pair=1)
    d2, i2, st2 = ix.knn(q, k, stats=True)
    assert st2["dense_queries"] == Q
    assert torch.equal(i1, i2) and torch.equal(d1, d2)


@pytest.mark.parametrize("kind,N,k,Q", [("cfg3", 30_000 + 5, 1, 300), ("cfg3", 20_000, 4, 600),
                                        ("cfg3", 12_000, 2, 1000), ("cfg3", 9_000, 1, 100)])
def test_dense_mcast_identical(kind, N, k, Q):
    """clusters of 2 sharing row tiles by TMA multicast (an even number of query groups: 300 -> 2,
    1000 -> 4), or not (600 -> 3 groups, 100 -> 1: clusters without multicast, the idle CTA kept for the
    cluster barriers) return the same bits as the cooperative one-CTA-per-worker launch"""
    w = datagen.scaled(datagen.WORKLOADS[kind], N, Q)
    x, q = _data(w)
    ix, d1, i1, st = _check(x, q, k, sample_size=datagen.default_sample_size(w), dense_permille=1000)
    assert st["dense_queries"] == Q
    ix.set_tuning(dense_mcast=0)
    d2, i2, st2 = ix.knn(q, k, stats=True)
    assert st2["dense_queries"] == Q
    assert torch.equal(i1, i2) and torch.equal(d1, d2)
