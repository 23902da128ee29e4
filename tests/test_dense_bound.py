"""CPU pin of the dense path's error bound (reading 29; csrc/dense.cu, csrc/query.cu).

The dense screen computes approx d^2 = |q^|^2 + |x^|^2 - 2 dot from a bf16 tensor-core dot product
of the z-normalised row (the build's bfloat16 copy of x^ = (x - mu) * inv, float32) with the
z-normalised query (bfloat16), |x^|^2 taken as n (0 for a constant row), and refines a row iff
approx - eps <= (a proven bound on the k-th best).  Exactness needs |approx - d2_refine| <= eps,
where d2_refine is what the exact refine computes (float32: e_t = ((x_t - mu) * inv) - q_t, sum of
e_t^2).  This test emulates bf16 operands (round to nearest even), exact products, float32
accumulation in sequential order, and checks the bound with the constants the kernels use
(query.cu: gamma = 2^-7 + 2^-15 + n 2^-23, eps = 2 gamma sqrt(1.0001 n) |q^| + 2e-4 (|q^|^2 + n) +
1e-3), on rows built to stress it: large offsets and scales, constant rows, near-duplicates of the
query, rows correlated and anti-correlated with it.  The tensor cores' own accumulation is measured
against the same bound on the GPU (tests/test_gpu_dense.py::test_dense_dots_within_bound).
"""
import numpy as np
import pytest


def bf16(a: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 (round to nearest, ties to even) -> float32"""
    b = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((b >> np.uint64(16)) & np.uint64(1)) + np.uint64(0x7FFF)
    return ((b + r) & np.uint64(0xFFFF0000)).astype(np.uint32).view(np.float32)


def row_stats_f32(x: np.ndarray):
    """float32 mean, float64-derived 1/sigma (population), as row_stats_g() in common.cuh."""
    x64 = x.astype(np.float64)
    mu = x64.mean(axis=1)
    muf = mu.astype(np.float32)
    var = ((x - muf[:, None]).astype(np.float64) ** 2).mean(axis=1)
    sd = np.sqrt(var)
    inv = np.where(sd < 1e-12, 0.0, 1.0 / np.where(sd < 1e-12, 1.0, sd)).astype(np.float32)
    return muf, inv


def zn_f32(x, muf, inv):
    return ((x - muf[:, None]).astype(np.float32) * inv[:, None]).astype(np.float32)


def refine_d2(xh, qh):
    e = (xh - qh[None, :]).astype(np.float32)
    return (e ** 2).sum(axis=1, dtype=np.float32).astype(np.float64)


def dense_eps(n, qh):
    """eps of reading 29 (query.cu, dense slot publish)"""
    nq = float(np.sum(qh.astype(np.float64) ** 2))
    gamma = 2.0 ** -7 + 2.0 ** -15 + n * 2.0 ** -23
    return 2.0 * gamma * np.sqrt(1.0001 * n) * np.sqrt(nq) + 2e-4 * (nq + n) + 1e-3, nq


def _rows(rng, q, n, m):
    base = np.cumsum(rng.normal(size=(m, n)), axis=1)
    scale = 10.0 ** rng.uniform(-3, 4, size=(m, 1))
    offset = rng.choice([0.0, 1.0, 1e3, -5e4], size=(m, 1)) * rng.uniform(0.5, 2, size=(m, 1))
    x = (base * scale + offset).astype(np.float32)
    x[:50] = (q[None, :] * rng.uniform(0.1, 100, size=(50, 1)) + rng.normal(size=(50, 1)) * 10).astype(np.float32)
    x[50:60] = (q[None, :] + rng.normal(scale=1e-3, size=(10, n))).astype(np.float32)   # near-duplicates
    x[60:70] = (-q[None, :] + rng.normal(scale=1e-2, size=(10, n))).astype(np.float32)  # anti-correlated
    x[70:80] = rng.uniform(-5, 5, size=(10, 1)).astype(np.float32)                      # constant rows
    return x


@pytest.mark.parametrize("n", [64, 256, 1024])
def test_bf16_screen_bound_holds(n):
    rng = np.random.default_rng(n)
    m = 3000
    q = np.cumsum(rng.normal(size=n)).astype(np.float32)
    qmu, qinv = row_stats_f32(q[None, :])
    qh = zn_f32(q[None, :], qmu, qinv)[0]
    x = _rows(rng, q, n, m)
    muf, inv = row_stats_f32(x)
    xh = zn_f32(x, muf, inv)
    eps, nq = dense_eps(n, qh)
    xn = np.where(inv > 0, float(n), 0.0)
    prod = bf16(qh)[None, :].astype(np.float64) * bf16(xh).astype(np.float64)  # exact products
    dot_seq = np.zeros(m, dtype=np.float32)
    for t in range(n):  # float32 sequential accumulation
        dot_seq = (dot_seq + prod[:, t].astype(np.float32)).astype(np.float32)
    ref = refine_d2(xh, qh)
    for dot in (dot_seq.astype(np.float64), prod.sum(axis=1)):
        # epilogue arithmetic (float32): val = 2 dot + (thr + eps - |q^|^2) >= |x^|^2
        a = (np.float32(nq) + xn.astype(np.float32)) - np.float32(2.0) * dot.astype(np.float32)
        err = np.abs(a.astype(np.float64) - ref)
        assert np.all(err <= eps), (err / eps).max()
        assert (err / eps).max() > 0.02  # the rows reach a visible part of the window
    assert eps < 0.05 * np.median(ref[inv > 0])  # ... which is small next to typical distances


def test_bound_window_at_n256():
    """on z-normalised data eps is ~4.1 in d^2 at n = 256 (a candidate window of 2 eps ~ 8 above the
    k-th best), small next to the typical distances of the workloads (k-th best d^2 ~ 150-1200 for the
    queries that go dense: SURVEY SIM-10, SIM-c5)"""
    n = 256
    qh = np.random.default_rng(0).normal(size=n).astype(np.float32)
    qh = (qh - qh.mean()) / qh.std()
    eps, _ = dense_eps(n, qh)
    assert 3.5 < eps < 4.5
