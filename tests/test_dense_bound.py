"""CPU pin of the dense path's error bound (reading 29; csrc/dense.cu, csrc/query.cu).

The dense screen computes approx d^2 = |q^|^2 + |x^|^2 - 2 inv (q^.x - mu sum q^) from a TF32
tensor-core dot product of the z-normalised query with the RAW row, and refines a row iff
approx - eps <= (a proven bound on the k-th best).  Exactness needs |approx - d2_refine| <= eps,
where d2_refine is what the exact refine computes (float32: e_t = ((x_t - mu) * inv) - q_t,
sum of e_t^2).  This test emulates TF32 operands (10 explicit mantissa bits, by truncation and by
round-to-nearest), float32 accumulation in the worst order for cancellation, and checks the
bound with the same constants the kernels use, on rows built to stress it: large offsets and
scales, constant rows, near-duplicates of the query.
"""
import numpy as np
import pytest


def tf32(a: np.ndarray, mode: str) -> np.ndarray:
    b = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    if mode == "rn":
        b = b + np.uint32(0x1000)  # round half up on the 13 dropped bits
    return (b & np.uint32(0xFFFFE000)).view(np.float32)


def row_stats_f32(x: np.ndarray):
    """float32 mean, float64-derived 1/sigma (population), as row_stats() in common.cuh."""
    x64 = x.astype(np.float64)
    mu = x64.mean(axis=1)
    muf = mu.astype(np.float32)
    var = ((x - muf[:, None]).astype(np.float64) ** 2).mean(axis=1)
    sd = np.sqrt(var)
    inv = np.where(sd < 1e-12, 0.0, 1.0 / np.where(sd < 1e-12, 1.0, sd)).astype(np.float32)
    return muf, inv


def refine_d2(x, muf, inv, qh):
    e = ((x - muf[:, None]).astype(np.float32) * inv[:, None]).astype(np.float32) - qh[None, :]
    return (e.astype(np.float32) ** 2).sum(axis=1, dtype=np.float32).astype(np.float64)


def dense_eps(n, qh, muf, inv):
    """eps of reading 29, per row (the kernel uses the maximum over a tile's rows)."""
    nq = float(np.sum(qh.astype(np.float64) ** 2))
    sq = float(np.sum(qh.astype(np.float64)))
    gamma = 1.05 * 2.0 ** -9 + n * 2.0 ** -22
    kq = 2.0 * gamma * np.sqrt(nq) * 1.0001
    mi = muf.astype(np.float64) * inv
    e_s = np.where(inv > 0, np.sqrt(n * (1 + mi * mi)) * 1.0001, 0.0)
    c_s = np.where(inv > 0, n, 0.0)
    r_s = np.where(inv > 0, 2.4e-7 * e_s * e_s + 2e-4 * n, 0.0)
    return kq * e_s + (2e-4 * nq + 1e-3) + r_s + abs(sq) * np.abs(2 * mi), nq, sq, c_s


@pytest.mark.parametrize("n", [64, 256, 1024])
@pytest.mark.parametrize("mode", ["trunc", "rn"])
def test_tf32_screen_bound_holds(n, mode):
    rng = np.random.default_rng(n + (mode == "rn"))
    m = 3000
    q = np.cumsum(rng.normal(size=n)).astype(np.float32)
    qmu, qinv = row_stats_f32(q[None, :])
    qh = ((q - qmu[0]) * qinv[0]).astype(np.float32)
    base = np.cumsum(rng.normal(size=(m, n)), axis=1)
    scale = 10.0 ** rng.uniform(-3, 4, size=(m, 1))
    offset = rng.choice([0.0, 1.0, 1e3, -5e4], size=(m, 1)) * rng.uniform(0.5, 2, size=(m, 1))
    x = (base * scale + offset).astype(np.float32)
    x[:50] = (q[None, :] * rng.uniform(0.1, 100, size=(50, 1)) + rng.normal(size=(50, 1)) * 10).astype(np.float32)
    x[50:60] = x[60:70] + rng.normal(scale=1e-3, size=(10, n)).astype(np.float32)
    x[70:80] = rng.uniform(-5, 5, size=(10, 1)).astype(np.float32)  # constant rows
    muf, inv = row_stats_f32(x)
    eps, nq, sq, c_s = dense_eps(n, qh, muf, inv)
    # TF32 products accumulated in float32, sequentially (the accumulation order the bound assumes
    # nothing about); plus the pairwise float64 sum for reference
    prod = tf32(qh, mode)[None, :].astype(np.float64) * tf32(x, mode).astype(np.float64)
    dot_seq = np.zeros(m, dtype=np.float32)
    for t in range(n):
        dot_seq = (dot_seq + prod[:, t].astype(np.float32)).astype(np.float32)
    ref = refine_d2(x, muf, inv, qh)
    for dot in (dot_seq.astype(np.float64), prod.sum(axis=1)):
        # epilogue arithmetic in float32: approx' = -2 inv dot + (|q^|^2 + |x^|^2); the + 2 mu inv sum(q^)
        # term is dropped and covered by eps (its last term)
        a = (np.float32(-2.0) * inv).astype(np.float32) * dot.astype(np.float32) + np.float32(nq) + c_s.astype(np.float32)
        err = np.abs(a.astype(np.float64) - ref)
        assert np.all(err <= eps), (err / eps).max()
        assert (err / eps).max() < 0.9  # the bound is not vacuous at its edge ...
    assert np.median(eps[inv > 0][80:]) < 0.05 * np.median(ref[inv > 0][80:])  # ... nor loose for normal rows


def test_bound_is_tight_enough_to_screen():
    """on z-normalised data the window is ~1 in d^2 (n = 256), far below typical NN gaps"""
    n = 256
    qh = np.random.default_rng(0).normal(size=n).astype(np.float32)
    qh = (qh - qh.mean()) / qh.std()
    eps, *_ = dense_eps(n, qh, np.zeros(4, np.float32), np.ones(4, np.float32))
    assert 0.5 < eps[0] < 1.5
