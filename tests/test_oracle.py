"""Pins for the CPU oracle (oracle/sofa_oracle.py) against things other than itself:
printed/derived worked examples (tests/golden/), closed forms (Parseval, z-norm moments),
a naive O(n^2) DFT written from the definition, pure-Python brute force on tiny inputs,
the LB <= ED invariant (Eq. 1 / d_SFA), and known answers of the noisy-member
workloads (SURVEY 8(c) "Noisy-member queries")."""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import sofa_oracle as O
from paper_2411_17483_b200 import datagen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def _rw(N, n, seed):
    w = datagen.scaled(datagen.WORKLOADS["cfg1"], N, 4, length=n, seed=seed)
    return datagen.generate_rows(w, 0, N).numpy()


def _hf(N, n, seed):
    w = datagen.scaled(datagen.WORKLOADS["cfg3"], N, 4, length=n, seed=seed)
    return datagen.generate_rows(w, 0, N).numpy()


def naive_dft_interleaved(x):
    """X_k = n^-1/2 sum_t x_t (cos(2 pi k t/n) - i sin(2 pi k t/n)), explicit loops."""
    n = len(x)
    out = []
    for k in range(n // 2 + 1):
        re = sum(x[t] * math.cos(2 * math.pi * k * t / n) for t in range(n)) / math.sqrt(n)
        im = -sum(x[t] * math.sin(2 * math.pi * k * t / n) for t in range(n)) / math.sqrt(n)
        out += [re, im]
    return np.array(out)


# ------------------------------------------------------------------ z-norm (Def. 2)
def test_znorm_golden():
    g = GOLD["znorm"]
    xh, mu, sd, fl = O.znorm(np.array(g["x"]))
    np.testing.assert_allclose(xh, g["expected"], atol=1e-15)
    assert mu == g["mu"] and sd == g["sigma"] and not fl


def test_znorm_constant_and_moments():
    xh, mu, sd, fl = O.znorm(np.ones((1, 8)))
    assert fl[0] and sd[0] == 0 and np.all(xh == 0)
    x = np.random.default_rng(0).normal(3.0, 5.0, size=(50, 37))
    xh, _, _, _ = O.znorm(x)
    np.testing.assert_allclose(xh.mean(axis=1), 0, atol=1e-12)
    np.testing.assert_allclose(np.sqrt((xh ** 2).mean(axis=1)), 1, atol=1e-12)


# ------------------------------------------------------------------ DFT (reading 2)
def test_dft_golden_alternating():
    g = GOLD["dft_alternating"]
    np.testing.assert_allclose(O.spectrum(np.array(g["x"]))[0], g["expected_interleaved"], atol=1e-12)


@pytest.mark.parametrize("n", [4, 5, 8, 16, 64])
def test_spectrum_equals_naive_dft(n):
    x = np.random.default_rng(n).normal(size=n)
    np.testing.assert_allclose(O.spectrum(x)[0], naive_dft_interleaved(x), atol=1e-10)


@pytest.mark.parametrize("n", [4, 7, 256, 1024])
def test_parseval_weighted_energy_is_n(n):
    """Sum_pos w_pos X_pos^2 over the whole interleaved spectrum = sum x^2 = n (z-normed)."""
    x = np.random.default_rng(n).normal(size=(20, n))
    xh, _, _, _ = O.znorm(x)
    spec = O.spectrum(xh)
    w = O.position_weights(np.arange(spec.shape[1]), n)
    np.testing.assert_allclose((spec ** 2 * w).sum(axis=1), n, rtol=1e-12)
    assert np.abs(spec[:, 0]).max() < 1e-12            # DC of a z-normed series
    assert np.abs(spec[:, 1]).max() == 0.0
    if n % 2 == 0:
        assert np.abs(spec[:, n + 1]).max() < 1e-12    # Im of Nyquist


def test_full_spectrum_weighted_distance_is_ed2():
    """Eq. 1 with all positions is an equality."""
    n = 64
    x = np.random.default_rng(1).normal(size=(30, n))
    xh, _, _, _ = O.znorm(x)
    spec = O.spectrum(xh)
    w = O.position_weights(np.arange(spec.shape[1]), n)
    d_spec = ((spec[:15] - spec[15:]) ** 2 * w).sum(axis=1)
    d_ed = ((xh[:15] - xh[15:]) ** 2).sum(axis=1)
    np.testing.assert_allclose(d_spec, d_ed, rtol=1e-12)


def test_eligible_positions_and_weights():
    assert list(O.eligible_positions(8)) == [2, 3, 4, 5, 6, 7, 8]
    assert list(O.eligible_positions(7)) == [2, 3, 4, 5, 6, 7]
    assert list(O.eligible_positions(256, 2)) == [2, 3, 4, 5]
    assert list(O.position_weights([2, 3, 8, 0], 8)) == [2, 2, 1, 1]


# ------------------------------------------------------------------ selection (Alg. 1 l.5)
def test_mean_selected_index_golden():
    g = GOLD["mean_selected_index"]
    pos = [2 * k for k in g["complex_indices"]]
    assert O.mean_selected_index(pos) == g["expected"]


def test_select_unique_max_and_ties():
    spec = np.zeros((10, 12))
    spec[:, 5] = np.arange(10)
    elig = np.arange(2, 12)
    assert list(O.select_by_variance(spec, elig, 1)) == [5]
    spec = np.tile(np.array([1.0, -1.0])[:, None], (5, 12))   # every position equal variance
    assert list(O.select_by_variance(spec, elig, 3)) == [2, 3, 4]


def test_random_walk_selects_low_frequencies():
    """Random walks have ~1/k^2 spectra: the top-16 positions are Re/Im of k <= 9 (SIM-2)."""
    x = _rw(4000, 256, 11)
    m = O.learn_model(x, 16, 256)
    assert (m["best_pos"] // 2).max() <= 9 and (m["best_pos"] // 2).min() >= 1


def test_high_frequency_selects_band_and_nyquist_weight():
    x = _hf(4000, 256, 12)
    m = O.learn_model(x, 16, 256)
    k = m["best_pos"] // 2
    assert k.min() >= 20       # band [32,128] cycles (+leakage), never the low-pass pick
    assert np.all(m["weights"][k == 128] == 1.0)


# ------------------------------------------------------------------ binning
def test_equi_depth_golden():
    g = GOLD["equi_depth"]
    np.testing.assert_array_equal(O.equi_depth_edges(np.array(g["values"][::-1]), g["a"]), g["expected"])


def test_equi_width_golden():
    g = GOLD["equi_width"]
    np.testing.assert_allclose(O.equi_width_edges(np.array(g["values"]), g["a"]), g["expected"])


@pytest.mark.parametrize("S,a", [(1000, 4), (4096, 256), (10007, 256)])
def test_equi_depth_bins_hold_S_over_a(S, a):
    v = np.random.default_rng(S).normal(size=S)
    e = O.equi_depth_edges(v, a)
    m = {"edges": e[None, :], "a": a}
    counts = np.bincount(O.quantize(v[:, None], m)[:, 0], minlength=a)
    assert counts.min() >= S // a - 1 and counts.max() <= S // a + 1 + (S % a > 0)


# ------------------------------------------------------------------ symbols (Alg. 2)
def test_symbols_on_edge_go_right_and_match_linear_scan():
    e = np.array([-1.0, 0.0, 2.0])
    m = {"edges": e[None, :], "a": 4}
    v = np.array([-5.0, -1.0, -0.5, 0.0, 1.0, 2.0, 9.0])
    sym = O.quantize(v[:, None], m)[:, 0]
    assert list(sym) == [0, 1, 1, 2, 2, 3, 3]
    vals = np.random.default_rng(3).normal(size=500)
    lin = np.array([sum(1 for b in e if b <= x) for x in vals])
    assert np.array_equal(O.quantize(vals[:, None], m)[:, 0], lin)


# ------------------------------------------------------------------ lower bounds (d_SFA, mind)
@pytest.mark.parametrize("case", ["mind_upper", "mind_lower", "mind_inside"])
def test_mind_golden(case):
    g = GOLD[case]
    assert O.mind(g["q"], g["lo"], g["hi"]) == pytest.approx(g["expected"], abs=1e-15)


@pytest.mark.parametrize("kind", ["rw", "hf"])
def test_lb_never_exceeds_ed2_and_own_word_is_zero(kind):
    gen = _rw if kind == "rw" else _hf
    x = gen(3000, 128, 21)
    m = O.learn_model(x[:2000], 16, 256)
    words = O.sfa_words(x, m)
    xh, _, _, _ = O.znorm(x)
    q = gen(8, 128, 99)
    qh, _, _, _ = O.znorm(q)
    qp = O.project(q, m)
    total = 0
    for i in range(q.shape[0]):
        lb = O.lb_word(qp[i], words, m)
        ed2 = O.sq_dists_direct(xh, qh[i])
        assert np.all(lb <= ed2 * (1 + 1e-12) + 1e-9)
        total += len(lb)
    assert total >= 10_000
    own = O.project(x[:50], m)
    for i in range(50):
        assert O.lb_word(own[i], words[i:i + 1], m)[0] == 0.0


def test_envelope_lb_below_member_lb():
    x = _rw(2048, 64, 5)
    m = O.learn_model(x, 8, 16)
    words = O.sfa_words(x, m).astype(np.int64)
    qp = O.project(_rw(4, 64, 6), m)
    for b in range(0, 2048, 256):
        blk = words[b:b + 256]
        for i in range(qp.shape[0]):
            env = O.lb_envelope(qp[i], blk.min(axis=0), blk.max(axis=0), m)[0]
            assert env <= O.lb_word(qp[i], blk, m).min() + 1e-15


def test_lb_with_small_alphabet_and_equi_width():
    x = _rw(1500, 32, 8)
    for binning in ("equi-depth", "equi-width"):
        m = O.learn_model(x[:500], 6, 4, binning=binning)
        words = O.sfa_words(x, m)
        xh, _, _, _ = O.znorm(x)
        qp = O.project(x[:3] + 0.3, m)
        qh, _, _, _ = O.znorm(x[:3] + 0.3)
        for i in range(3):
            assert np.all(O.lb_word(qp[i], words, m) <= O.sq_dists_direct(xh, qh[i]) + 1e-9)


# ------------------------------------------------------------------ k-NN
def _py_knn(data, q, k):
    def zn(v):
        mu = sum(v) / len(v)
        sd = math.sqrt(sum((a - mu) ** 2 for a in v) / len(v))
        return [(a - mu) / sd for a in v]
    qq = zn(list(q))
    ds = []
    for i, row in enumerate(data):
        r = zn(list(row))
        ds.append((sum((a - b) ** 2 for a, b in zip(r, qq)), i))
    ds.sort()
    return [math.sqrt(d) for d, _ in ds[:k]], [i for _, i in ds[:k]]


@pytest.mark.parametrize("N,n,k", [(1, 4, 1), (2, 8, 1), (7, 16, 3), (100, 16, 5), (300, 32, 300)])
def test_bruteforce_equals_python_loops(N, n, k):
    rng = np.random.default_rng(N * n)
    data = rng.normal(size=(N, n)).astype(np.float32)
    qs = rng.normal(size=(3, n)).astype(np.float32)
    d, i = O.knn_bruteforce(data, qs, k, chunk=64)
    for r in range(3):
        pd, pi = _py_knn(data.astype(np.float64), qs[r].astype(np.float64), k)
        np.testing.assert_allclose(d[r], pd, rtol=1e-12)
        assert list(i[r]) == pi


def test_bruteforce_query_in_corpus_duplicates_and_padding():
    rng = np.random.default_rng(4)
    data = rng.normal(size=(50, 16)).astype(np.float32)
    data[30] = data[7]
    d, i = O.knn_bruteforce(data, data[[7, 12]], 2)
    assert d[0, 0] == 0 and d[0, 1] == 0 and list(i[0]) == [7, 30]   # tie -> smaller index
    assert d[1, 0] == 0 and i[1, 0] == 12
    d, i = O.knn_bruteforce(data[:3], data[:1], 5)
    assert list(i[0, 3:]) == [-1, -1] and np.all(np.isinf(d[0, 3:]))


def _chunks(data, sizes):
    s = 0
    for c in sizes:
        yield s, data[s:s + c]
        s += c


@pytest.mark.parametrize("N,n,k,sizes,gemm", [(1, 4, 1, [1], 8), (7, 16, 3, [2, 5], 3), (100, 16, 5, [33, 0, 67], 16),
                                              (300, 32, 300, [100, 100, 100], 64), (257, 8, 4, [1, 255, 1], 7)])
def test_stream_bruteforce_equals_python_loops(N, n, k, sizes, gemm):
    """the streamed brute force (chunked rows, float64 GEMM shortlist + exact direct sums) against
    the pure-Python definition, including empty chunks, k = N and k above a chunk's size"""
    rng = np.random.default_rng(N * n + k)
    data = rng.normal(size=(N, n)).astype(np.float32)
    qs = rng.normal(size=(3, n)).astype(np.float32)
    d, i = O.knn_bruteforce_stream(_chunks(data, sizes), qs, k, rows_per_gemm=gemm)
    for r in range(3):
        pd, pi = _py_knn(data.astype(np.float64), qs[r].astype(np.float64), k)
        np.testing.assert_allclose(d[r, :len(pd)], pd, rtol=1e-12)
        assert list(i[r, :len(pi)]) == pi


def test_stream_bruteforce_ties_across_chunks_and_padding():
    """exact duplicates in different chunks -> smaller index first; a constant row -> zero vector;
    k above N pads with (+inf, -1); agrees with knn_bruteforce on a random-walk set"""
    rng = np.random.default_rng(12)
    data = np.cumsum(rng.normal(size=(500, 64)), axis=1).astype(np.float32)
    data[420] = data[17]
    data[421] = 5.0
    qs = np.concatenate([data[[17, 421]], np.cumsum(rng.normal(size=(4, 64)), axis=1).astype(np.float32)])
    d, i = O.knn_bruteforce_stream(_chunks(data, [100, 300, 100]), qs, 3, rows_per_gemm=64)
    assert list(i[0, :2]) == [17, 420] and d[0, 0] == 0 and d[0, 1] == 0
    assert i[1, 0] == 421 and d[1, 0] == 0   # constant query vs constant row: both zero vectors
    d2, i2 = O.knn_bruteforce(data, qs, 3)
    np.testing.assert_allclose(d, d2, rtol=1e-12)
    keep = [0, 2, 3, 4, 5]   # (the constant query ties every row at d^2 = n up to float64 rounding)
    assert np.array_equal(i[keep], i2[keep])
    d3, i3 = O.knn_bruteforce_stream(_chunks(data[:2], [2]), qs[:1], 4)
    assert list(i3[0, 2:]) == [-1, -1] and np.all(np.isinf(d3[0, 2:]))


@pytest.mark.parametrize("n,l,a,k", [(16, 4, 4, 1), (32, 8, 16, 3), (64, 16, 256, 1), (64, 16, 256, 10)])
def test_gemini_equals_bruteforce(n, l, a, k):
    x = _rw(1200, n, n + l)
    m = O.learn_model(x[::4], l, a)
    q = np.concatenate([_rw(5, n, 77), x[:2] + 0.05])
    d1, i1 = O.knn_bruteforce(x, q, k)
    d2, i2, refined = O.knn_gemini(x, q, k, m)
    np.testing.assert_allclose(d1, d2, rtol=1e-12)
    assert np.array_equal(i1, i2)
    assert refined.mean() < x.shape[0]


@pytest.mark.parametrize("sigma", [0.01, 0.1])
def test_noisy_member_known_answer(sigma):
    """for sigma <= 0.1 the 1-NN of a noisy member is its source row, at
    d^2 ~ n[(1-1/s)^2 + sigma^2/s^2], s = sqrt(1+sigma^2)."""
    w = datagen.scaled(datagen.WORKLOADS["cfg2"], 20_000, 12, noise_sigmas=(sigma,))
    data = datagen.generate_rows(w, 0, w.n_series)
    q = datagen.generate_queries(w, data=data)
    d, i = O.knn_bruteforce(data.numpy(), q.numpy(), 1)
    assert np.array_equal(i[:, 0], datagen.query_sources(w))
    s = math.sqrt(1 + sigma ** 2)
    pred = 256 * ((1 - 1 / s) ** 2 + sigma ** 2 / s ** 2)
    assert np.median(d[:, 0] ** 2) == pytest.approx(pred, rel=0.25)


def test_merge_topk_equals_global():
    rng = np.random.default_rng(9)
    data = rng.normal(size=(90, 16)).astype(np.float32)
    qs = rng.normal(size=(4, 16)).astype(np.float32)
    d, i = O.knn_bruteforce(data, qs, 5)
    parts = [(0, 40), (40, 41), (41, 90)]
    pd, pi = [], []
    for a, b in parts:
        dd, ii = O.knn_bruteforce(data[a:b], qs, 5)
        pd.append(dd)
        pi.append(np.where(ii >= 0, ii + a, -1))
    md, mi = O.merge_topk(np.stack(pd), np.stack(pi), 5)
    np.testing.assert_allclose(md, d)
    assert np.array_equal(mi, i)


def test_sample_indices():
    s = O.sample_indices(100, 7)
    assert list(s) == [0, 14, 28, 42, 57, 71, 85]
    assert len(np.unique(O.sample_indices(10_000_000, 100_000))) == 100_000


# ------------------------------------------------------------------ iSAX baseline, SURVEY 8(f) f4
@pytest.mark.parametrize("key", ["isax_breakpoints_a4", "isax_breakpoints_a2"])
def test_isax_breakpoints_golden(key):
    g = GOLD[key]
    np.testing.assert_allclose(O.isax_breakpoints(g["a"]), g["expected"], atol=g["abs_tol"])


@pytest.mark.parametrize("a", [4, 16, 256])
def test_isax_breakpoints_equal_depth_and_symmetric(a):
    b = O.isax_breakpoints(a)
    assert np.all(np.diff(b) > 0)
    np.testing.assert_allclose(b, -b[::-1], atol=1e-9)
    # equal depth under N(0,1): each bin holds 1/a of a large normal sample (Monte Carlo, 4 sigma)
    z = np.random.default_rng(a).normal(size=400_000)
    counts = np.bincount(np.searchsorted(b, z, side="right"), minlength=a) / z.size
    assert np.all(np.abs(counts - 1 / a) < 4 * np.sqrt(1 / a / z.size) + 1e-12)


@pytest.mark.parametrize("key", ["paa_two_segments", "paa_alternating_flat"])
def test_paa_golden(key):
    g = GOLD[key]
    np.testing.assert_allclose(O.paa(np.array(g["x"]), g["l"])[0], g["expected"], atol=1e-15)


def test_isax_mindist_lower_bounds_ed_and_own_word_is_zero():
    """n/l * sum mind^2 <= ED^2 (PAA contraction + mind <= |paa difference|) on >= 10k pairs"""
    x = _rw(2500, 128, 31)
    m = O.isax_model(128, 16, 256)
    words = O.sfa_words(x, m)
    xh, _, _, _ = O.znorm(x)
    q = _rw(6, 128, 32)
    qh, _, _, _ = O.znorm(q)
    qp = O.project(q, m)
    for i in range(q.shape[0]):
        assert np.all(O.lb_word(qp[i], words, m) <= O.sq_dists_direct(xh, qh[i]) * (1 + 1e-12) + 1e-9)
    own = O.project(x[:40], m)
    for i in range(40):
        assert O.lb_word(own[i], words[i:i + 1], m)[0] == 0.0
    # PAA contraction itself: (n/l) |paa(x) - paa(q)|^2 <= |x - q|^2
    px, pq = O.paa(xh, 16), O.paa(qh, 16)
    assert np.all(8.0 * ((px - pq[0]) ** 2).sum(axis=1) <= O.sq_dists_direct(xh, qh[0]) + 1e-9)


def test_isax_flat_on_high_frequency_sfa_is_not():
    """Fig. 1: on high-frequency series the PAA is nearly flat, so the iSAX bound is far
    looser than SFA's (mean TLB), the paper's motivation for learned summaries"""
    x = _hf(1500, 256, 41)
    q = _hf(6, 256, 42)
    xh, _, _, _ = O.znorm(x)
    qh, _, _, _ = O.znorm(q)
    sfa = O.learn_model(x, 16, 256)
    isx = O.isax_model(256, 16, 256)
    tlb = {}
    for name, m in (("sfa", sfa), ("isax", isx)):
        words, qp = O.sfa_words(x, m), O.project(q, m)
        r = [np.sqrt(O.lb_word(qp[i], words, m) / O.sq_dists_direct(xh, qh[i])).mean() for i in range(6)]
        tlb[name] = float(np.mean(r))
    assert tlb["isax"] < 0.1 and tlb["sfa"] > 2 * tlb["isax"], tlb
