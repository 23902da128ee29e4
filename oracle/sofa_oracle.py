"""CPU float64 ORACLE for SOFA's exact Euclidean k-NN path (arxiv 2411.17483).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
cpu_baseline / `--impl reference` leg may import this module.  The product path
(`paper_2411_17483_b200`, `libsofa.so`) never imports, links or calls it, and this
module imports nothing from the product path.

Plain, slow, obviously-correct numpy float64, written step by step in the paper's order.
Citations are PAPER.md line numbers (`P:<line>`) plus section / equation / algorithm;
readings where the paper is silent or garbled are numbered as in SURVEY.md 8(c) and
restated in DESIGN.md "Readings".

What each part computes (and what pins it, tests/test_oracle.py):
  znorm            Def. 2, population std (reading 1)       pinned: closed forms
  spectrum         DFT, orthonormal, e^{-2 pi i k t/n} (reading 2)    pinned: naive DFT, Parseval
  eligible/weights Eq. 1 generalised per position (reading 10) pinned: Parseval = n
  learn_model      Alg. 1: sample -> DFT -> variance top-l
                   (reading 5) -> per-position bins
                   (equi-depth, reading 8; equi-width, Alg. 1 l.8-11)  pinned: SPEC examples, bin counts
  symbols          Alg. 2, bins [b(a-1), b(a)) pinned: on-edge, binary==linear
  mind / lb_word   d_SFA + mind_i, squared, weighted        pinned: LB <= ED^2, LB(own)=0
  lb_envelope      leaf LB of a block, reading 10           pinned: env LB <= member LB
  knn_bruteforce   NN definition (reading 14), k-NN       pinned: pure-python loops,
                                                                         noisy-member known answers
  knn_bruteforce_stream  the same, over row chunks (torch CPU float64)  pinned: == pure-python loops,
                                                                         chunk-boundary ties
  knn_gemini       GEMINI filter+refine              pinned: == brute force
  paa / isax_*     the iSAX baseline: PAA segments, N(0,1)  pinned: textbook breakpoints,
                   breakpoints, mindist weight n/l                      PAA closed forms, LB <= ED^2
Nothing here is "parity unpinned".
"""
from __future__ import annotations

import numpy as np

F64 = np.float64


# ----------------------------------------------------------------------------- a1 z-norm
def znorm(x: np.ndarray):
    """Def. 2: (x - mu) / sigma per row, population std (reading 1).

    Returns (xhat float64, mu, sigma, degenerate_flag).  sigma < 1e-12 -> all-zero row,
    flagged, not fatal (reading / S:44).
    """
    x = np.asarray(x, dtype=F64)
    if x.ndim == 1:
        xh, mu, sd, fl = znorm(x[None, :])
        return xh[0], mu[0], sd[0], fl[0]
    mu = x.mean(axis=1)
    sd = np.sqrt(((x - mu[:, None]) ** 2).mean(axis=1))
    flag = sd < 1e-12
    safe = np.where(flag, 1.0, sd)
    xh = (x - mu[:, None]) / safe[:, None]
    xh[flag] = 0.0
    return xh, mu, np.where(flag, 0.0, sd), flag


# ----------------------------------------------------------------------------- spectrum
def spectrum(xhat: np.ndarray) -> np.ndarray:
    """Full orthonormal DFT, interleaved (reading 2).

    X_k = n^{-1/2} sum_{t=0}^{n-1} x_t e^{-2 pi i k t / n}, k = 0..n//2 (numpy.fft.rfft,
    norm="ortho"); position 2k = Re X_k, 2k+1 = Im X_k.  Shape (N, 2*(n//2+1)).
    """
    xhat = np.atleast_2d(np.asarray(xhat, dtype=F64))
    X = np.fft.rfft(xhat, axis=1, norm="ortho")
    out = np.empty((xhat.shape[0], 2 * X.shape[1]), dtype=F64)
    out[:, 0::2] = X.real
    out[:, 1::2] = X.imag
    return out


def eligible_positions(n: int, candidate_limit: int = 0) -> np.ndarray:
    """Positions a variance selection may pick (reading 3).

    Re and Im of k = 1..(n-1)//2, plus Re of the Nyquist bin k = n/2 for even n.  DC is
    excluded (both parts are 0 after z-norm) and so is Im of Nyquist (always 0).
    candidate_limit > 0 keeps only complex indices k <= candidate_limit.
    """
    kmax = n // 2
    pos = []
    for k in range(1, kmax + 1):
        if candidate_limit and k > candidate_limit:
            break
        if n % 2 == 0 and k == kmax:
            pos.append(2 * k)
        else:
            pos.extend([2 * k, 2 * k + 1])
    return np.array(pos, dtype=np.int64)


def position_weights(positions, n: int) -> np.ndarray:
    """Eq. 1 weights per position (reading 10): 1 for DC and Nyquist, 2 otherwise."""
    positions = np.asarray(positions, dtype=np.int64)
    k = positions // 2
    w = np.full(positions.shape, 2.0, dtype=F64)
    w[k == 0] = 1.0
    if n % 2 == 0:
        w[k == n // 2] = 1.0
    return w


def mean_selected_index(positions) -> float:
    """Mean complex-coefficient index of a selection."""
    return float(np.mean(np.asarray(positions, dtype=np.int64) // 2))


# ----------------------------------------------------------------------------- a2 MCB learning
def sample_indices(n_total: int, s: int) -> np.ndarray:
    """Alg. 1 l.2 `sample(X, r)`: deterministic strided rows floor(j*N/S) (reading 6)."""
    j = np.arange(s, dtype=np.int64)
    return (j * n_total) // s


def select_by_variance(spec_sample: np.ndarray, eligible: np.ndarray, l: int) -> np.ndarray:
    """Alg. 1 l.5, P:248-250 (reading 5): the l eligible positions with the largest
    sample variance (ddof=1) across the sample's series; order = descending variance, ties
    to the lower position (reading 9)."""
    if l > len(eligible):
        raise ValueError("l exceeds the number of eligible positions")
    var = np.var(spec_sample[:, eligible], axis=0, ddof=1)
    order = np.lexsort((eligible, -var))
    return eligible[order[:l]].astype(np.int64)


def equi_depth_edges(values: np.ndarray, a: int) -> np.ndarray:
    """Equi-depth bins (reading 8): beta(i) = sorted[ceil(i*S/a)], i=1..a-1."""
    v = np.sort(np.asarray(values, dtype=F64))
    s = v.shape[0]
    if s < a:
        raise ValueError("equi-depth needs at least `alphabet` sample values")
    ranks = [(i * s + a - 1) // a for i in range(1, a)]
    return v[ranks]


def equi_width_edges(values: np.ndarray, a: int) -> np.ndarray:
    """Equi-width bins, Alg. 1 l.8-11: min + i*(max-min)/a, i=1..a-1."""
    v = np.asarray(values, dtype=F64)
    lo, hi = float(v.min()), float(v.max())
    return np.array([lo + i * (hi - lo) / a for i in range(1, a)], dtype=F64)


def learn_model(sample: np.ndarray, l: int, a: int, binning: str = "equi-depth",
                candidate_limit: int = 0) -> dict:
    """Alg. 1 MCB on an already drawn sample (S x n, rows as given).

    Step 1: DFT of the z-normalised sample (l.3).  Step 2: best_l by variance (l.5).
    Step 3: one bin row per selected position (l.8-11).  Returns a dict with n, l, a,
    best_pos (interleaved positions, descending variance), edges (l x (a-1) float64),
    weights (l,).
    """
    sample = np.asarray(sample)
    n = sample.shape[1]
    xh, _, _, _ = znorm(sample)
    spec = spectrum(xh)
    best = select_by_variance(spec, eligible_positions(n, candidate_limit), l)
    fn = equi_depth_edges if binning == "equi-depth" else equi_width_edges
    edges = np.stack([fn(spec[:, p], a) for p in best]) if a > 1 else np.zeros((l, 0))
    return {"n": n, "l": l, "a": a, "best_pos": best, "edges": edges,
            "weights": position_weights(best, n), "binning": binning}


# ----------------------------------------------------------------------------- iSAX baseline (f4)
def paa(xhat: np.ndarray, l: int) -> np.ndarray:
    """Segmentation + aggregation: means of l segments of equal length n/l."""
    xhat = np.atleast_2d(np.asarray(xhat, dtype=F64))
    m, n = xhat.shape
    if n % l:
        raise ValueError("iSAX needs n % l == 0")
    return xhat.reshape(m, l, n // l).mean(axis=2)


def isax_breakpoints(a: int) -> np.ndarray:
    """Fixed quantization: equal-depth bins of N(0,1), beta_i = Phi^-1(i/a)."""
    from scipy.stats import norm
    return norm.ppf(np.arange(1, a) / a)


def isax_model(n: int, l: int, a: int) -> dict:
    """The iSAX summarization as a model: positions = PAA segments, the same breakpoints for every
    segment, mindist weight n/l per segment (SAX mindist = sqrt(n/l) sqrt(sum dist^2))."""
    e = isax_breakpoints(a)
    return {"n": n, "l": l, "a": a, "best_pos": np.arange(l), "edges": np.stack([e] * l),
            "weights": np.full(l, n / l), "binning": "isax"}


# ----------------------------------------------------------------------------- a3 SFA transform
def project(x: np.ndarray, model: dict) -> np.ndarray:
    """Alg. 2 l.2-3: DFT of the z-normalised series, keep best_l positions
    (for the iSAX baseline: the PAA of the z-normalised series)."""
    xh, _, _, _ = znorm(np.atleast_2d(x))
    if model.get("binning") == "isax":
        return paa(xh, model["l"])
    return spectrum(xh)[:, model["best_pos"]]


def quantize(values: np.ndarray, model: dict) -> np.ndarray:
    """Alg. 2 l.5: symbol = #{i : beta(i) <= v} (bins [beta(s), beta(s+1)),
    P:225-228; a value on an edge goes right)."""
    values = np.atleast_2d(values)
    out = np.empty(values.shape, dtype=np.int64)
    for j in range(values.shape[1]):
        out[:, j] = np.searchsorted(model["edges"][j], values[:, j], side="right")
    return out


def sfa_words(x: np.ndarray, model: dict) -> np.ndarray:
    return quantize(project(x, model), model).astype(np.uint8)


def bin_bounds(model: dict, j: int, s):
    """(lo, hi) = (beta_j(s), beta_j(s+1)) with beta(0) = -inf, beta(a) = +inf."""
    e = model["edges"][j]
    s = np.asarray(s, dtype=np.int64)
    lo = np.where(s > 0, e[np.clip(s - 1, 0, len(e) - 1)] if len(e) else -np.inf, -np.inf)
    hi = np.where(s < model["a"] - 1, e[np.clip(s, 0, len(e) - 1)] if len(e) else np.inf, np.inf)
    return lo, hi


# ----------------------------------------------------------------------------- a5/a6/a7 lower bounds
def mind(q, lo, hi):
    """mind_i: 0 inside [lo, hi), lo - q below, q - hi above (reading 12)."""
    q = np.asarray(q, dtype=F64)
    return np.maximum(0.0, np.maximum(lo - q, q - hi))


def lb_word(qproj: np.ndarray, word: np.ndarray, model: dict) -> np.ndarray:
    """d_SFA^2 with per-position weights (reading 10): sum_j w_j mind_j^2.

    qproj: (l,) query projection; word: (M, l) symbols -> (M,) squared lower bounds.
    """
    word = np.atleast_2d(word)
    tot = np.zeros(word.shape[0], dtype=F64)
    for j in range(model["l"]):
        lo, hi = bin_bounds(model, j, word[:, j])
        tot += model["weights"][j] * mind(qproj[j], lo, hi) ** 2
    return tot


def lb_envelope(qproj: np.ndarray, wmin: np.ndarray, wmax: np.ndarray, model: dict) -> np.ndarray:
    """Leaf LB of a block with envelope [beta(min_j), beta(max_j+1)) per position:
    sum_j w_j max(0, beta(min_j) - q_j, q_j - beta(max_j + 1))^2 (reading 10)."""
    wmin, wmax = np.atleast_2d(wmin), np.atleast_2d(wmax)
    tot = np.zeros(wmin.shape[0], dtype=F64)
    for j in range(model["l"]):
        lo, _ = bin_bounds(model, j, wmin[:, j])
        _, hi = bin_bounds(model, j, wmax[:, j])
        tot += model["weights"][j] * mind(qproj[j], lo, hi) ** 2
    return tot


# ----------------------------------------------------------------------------- a8 exact k-NN
def sq_dists_direct(xhat: np.ndarray, qhat: np.ndarray) -> np.ndarray:
    """sum_t (x_t - q_t)^2 computed directly (Def. 2), float64."""
    d = xhat - qhat[None, :]
    return np.einsum("ij,ij->i", d, d)


def _topk(d2: np.ndarray, idx: np.ndarray, k: int):
    order = np.lexsort((idx, d2))[:k]          # ties -> smaller index (reading 14)
    return d2[order], idx[order]


def knn_bruteforce(data: np.ndarray, queries: np.ndarray, k: int, chunk: int = 1 << 16):
    """k nearest neighbours under z-ED (P:96 with reading 14; k-NN P:177), brute force.

    Distances are exact float64 direct sums over the float32 inputs.  A float64 GEMM
    (norm expansion) only *shortlists*: every row whose expanded d^2 is within a margin
    far above the expansion's error bound (n * 2^-50 * |q||x|) of the k-th smallest is
    recomputed directly, so the result equals a full direct scan.
    Returns (dist (Q,k) = sqrt(d^2), idx (Q,k) int64); k > N pads with (+inf, -1).
    """
    data = np.asarray(data)
    qh, _, _, _ = znorm(np.atleast_2d(queries))
    nq, n = qh.shape
    N = data.shape[0]
    kk = min(k, N)
    best_d = np.full((nq, k), np.inf)
    best_i = np.full((nq, k), -1, dtype=np.int64)
    cand_d = [np.empty(0)] * nq
    cand_i = [np.empty(0, dtype=np.int64)] * nq
    qn = (qh * qh).sum(axis=1)
    for s in range(0, N, chunk):
        xh, _, _, _ = znorm(data[s:s + chunk])
        xn = (xh * xh).sum(axis=1)
        approx = qn[:, None] + xn[None, :] - 2.0 * (qh @ xh.T)
        margin = 1e-9 * n + 64 * n * 2.0 ** -52 * np.sqrt(qn[:, None] * xn[None, :]).max()
        for q in range(nq):
            a = approx[q]
            kth = np.partition(a, kk - 1)[kk - 1] if a.shape[0] >= kk else np.inf
            sel = np.nonzero(a <= kth + margin)[0]
            d2 = sq_dists_direct(xh[sel], qh[q])
            cd = np.concatenate([cand_d[q], d2])
            ci = np.concatenate([cand_i[q], sel + s])
            cd, ci = _topk(cd, ci, kk)
            cand_d[q], cand_i[q] = cd, ci
    for q in range(nq):
        best_d[q, :kk] = np.sqrt(cand_d[q])
        best_i[q, :kk] = cand_i[q]
    return best_d, best_i


def knn_bruteforce_stream(chunks, queries: np.ndarray, k: int, rows_per_gemm: int = 1 << 17):
    """knn_bruteforce over a dataset too large for host memory, read as consecutive row chunks.

    The same definition (P:96 with reading 14; k-NN P:177) and the same two steps as
    knn_bruteforce — a float64 norm-expansion GEMM that only shortlists, then exact float64
    direct sums — written with torch CPU float64 ops so a 10^8-row dataset is checked in
    minutes on the host's cores.  `chunks` yields (first_row, float32 array) in row order.
    Shortlist rule per query: expanded d^2 <= (the running exact k-th best, or, while fewer than
    k rows are known, the chunk's own k-th smallest expanded d^2) + margin, with the margin of
    knn_bruteforce (far above the expansion's error).  A row of the final top-k has expanded
    d^2 <= its exact d^2 + err <= the running k-th best + err, so it is always shortlisted.
    Returns (dist (Q,k) = sqrt(d^2), idx (Q,k) int64), padded with (+inf, -1).
    """
    import torch

    qh = torch.from_numpy(znorm(np.atleast_2d(queries))[0])          # float64, Q x n
    nq, n = qh.shape
    qn = (qh * qh).sum(dim=1)
    cand_d = [np.empty(0)] * nq
    cand_i = [np.empty(0, dtype=np.int64)] * nq
    kth = np.full(nq, np.inf)                                        # running exact k-th best d^2
    for first, data in chunks:
        data = np.asarray(data)
        for s in range(0, data.shape[0], rows_per_gemm):
            x = torch.from_numpy(np.ascontiguousarray(data[s:s + rows_per_gemm])).to(torch.float64)
            # z-norm (Def. 2, population std, reading 1), same arithmetic as znorm()
            mu = x.mean(dim=1, keepdim=True)
            x -= mu
            sd = (x * x).mean(dim=1, keepdim=True).sqrt()
            flag = sd < 1e-12
            x /= torch.where(flag, torch.ones_like(sd), sd)
            x[flag[:, 0]] = 0.0
            xn = (x * x).sum(dim=1)
            approx = qn[:, None] + xn[None, :] - 2.0 * (qh @ x.T)
            margin = 1e-9 * n + 64 * n * 2.0 ** -52 * float(torch.sqrt(qn.max() * xn.max()))
            thr = torch.from_numpy(kth.copy())
            open_q = np.nonzero(~np.isfinite(kth))[0]
            if len(open_q):                                          # fewer than k rows known yet
                kk = min(k, approx.shape[1])
                ck = torch.kthvalue(approx[open_q], kk, dim=1).values
                thr[open_q] = torch.minimum(thr[open_q], ck)
            qs, cols = torch.nonzero(approx <= (thr + margin)[:, None], as_tuple=True)
            if len(qs) == 0:
                continue
            qs, cols = qs.numpy(), cols.numpy()
            diff = x[cols] - qh[qs]
            d2 = (diff * diff).sum(dim=1).numpy()                    # exact direct sums
            for q in np.unique(qs):
                sel = qs == q
                cd = np.concatenate([cand_d[q], d2[sel]])
                ci = np.concatenate([cand_i[q], cols[sel] + first + s])
                cd, ci = _topk(cd, ci, k)
                cand_d[q], cand_i[q] = cd, ci
                if len(cd) >= k:
                    kth[q] = cd[k - 1]
    best_d = np.full((nq, k), np.inf)
    best_i = np.full((nq, k), -1, dtype=np.int64)
    for q in range(nq):
        m = len(cand_d[q])
        best_d[q, :m] = np.sqrt(cand_d[q])
        best_i[q, :m] = cand_i[q]
    return best_d, best_i


def knn_gemini(data: np.ndarray, queries: np.ndarray, k: int, model: dict):
    """GEMINI exact search with LB-ordered refinement.

    Visit series in ascending d_SFA^2 order; stop at the first whose LB exceeds the
    current k-th best d^2 (refine iff LB < BSF, reading 15).  Also returns the number of
    exact distance computations.
    """
    data = np.asarray(data)
    xh, _, _, _ = znorm(data)
    words = sfa_words(data, model)
    qh, _, _, _ = znorm(np.atleast_2d(queries))
    out_d = np.full((qh.shape[0], k), np.inf)
    out_i = np.full((qh.shape[0], k), -1, dtype=np.int64)
    refined = np.zeros(qh.shape[0], dtype=np.int64)
    for q in range(qh.shape[0]):
        qp = spectrum(qh[q:q + 1])[0, model["best_pos"]]
        lb = lb_word(qp, words, model)
        order = np.lexsort((np.arange(len(lb)), lb))
        best: list[tuple[float, int]] = []
        for i in order:
            bsf = best[k - 1][0] if len(best) >= k else np.inf
            if lb[i] > bsf:
                break
            d2 = float(sq_dists_direct(xh[i:i + 1], qh[q])[0])
            refined[q] += 1
            best.append((d2, int(i)))
            best.sort()
            best = best[:k]
        for r, (d2, i) in enumerate(best):
            out_d[q, r] = np.sqrt(d2)
            out_i[q, r] = i
    return out_d, out_i, refined


def merge_topk(dist: np.ndarray, idx: np.ndarray, k: int):
    """k smallest (dist, idx) of P per-shard lists (P, Q, k) -> (Q, k); ties -> smaller idx."""
    P, nq, _ = dist.shape
    od = np.full((nq, k), np.inf)
    oi = np.full((nq, k), -1, dtype=np.int64)
    for q in range(nq):
        d = dist[:, q, :].ravel()
        i = idx[:, q, :].ravel()
        valid = i >= 0
        d, i = d[valid], i[valid]
        order = np.lexsort((i, d))[:k]
        od[q, :len(order)] = d[order]
        oi[q, :len(order)] = i[order]
    return od, oi
