"""GPU parity: the CUDA path (through the C ABI) against the CPU float64 oracle on the same seeded
inputs.  Acceptance (BASELINE.json north_star): neighbour indices exact except ties within 1e-5
relative distance; distances within 1e-4 relative; SFA symbols bit-exact except values within
1e-5 of a bin edge; the learned model equal to the oracle's (best_l identical, edges within
float32 rounding)."""
import numpy as np
import pytest
import torch

from oracle import sofa_oracle as O
from paper_2411_17483_b200 import datagen
from paper_2411_17483_b200.index import SofaIndex, learn_model, merge_topk, transform

pytestmark = pytest.mark.gpu

from knn_check import DIST_RTOL, TIE_RTOL, assert_knn_parity  # noqa: F401  (re-exported to the other GPU tests)


def _data(w, device="cuda"):
    x = datagen.generate_rows(w, 0, w.n_series, device=device)
    q = datagen.generate_queries(w, device=device, data=x)
    return x, q


# ------------------------------------------------------------------------------------- a2 model
@pytest.mark.parametrize("kind,n,l,binning", [("cfg1", 256, 16, "equi-depth"), ("cfg3", 256, 16, "equi-depth"),
                                              ("cfg1", 256, 16, "equi-width"), ("cfg5", 1024, 32, "equi-depth"),
                                              ("cfg1", 64, 8, "equi-depth")])
def test_model_parity(kind, n, l, binning):
    w = datagen.scaled(datagen.WORKLOADS[kind], 6000, 4, length=n, l=l)
    x = datagen.generate_rows(w, 0, w.n_series, device="cuda")
    S = 3000
    idx = O.sample_indices(w.n_series, S)
    sample = x[torch.as_tensor(idx, device="cuda")]
    mg = learn_model(sample, l, 256, binning=binning)
    mo = O.learn_model(sample.cpu().numpy(), l, 256, binning=binning)
    assert np.array_equal(mg["best_pos"], mo["best_pos"])
    np.testing.assert_array_equal(mg["weights"], mo["weights"])
    np.testing.assert_allclose(mg["edges"], mo["edges"], rtol=1e-7, atol=1e-9)
    # the index's own model (learned from the strided sample inside sofa_build) is the same model
    ix = SofaIndex(x, l=l, alphabet=256, sample_size=S, binning=binning)
    mi = ix.model
    assert np.array_equal(mi["best_pos"], mo["best_pos"])
    np.testing.assert_allclose(mi["edges"], mo["edges"], rtol=1e-7, atol=1e-9)


# ------------------------------------------------------------------------------------- a1 + a3 transform
def _edge_exempt(vals, model):
    """True where the oracle value lies within 1e-5 (relative above 1) of a bin edge."""
    ex = np.zeros(vals.shape, dtype=bool)
    for j in range(vals.shape[1]):
        e = model["edges"][j]
        pos = np.searchsorted(e, vals[:, j])
        for cand in (pos - 1, pos):
            c = np.clip(cand, 0, len(e) - 1)
            ex[:, j] |= np.abs(vals[:, j] - e[c]) <= 1e-5 * np.maximum(1.0, np.abs(e[c]))
    return ex


@pytest.mark.parametrize("kind,n,l", [("cfg1", 256, 16), ("cfg3", 256, 16), ("cfg5", 1024, 32), ("cfg1", 128, 24),
                                      ("cfg3", 96, 40)])
def test_transform_parity(kind, n, l):
    w = datagen.scaled(datagen.WORKLOADS[kind], 40_000, 4, length=n, l=l)
    x = datagen.generate_rows(w, 0, w.n_series, device="cuda")
    xn = x.cpu().numpy()
    mo = O.learn_model(xn[O.sample_indices(w.n_series, 4000)], l, 256)
    vals, words = transform(x, mo)
    vo = O.project(xn, mo)
    err = np.abs(vals.cpu().numpy() - vo)
    assert err.max() < 5e-6, err.max()
    so = O.quantize(vo, mo)
    sg = words.cpu().numpy().astype(np.int64)
    mism = (so != sg) & ~_edge_exempt(vo, mo)
    assert mism.sum() == 0, (mism.sum(), np.argwhere(mism)[:5])
    assert np.all(np.abs(so - sg) <= 1)


def test_index_invariants():
    w = datagen.scaled(datagen.WORKLOADS["cfg1"], 50_000 + 77, 4)
    x = datagen.generate_rows(w, 0, w.n_series, device="cuda")
    ix = SofaIndex(x, sample_size=5000, block_size=256)
    inf = ix.info
    assert inf["n_blocks"] == (w.n_series + 255) // 256
    ex = ix.export()
    perm = ex["perm"].cpu().numpy()
    assert np.array_equal(np.sort(perm), np.arange(w.n_series))
    _, words = transform(x, ix.raw_model)
    wsorted = ex["words"][:, :16].cpu().numpy()
    assert np.array_equal(wsorted, words.cpu().numpy()[perm])
    # keys: 2-bit interleave of the first 16 positions, MSB first -> sorted order non-decreasing
    s = wsorted.astype(np.uint64)
    key = np.zeros(len(s), dtype=np.uint64)
    for r in range(2):
        for p in range(16):
            key = (key << np.uint64(2)) | ((s[:, p] >> np.uint64(6 - 2 * r)) & np.uint64(3))
    assert np.all(np.diff(key.astype(np.float64)) >= 0) or np.all(key[1:] >= key[:-1])
    env = ex["env"].cpu().numpy()
    for b in range(inf["n_blocks"]):
        blk = wsorted[b * 256:(b + 1) * 256]
        assert np.array_equal(env[b, 0, :16], blk.min(axis=0))
        assert np.array_equal(env[b, 1, :16], blk.max(axis=0))
    assert np.array_equal(ex["block_keys"].cpu().numpy().astype(np.uint64), key[::256])


# ------------------------------------------------------------------------------------- k-NN parity
@pytest.mark.parametrize("kind,N,n,l,k,Q", [
    ("cfg1", 100_000, 256, 16, 1, 100),     # BJ configs[0] at full size
    ("cfg2", 200_000, 256, 16, 1, 200),     # noisy members sigma 0.1
    ("cfg3", 60_000, 256, 16, 1, 40),       # high frequency (low pruning)
    ("cfg4", 200_000, 256, 16, 1, 150),     # sigma mix 0.01 / 0.1 / 1.0
    ("cfg5", 40_000, 1024, 32, 10, 40),     # mixed n=1024, l=32, 10-NN
    ("cfg1", 30_000, 256, 16, 10, 50),
    ("cfg3", 20_000, 128, 16, 5, 30),
])
def test_knn_parity(kind, N, n, l, k, Q):
    w = datagen.scaled(datagen.WORKLOADS[kind], N, Q, length=n, l=l, k=k)
    x, q = _data(w)
    ix = SofaIndex(x, l=l, alphabet=256, sample_size=datagen.default_sample_size(w))
    d, i, st = ix.knn(q, k, stats=True)
    torch.cuda.synchronize()
    xn, qn = x.cpu().numpy(), q.cpu().numpy()
    do, io = O.knn_bruteforce(xn, qn, k)
    assert_knn_parity(d.cpu().numpy(), i.cpu().numpy(), do, io, xn, qn)
    assert st["queries"] == Q and st["refined"] >= Q * min(k, 1)
    if kind in ("cfg2",):
        assert st["refined"] < 0.01 * N * Q          # pruning works on noisy-member queries


@pytest.mark.parametrize("B", [32, 64, 1024, 4096])
def test_result_invariant_to_block_size(B):
    w = datagen.scaled(datagen.WORKLOADS["cfg4"], 40_000, 60)
    x, q = _data(w)
    ref = SofaIndex(x, sample_size=4000, block_size=256).knn(q, 3)
    got = SofaIndex(x, sample_size=4000, block_size=B).knn(q, 3)
    assert torch.equal(ref[1], got[1]) and torch.equal(ref[0], got[0])


@pytest.mark.parametrize("parts", [2, 3, 5])
def test_sharded_merge_equals_unsharded(parts):
    """a9: per-shard indices (global model, global offsets) + the merge kernel equal the single index
    bit for bit AND the oracle: the merge against O.merge_topk of the oracle's per-shard lists, the
    merged result against the oracle's brute force over all rows"""
    w = datagen.scaled(datagen.WORKLOADS["cfg1"], 30_011, 40)
    x, q = _data(w)
    k = 4
    full = SofaIndex(x, sample_size=3000)
    d0, i0 = full.knn(q, k)
    model = full.raw_model
    xn, qn = x.cpu().numpy(), q.cpu().numpy()
    ds, is_, ods, ois = [], [], [], []
    for r in range(parts):
        a, b = datagen.shard_range(w.n_series, r, parts)
        sh = x[a:b].contiguous()
        ix = SofaIndex(sh, model=model, global_offset=a, global_n=w.n_series)
        d, i = ix.knn(q, k)
        ds.append(d)
        is_.append(i)
        do_, io_ = O.knn_bruteforce(xn[a:b], qn, k)
        assert_knn_parity(d.cpu().numpy(), i.cpu().numpy() - a, do_, io_, xn[a:b], qn)  # each shard is exact
        ods.append(do_)
        ois.append(np.where(io_ >= 0, io_ + a, -1))
        del ix
    md, mi = merge_topk(torch.stack(ds), torch.stack(is_))
    assert torch.equal(mi, i0) and torch.equal(md, d0)
    od, oi = O.merge_topk(np.stack(ods), np.stack(ois), k)
    assert_knn_parity(md.cpu().numpy(), mi.cpu().numpy(), od, oi, xn, qn)
    do, io = O.knn_bruteforce(xn, qn, k)
    assert_knn_parity(md.cpu().numpy(), mi.cpu().numpy(), do, io, xn, qn)


@pytest.mark.parametrize("P,Q,k", [(2, 50, 1), (3, 17, 5), (8, 9, 16), (5, 4, 128)])
def test_merge_kernel_equals_oracle_merge(P, Q, k):
    """k_merge_topk alone on synthetic sorted lists with exact ties (across and within parts),
    padding and empty parts: equal to O.merge_topk element by element (ties -> smaller index)"""
    rng = np.random.default_rng(P * 100 + k)
    d = np.sort(rng.integers(0, 6, size=(P, Q, k)).astype(np.float32) * 0.25, axis=2)
    i = np.empty((P, Q, k), dtype=np.int64)
    for p in range(P):
        for qq in range(Q):  # distinct global indices per part, increasing within equal distances
            i[p, qq] = np.sort(rng.choice(10 ** 6, size=k, replace=False)) * P + p
    pad = rng.random((P, Q, k)) < 0.2
    pad = np.cumsum(pad, axis=2) > 0          # padding is a suffix of each list
    d[pad] = np.inf
    i[pad] = -1
    d[0, 0] = np.inf                          # an empty part
    i[0, 0] = -1
    md, mi = merge_topk(torch.from_numpy(d).cuda(), torch.from_numpy(i).cuda())
    od, oi = O.merge_topk(d.astype(np.float64), i, k)
    assert np.array_equal(mi.cpu().numpy(), oi)
    assert np.array_equal(md.cpu().numpy().astype(np.float64), od)


@pytest.mark.parametrize("k", [1, 5])
def test_large_leaf_list_branch_parity(k):
    """the front's large-list branch (more than CAP_B = 2048 leaves survive the envelope filter and
    the top-M re-filter: the ~1536 lowest-LB leaves are sorted and scanned first, the rest is
    re-filtered and scanned in storage order): 1M rows in blocks of 32 (31,250 leaves), noisy
    members with sigma = 1 (SFA bound weak: most leaves survive), sparse path forced"""
    w = datagen.scaled(datagen.WORKLOADS["cfg4"], 1_000_000, 12, noise_sigmas=(1.0,))
    x, q = _data(w)
    ix = SofaIndex(x, sample_size=10_000, block_size=32, dense_permille=-1)
    d, i, st = ix.knn(q, k, stats=True)
    torch.cuda.synchronize()
    assert st["rounds"] > 0 and st["max_list_blocks"] > 2048, st  # the cnt > CAP_B branch ran
    xn, qn = x.cpu().numpy(), q.cpu().numpy()
    do, io = O.knn_bruteforce(xn, qn, k)
    assert_knn_parity(d.cpu().numpy(), i.cpu().numpy(), do, io, xn, qn)


def test_bsf_init_prunes_without_changing_results():
    w = datagen.scaled(datagen.WORKLOADS["cfg2"], 50_000, 64)
    x, q = _data(w)
    ix = SofaIndex(x, sample_size=5000)
    d0, i0, s0 = ix.knn(q, 1, stats=True)
    bsf = (d0[:, 0] ** 2) * 1.001
    d1, i1, s1 = ix.knn(q, 1, bsf_init=bsf.contiguous(), stats=True)
    assert torch.equal(i0, i1)
    tight = (d0[:, 0] ** 2) * 0.5          # bound below the true NN: nothing within it exists
    d2, i2 = ix.knn(q, 1, bsf_init=tight.contiguous())
    assert bool((i2 == -1).all()) and bool(torch.isinf(d2).all())


# ------------------------------------------------------------------------------------- edge cases
def test_edge_cases_small_and_degenerate():
    rng = np.random.default_rng(5)
    base = np.cumsum(rng.normal(size=(300, 32)), axis=1).astype(np.float32)
    base[17] = base[3]                      # exact duplicate -> tie to the smaller index
    base[40] = 7.0                          # constant series -> zero vector
    base[41] = base[41] * 1000 + 55.0       # large offset/scale -> same z-normalised shape
    x = torch.from_numpy(base).cuda()
    ix = SofaIndex(x, l=8, alphabet=16, sample_size=300, block_size=32)
    qs = torch.from_numpy(base[[3, 40, 41, 100]]).cuda()
    d, i = ix.knn(qs, 3)
    do, io = O.knn_bruteforce(base, base[[3, 40, 41, 100]], 3)
    assert_knn_parity(d.cpu().numpy(), i.cpu().numpy(), do, io, base, base[[3, 40, 41, 100]])
    assert i[0, 0].item() == 3 and i[0, 1].item() == 17 and d[0, 0].item() == 0.0
    # k = N: the full sorted list
    small = x[:37].contiguous()
    ixs = SofaIndex(small, l=4, alphabet=4, sample_size=37, block_size=32)
    d, i = ixs.knn(qs, 37)
    do, io = O.knn_bruteforce(base[:37], base[[3, 40, 41, 100]], 37)
    assert_knn_parity(d.cpu().numpy(), i.cpu().numpy(), do, io, base[:37], base[[3, 40, 41, 100]])


def test_single_series_and_padding_and_short_len():
    rng = np.random.default_rng(6)
    from paper_2411_17483_b200.sofa import SofaError
    x = torch.from_numpy(rng.normal(size=(1, 8)).astype(np.float32)).cuda()
    with pytest.raises(SofaError, match="at least 2 rows"):      # variance needs >= 2 sample rows
        SofaIndex(x, l=3, alphabet=2, sample_size=2, binning="equi-width")
    other = torch.from_numpy(rng.normal(size=(64, 8)).astype(np.float32)).cuda()
    m1 = SofaIndex(other, l=3, alphabet=2, sample_size=64, binning="equi-width").raw_model
    ix = SofaIndex(x, l=3, alphabet=2, model=m1)                # a single series with a given model
    d, i = ix.knn(x, 1)
    assert i.item() == 0 and d.item() == 0.0
    x4 = torch.from_numpy(rng.normal(size=(500, 4)).astype(np.float32)).cuda()
    ix4 = SofaIndex(x4, l=3, alphabet=4, sample_size=100, block_size=32)
    q4 = torch.from_numpy(rng.normal(size=(7, 4)).astype(np.float32)).cuda()
    d, i = ix4.knn(q4, 2)
    do, io = O.knn_bruteforce(x4.cpu().numpy(), q4.cpu().numpy(), 2)
    assert_knn_parity(d.cpu().numpy(), i.cpu().numpy(), do, io, x4.cpu().numpy(), q4.cpu().numpy())
    # empty shard with a model pads
    m = ix4.raw_model
    empty = torch.empty(0, 4, dtype=torch.float32, device="cuda")
    ixe = SofaIndex(empty, l=3, alphabet=4, model=m, global_n=500)
    d, i = ixe.knn(q4, 2)
    assert bool((i == -1).all()) and bool(torch.isinf(d).all())


def test_host_path_equals_device_path():
    w = datagen.scaled(datagen.WORKLOADS["cfg2"], 20_000, 32)
    x, q = _data(w)
    ix = SofaIndex(x, sample_size=2000)
    d, i = ix.knn(q, 2)
    hd, hi = ix.knn_host(q.cpu().numpy(), 2)
    assert np.array_equal(hi, i.cpu().numpy()) and np.array_equal(hd, d.cpu().numpy())


@pytest.mark.parametrize("Q,k", [(3, 1), (7, 4), (40, 2)])
def test_scan_pool_heavy_queries(Q, k):
    """few queries with long leaf lists (cfg4 recipe, sigma 1.0 members) on the sparse path: their
    leaf chunks are spread over all CTAs as scan tasks; results equal the oracle's brute force"""
    w = datagen.scaled(datagen.WORKLOADS["cfg4"], 300_000 + 77, Q, noise_sigmas=(1.0,))
    x, q = _data(w)
    ix = SofaIndex(x, sample_size=3000, dense_permille=-1)
    d, i, st = ix.knn(q, k, stats=True)
    torch.cuda.synchronize()
    do, io = O.knn_bruteforce(x.cpu().numpy(), q.cpu().numpy(), k)
    assert_knn_parity(d.cpu().numpy(), i.cpu().numpy(), do, io, x.cpu().numpy(), q.cpu().numpy())
    assert st["scan_tasks"] > st["scan_queries"] > 0


def test_large_batch_runs_in_sub_batches():
    """q = 2500 > the internal sub-batch (1024): results, stats and the trace cover every query"""
    from paper_2411_17483_b200 import sofa as S
    w = datagen.scaled(datagen.WORKLOADS["cfg1"], 40_000, 2500)
    x, q = _data(w)
    ix = SofaIndex(x, sample_size=4000)
    d, i, st = ix.knn(q, 3, stats=True)
    torch.cuda.synchronize()
    assert st["queries"] == 2500
    tr = S.sofa_knn_trace(ix.handle, 2500)
    assert np.all(tr[:, :4].sum(axis=1) > 0)  # every query's row was written
    pick = np.r_[0:5, 1020:1030, 2040:2050, 2495:2500]
    do, io = O.knn_bruteforce(x.cpu().numpy(), q[pick].cpu().numpy(), 3)
    assert_knn_parity(d[pick].cpu().numpy(), i[pick].cpu().numpy(), do, io, x.cpu().numpy(), q[pick].cpu().numpy())
    d1, i1 = ix.knn(q[1000:1100].contiguous(), 3)  # a batch straddling the split gives the same rows
    assert torch.equal(i1, i[1000:1100]) and torch.equal(d1, d[1000:1100])
    # live kernel timing (bench.py's roofline): one event group per sub-batch, results unchanged
    ix.kernel_timing(1)
    d2, i2 = ix.knn(q, 3)
    d3, i3 = ix.knn(q[:10].contiguous(), 3)
    km, groups = ix.kernel_timing(0)
    assert groups == 3 + 1 and km["front"] > 0 and km["scan"] > 0 and km["dense"] >= 0
    assert torch.equal(i2, i) and torch.equal(d2, d) and torch.equal(i3, i[:10])
    km0, g0 = ix.kernel_timing(-1)  # stopped and cleared
    assert g0 == 0 and set(km0) == {"front", "dense", "scan", "dense_screen", "dense_post"} and not any(km0.values())
    assert abs(km["dense"] - km["dense_screen"] - km["dense_post"]) < 1e-9
    ix.knn(q[:10].contiguous(), 3)
    assert ix.kernel_timing(-1)[1] == 0


def test_max_k_and_single_query():
    w = datagen.scaled(datagen.WORKLOADS["cfg4"], 20_000, 1)
    x, q = _data(w)
    ix = SofaIndex(x, sample_size=2000)
    d, i = ix.knn(q, 128)
    do, io = O.knn_bruteforce(x.cpu().numpy(), q.cpu().numpy(), 128)
    assert_knn_parity(d.cpu().numpy(), i.cpu().numpy(), do, io, x.cpu().numpy(), q.cpu().numpy())


@pytest.mark.parametrize("kind,k", [("cfg2", 1), ("cfg1", 4), ("cfg3", 2)])
def test_knn_seed_bound_is_a_valid_upper_bound(kind, k):
    """sofa_knn_seed: per query an upper bound on the k-th best squared distance (the k-th best of
    real rows); for noisy members it is already the nearest neighbour's distance"""
    w = datagen.scaled(datagen.WORKLOADS[kind], 60_000, 40)
    x, q = _data(w)
    ix = SofaIndex(x, sample_size=6000)
    b = ix.knn_seed(q, k).cpu().numpy().astype(np.float64)
    do, _ = O.knn_bruteforce(x.cpu().numpy(), q.cpu().numpy(), k)
    kth2 = do[:, -1] ** 2
    assert np.all(b >= kth2 * (1 - 1e-4) - 1e-6)
    if kind == "cfg2":
        assert np.mean(np.abs(b - kth2) <= 1e-4 * kth2 + 1e-6) > 0.9
    d1, i1 = ix.knn(q, k)
    d2, i2 = ix.knn(q, k, bsf_init=torch.from_numpy(b.astype(np.float32)).cuda())
    assert torch.equal(i1, i2) and torch.equal(d1, d2)


@pytest.mark.parametrize("rev_rounds", [0, 1, 1000000])
@pytest.mark.parametrize("kind,k,front_batches", [("cfg1", 5, 16), ("cfg4", 3, 2)])
def test_revisit_pass_and_front_split(rev_rounds, kind, k, front_batches):
    """scan_blocks' revisit pass (a leaf part with more than rev_rounds x R candidates is deferred
    until after the list; 0 defers every part with a candidate and overflows the revisit queue,
    1e6 never defers) and the front/scan split (front_batches word batches in the front, the rest
    as scan tasks) change the refinement order only: results equal the oracle's brute force and
    each other bit for bit (sofa_set_tuning)"""
    w = datagen.scaled(datagen.WORKLOADS[kind], 200_000 + 33, 24)
    x, q = _data(w)
    ix = SofaIndex(x, sample_size=3000, dense_permille=-1)
    ix.set_tuning(rev_rounds=rev_rounds, front_batches=front_batches)
    d, i, st = ix.knn(q, k, stats=True)
    torch.cuda.synchronize()
    do, io = O.knn_bruteforce(x.cpu().numpy(), q.cpu().numpy(), k)
    assert_knn_parity(d.cpu().numpy(), i.cpu().numpy(), do, io, x.cpu().numpy(), q.cpu().numpy())
    ix.set_tuning(rev_rounds=1000000, front_batches=1000000)
    d2, i2 = ix.knn(q, k)
    assert torch.equal(d, d2) and torch.equal(i, i2)


@pytest.mark.parametrize("front_wide,scan_wide", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("kind,k,Q", [("cfg1", 1, 37), ("cfg4", 5, 37), ("cfg4", 2, 400)])
def test_wide_and_narrow_query_builds_agree(front_wide, scan_wide, kind, k, Q):
    """the 16-warp (query512.cu) and 8-warp builds of the front and the scan pool, in every pairing —
    they share QState, the leaf pool and the tasks — give the same bits as the automatic choice and
    equal the oracle's brute force; the scan pool must actually run (scan tasks published).  Q = 400
    is more queries than SMs, so 'wide' there forces the 16-warp build past its automatic range."""
    kw = {"noise_sigmas": (1.0,)} if kind == "cfg4" else {}
    w = datagen.scaled(datagen.WORKLOADS[kind], 150_000 + 7, Q, **kw)
    x, q = _data(w)
    ix = SofaIndex(x, sample_size=3000, dense_permille=-1)
    ix.set_tuning(front_batches=1)  # publish most leaves as scan tasks so the scan pool has work
    d, i, st = ix.knn(q, k, stats=True)
    assert st["scan_tasks"] > 0
    ix.set_tuning(front_batches=1, front_wide=front_wide, scan_wide=scan_wide)
    d2, i2 = ix.knn(q, k)
    torch.cuda.synchronize()
    assert torch.equal(d, d2) and torch.equal(i, i2)
    do, io = O.knn_bruteforce(x.cpu().numpy(), q.cpu().numpy(), k)
    assert_knn_parity(d.cpu().numpy(), i.cpu().numpy(), do, io, x.cpu().numpy(), q.cpu().numpy())


@pytest.mark.parametrize("kind,N,Q,k", [("cfg2", 300_000, 900, 1), ("cfg4", 250_000, 600, 3), ("cfg1", 120_000, 40, 2)])
def test_fused_scan_identical(kind, N, Q, k):
    """front CTAs without a query left drain the published set-0 tasks from a FIFO in the same launch
    (scan_fused = 1, default) or leave them to the separate scan launch (0): the same bits, and the
    oracle's answer; the FIFO path must really have carried tasks"""
    w = datagen.scaled(datagen.WORKLOADS[kind], N, Q, k=k)
    x, q = _data(w)
    ix = SofaIndex(x, sample_size=datagen.default_sample_size(w))
    ix.set_tuning(front_batches=1)  # small front budget: most lists go through the task pool
    d1, i1, st = ix.knn(q, k, stats=True)
    assert st["scan_tasks"] > 0
    ix.set_tuning(front_batches=1, scan_fused=0)
    d0, i0 = ix.knn(q, k)
    assert torch.equal(i1, i0) and torch.equal(d1, d0)
    do, io = O.knn_bruteforce(x.cpu().numpy(), q.cpu().numpy(), k)
    assert_knn_parity(d1.cpu().numpy(), i1.cpu().numpy(), do, io, x.cpu().numpy(), q.cpu().numpy())


@pytest.mark.parametrize("kind", ["cfg1", "cfg3"])
def test_stored_row_as_query_has_distance_zero(kind):
    """a1: the transform's (mu, 1/sigma) of a row and the query prep's of the same values come from one
    function with one arithmetic order (common.cuh row_stats_g), so they are the same float32 bits and
    the exact refine of a row against itself is 0.0 (rows of a ragged last warp group included)"""
    w = datagen.scaled(datagen.WORKLOADS[kind], 25_000 + 2, 4)
    x = datagen.generate_rows(w, 0, w.n_series, device="cuda")
    ix = SofaIndex(x, l=16, sample_size=3000)
    rows = torch.tensor([0, 1, 2, 3, 5, 4097, 12_345, w.n_series - 2, w.n_series - 1], device="cuda")
    d, i = ix.knn(x[rows].contiguous(), 1)
    torch.cuda.synchronize()
    assert torch.all(d[:, 0] == 0.0), d[:, 0]
    assert torch.equal(x[i[:, 0]], x[rows])  # the row itself, or an exact duplicate of it
    ix.close()
