"""World-size-2 gloo tests of the multi-GPU host logic (paper_2411_17483_b200/distributed.py) on
CPU: global strided sample assembly (C1), model byte broadcast, top-k all-gather + merge (C4).
The compute steps are the oracle's here (test infrastructure); on a GPU box the same functions
run with libsofa kernels and NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sofa_oracle as O
from paper_2411_17483_b200 import datagen
from paper_2411_17483_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = datagen.scaled(datagen.WORKLOADS["cfg1"], 4001, 9, length=32)
        a, b = datagen.shard_range(w.n_series, rank, world)
        shard = datagen.generate_rows(w, a, b)
        queries = datagen.generate_queries(w)
        S = 500
        sample = D.gather_global_sample(shard, a, w.n_series, S)
        full = datagen.generate_rows(w, 0, w.n_series)
        ok_sample = torch.equal(sample, full[torch.as_tensor(O.sample_indices(w.n_series, S))])
        mb = b"model-bytes-%d" % 7 if rank == 0 else None
        got = D.broadcast_model_bytes(mb, "cpu")
        k = 5

        def local_knn(qs, kk):
            d, i = O.knn_bruteforce(shard.numpy(), qs.numpy(), kk)
            i = np.where(i >= 0, i + a, -1)
            return torch.from_numpy(d.astype(np.float32)), torch.from_numpy(i)

        def merge(Dd, Ii):
            d, i = O.merge_topk(Dd.numpy().astype(np.float64), Ii.numpy(), k)
            return torch.from_numpy(d), torch.from_numpy(i)

        d, i = D.sharded_knn(queries, k, local_knn, merge)
        do, io = O.knn_bruteforce(full.numpy(), queries.numpy(), k)
        # with the seed-bound exchange (C3): each rank's bound = the k-th best of a few of its rows,
        # the all-reduced minimum bounds the global k-th best; shards drop rows above it
        def local_seed(qs, kk):
            ds, _ = O.knn_bruteforce(shard.numpy()[:64], qs.numpy(), kk)
            return torch.from_numpy((ds[:, -1] ** 2).astype(np.float32))

        def local_knn_bounded(qs, kk, bound):
            dd, ii = local_knn(qs, kk)
            drop = dd.double() ** 2 > bound.double()[:, None] * (1 + 1e-6)
            return torch.where(drop, torch.full_like(dd, float("inf")), dd), torch.where(drop, -1, ii)

        d2, i2 = D.sharded_knn(queries, k, local_knn_bounded, merge, local_seed=local_seed)
        ok_bound = bool(np.array_equal(i2.numpy(), io))
        q.put((rank, ok_sample, got == b"model-bytes-7", bool(np.array_equal(i.numpy(), io)) and ok_bound,
               float(np.max(np.abs(d.numpy() - do) / do))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_pipeline(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_sample, ok_bytes, ok_idx, rel in res:
        assert ok_sample and ok_bytes and ok_idx and rel < 1e-6, (rank, ok_sample, ok_bytes, ok_idx, rel)


def test_sample_indices_match_oracle():
    assert np.array_equal(D.global_sample_indices(10_000_000, 100_000), O.sample_indices(10_000_000, 100_000))


def _worker_shards(rank, world, port, q, N, k):
    """uneven shards (and an empty one when N < world): local oracle k-NN on each rank's rows, then the
    exchange — k = 1 the packed-key all-reduce MIN, k > 1 the all-gather + merge — with and without the
    seed-bound exchange; every rank must hold the oracle's global answer"""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = datagen.scaled(datagen.WORKLOADS["cfg1"], N, 7, length=32)
        full = datagen.generate_rows(w, 0, N)
        queries = datagen.generate_queries(w)
        a, b = datagen.shard_range(N, rank, world)
        shard = full[a:b]

        def local_knn(qs, kk, bound=None):
            dd = np.full((qs.shape[0], kk), np.inf)
            ii = np.full((qs.shape[0], kk), -1, dtype=np.int64)
            if shard.shape[0]:
                dd, ii = O.knn_bruteforce(shard.numpy(), qs.numpy(), kk)
                ii = np.where(ii >= 0, ii + a, -1)
            if bound is not None:  # results above the exchanged bound are never returned (bsf_init)
                drop = dd ** 2 > bound.double().numpy()[:, None] * (1 + 1e-6)
                dd, ii = np.where(drop, np.inf, dd), np.where(drop, -1, ii)
            return torch.from_numpy(dd.astype(np.float32)), torch.from_numpy(ii)

        def local_seed(qs, kk):
            if shard.shape[0] < kk:
                return torch.full((qs.shape[0],), float("inf"))
            ds, _ = O.knn_bruteforce(shard.numpy()[: max(kk, shard.shape[0] // 3)], qs.numpy(), kk)
            return torch.from_numpy((ds[:, -1] ** 2).astype(np.float32))

        def merge(Dd, Ii):
            d, i = O.merge_topk(Dd.numpy().astype(np.float64), Ii.numpy(), k)
            return torch.from_numpy(d.astype(np.float32)), torch.from_numpy(i)

        do, io = O.knn_bruteforce(full.numpy(), queries.numpy(), k)
        d1, i1 = D.sharded_knn(queries, k, local_knn, merge)
        d2, i2 = D.sharded_knn(queries, k, local_knn, merge, local_seed=local_seed)
        ok = all(np.array_equal(i.numpy(), io) for i in (i1, i2))
        fin = np.isfinite(do)
        rel = max(float(np.max(np.abs(d.numpy()[fin] - do[fin]) / np.maximum(do[fin], 1e-12), initial=0.0))
                  for d in (d1, d2))
        pad_ok = all(np.array_equal(np.isfinite(d.numpy()), fin) for d in (d1, d2))
        q.put((rank, ok and pad_ok, rel, b - a))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N,k", [(4, 4003, 1), (4, 4003, 5), (4, 3, 1), (4, 3, 5), (3, 1000, 2)])
def test_gloo_uneven_and_empty_shards(world, N, k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_shards, args=(r, world, port, q, N, k)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sizes = sorted(r[3] for r in res)
    assert sum(sizes) == N and sizes[-1] - sizes[0] <= 1
    for rank, ok, rel, _ in res:
        assert ok and rel < 1e-6, (rank, ok, rel)


def test_packed_keys_order_like_distance_then_index():
    """the k = 1 exchange key: int64 order == lexicographic (distance, index) order; padding last"""
    rng = np.random.default_rng(3)
    d = np.concatenate([rng.uniform(0, 30, 200), [0.0, 0.0, 5.0, 5.0, np.inf, np.inf]]).astype(np.float32)
    i = np.concatenate([rng.integers(0, 100_000_000, 200), [7, 3, 9, 2, -1, -1]]).astype(np.int64)
    key = D.pack_keys(torch.from_numpy(d), torch.from_numpy(i)).numpy()
    big = np.where(i < 0, 0xFFFFFFFF, i)
    order = np.lexsort((big, d))
    assert np.array_equal(np.argsort(key, kind="stable"), order) or np.array_equal(key[np.argsort(key)], key[order])
    dd, ii = D.unpack_keys(torch.from_numpy(key))
    assert np.array_equal(dd.numpy(), d) and np.array_equal(ii.numpy(), i)
