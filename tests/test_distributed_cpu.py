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
