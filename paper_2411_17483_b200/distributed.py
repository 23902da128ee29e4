"""One process per GPU: dataset sharding, the global MCB model (C1) and the top-k exchange (C4).

SURVEY 8(e): series are independent, so each rank holds a contiguous shard (datagen.shard_range)
and builds its own index with the GLOBAL model; a query batch is replicated on every rank, each
rank returns its local top-k with global indices, and an all-gather (NCCL over NVLink on a GPU
box) followed by the libsofa min-merge kernel (a9) gives the global answer.  The exchange is
tiny (P x Q x k x 12 bytes), so it is latency-bound.

The collective plumbing is written against torch.distributed only; the compute steps (learning,
local k-NN, merge) are passed in, so the same host logic runs over gloo on CPU in the tests
(with oracle functions injected by the test) and over NCCL with the CUDA kernels in the product.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist


def global_sample_indices(global_n: int, S: int) -> np.ndarray:
    """Alg. 1 sample(X, r) as strided global rows floor(j * N / S) (reading 6)."""
    return (np.arange(S, dtype=np.int64) * global_n) // S


def gather_global_sample(shard: torch.Tensor, global_offset: int, global_n: int, S: int, group=None) -> torch.Tensor:
    """Every rank contributes the sample rows that fall in its shard; all ranks receive the
    S x len sample in j order (ranks hold contiguous ranges, so rank order is j order)."""
    idx = global_sample_indices(global_n, S)
    mine = idx[(idx >= global_offset) & (idx < global_offset + shard.shape[0])] - global_offset
    local = shard[torch.as_tensor(mine, device=shard.device)] if len(mine) else shard[:0]
    world = dist.get_world_size(group)
    counts = [torch.zeros(1, dtype=torch.int64, device=shard.device) for _ in range(world)]
    dist.all_gather(counts, torch.tensor([local.shape[0]], dtype=torch.int64, device=shard.device), group=group)
    counts = [int(c.item()) for c in counts]
    mx = max(counts)
    pad = torch.zeros(mx, shard.shape[1], dtype=shard.dtype, device=shard.device)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    out = torch.cat([p[:c] for p, c in zip(parts, counts)])
    assert out.shape[0] == S
    return out


def broadcast_model_bytes(model_bytes: bytes | None, device, group=None, src: int = 0) -> bytes:
    """C1: rank `src` learned the model; every rank gets the same plain-data bytes."""
    n = torch.tensor([len(model_bytes) if model_bytes is not None else 0], dtype=torch.int64, device=device)
    dist.broadcast(n, src=src, group=group)
    buf = torch.zeros(int(n.item()), dtype=torch.uint8, device=device)
    if dist.get_rank(group) == src:
        buf.copy_(torch.frombuffer(bytearray(model_bytes), dtype=torch.uint8).to(device))
    dist.broadcast(buf, src=src, group=group)
    return bytes(buf.cpu().numpy().tobytes())


def allgather_topk(dist_local: torch.Tensor, idx_local: torch.Tensor, group=None):
    """C4: every rank's (Q, k) local top-k -> (P, Q, k) on every rank."""
    world = dist.get_world_size(group)
    dl = [torch.empty_like(dist_local) for _ in range(world)]
    il = [torch.empty_like(idx_local) for _ in range(world)]
    dist.all_gather(dl, dist_local.contiguous(), group=group)
    dist.all_gather(il, idx_local.contiguous(), group=group)
    return torch.stack(dl), torch.stack(il)


def exchange_bound(bound: torch.Tensor, group=None) -> torch.Tensor:
    """C3: per query, the minimum over ranks of the local bound on the k-th best squared distance —
    a bound on the GLOBAL k-th best (the k rows behind any rank's bound are k distinct rows)."""
    dist.all_reduce(bound, op=dist.ReduceOp.MIN, group=group)
    return bound


def pack_keys(dist: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    """k = 1 exchange key: float bits of the (non-negative) distance in the high 32 bits, the global
    index in the low 32 (padding -1 -> 0xffffffff).  For d >= 0 the float bit pattern orders like the
    value, so the int64 minimum is the lexicographic (distance, index) minimum — the a9 tie rule
    (indices < 2^32 at N <= 100M)."""
    bits = dist.contiguous().view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    lo = torch.where(idx < 0, torch.full_like(idx, 0xFFFFFFFF), idx)
    return (bits << 32) | lo


def unpack_keys(key: torch.Tensor):
    bits = (key >> 32).to(torch.int32)
    d = bits.view(torch.float32)
    i = key & 0xFFFFFFFF
    return d, torch.where(i == 0xFFFFFFFF, torch.full_like(i, -1), i)


def allreduce_min_k1(dist_local: torch.Tensor, idx_local: torch.Tensor, group=None):
    """C4 for k = 1: ONE all-reduce MIN of packed (distance, index) keys instead of all-gather + merge."""
    key = pack_keys(dist_local, idx_local)
    dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
    return unpack_keys(key)


def sharded_knn(queries, k, local_knn, merge, group=None, local_seed=None):
    """Local k-NN on this rank's shard, then the exchange: k = 1 one all-reduce MIN of packed keys,
    k > 1 all-gather + min-merge (a9).  With `local_seed`, the ranks first exchange their seed bounds
    (C3) and every shard searches under the global one, so a shard that does not hold a query's
    neighbours prunes almost everything."""
    if local_seed is not None:
        bound = exchange_bound(local_seed(queries, k), group)
        d, i = local_knn(queries, k, bound)
    else:
        d, i = local_knn(queries, k)
    if k == 1:
        dd, ii = allreduce_min_k1(d.reshape(-1), i.reshape(-1), group)
        return dd.reshape(-1, 1), ii.reshape(-1, 1)
    D, I = allgather_topk(d, i, group)
    return merge(D, I)


# ------------------------------------------------------------------------------ product wiring
class ShardedSofa:
    """Product path: libsofa on this rank's GPU, NCCL for C1 / C4."""

    def __init__(self, shard: torch.Tensor, global_offset: int, global_n: int, l: int = 16, alphabet: int = 256,
                 sample_size: int = 0, block_size: int = 256, group=None):
        from . import sofa as S
        from .index import SofaIndex, learn_model  # noqa: F401

        self.group = group
        S_ = sample_size or max(alphabet, int(round(0.01 * global_n)))
        sample = gather_global_sample(shard, global_offset, global_n, S_, group)
        mb = None
        if dist.get_rank(group) == 0:
            m = S.sofa_learn_model(sample, S_, shard.shape[1], l, alphabet)
            mb = ctypes.string_at(ctypes.addressof(m), ctypes.sizeof(m))
        mb = broadcast_model_bytes(mb, shard.device, group)
        model = S.sofa_model.from_buffer_copy(mb)
        del sample
        self.index = SofaIndex(shard, l=l, alphabet=alphabet, block_size=block_size, model=model,
                               global_offset=global_offset, global_n=global_n)

    def knn(self, queries: torch.Tensor, k: int, exchange_bound: bool = True):
        from .index import merge_topk
        seed = self.index.knn_seed if exchange_bound else None
        local = (lambda qs, kk, b=None: self.index.knn(qs, kk, bsf_init=b)) if exchange_bound else self.index.knn
        return sharded_knn(queries, k, local, merge_topk, self.group, local_seed=seed)
