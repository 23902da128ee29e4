"""User-facing API over the C ABI: build an index over a device-resident float32 tensor and run
exact k-NN batches.  All compute happens in libsofa.so; this module only allocates outputs and
marshals pointers."""
from __future__ import annotations

import numpy as np
import torch

from . import sofa as S


class SofaIndex:
    """SOFA exact z-ED k-NN index over `series` (N x len float32, CUDA, borrowed: keep it alive).

    Parameters mirror sofa_build_opts (include/sofa.h).  `model` (dict or sofa_model) skips
    learning (sharded builds pass the global model here)."""

    def __init__(self, series: torch.Tensor, l: int = 16, alphabet: int = 256, *, block_size: int = 256,
                 sample_size: int = 0, sample_ratio: float = 0.01, binning: str = "equi-depth",
                 candidate_limit: int = 0, model=None, global_offset: int = 0, global_n: int = 0,
                 dense_permille: int = 0, stream=None):
        if not (series.is_cuda and series.dtype == torch.float32 and series.dim() == 2 and series.is_contiguous()):
            raise ValueError("series must be a contiguous 2-D float32 CUDA tensor")
        self.series = series
        self.n, self.len = series.shape
        opts = S.sofa_default_opts()
        opts.sample_size, opts.sample_ratio, opts.block_size = sample_size, sample_ratio, block_size
        opts.binning, opts.candidate_limit = S.BINNING[binning], candidate_limit
        opts.global_offset, opts.global_n = global_offset, global_n
        opts.dense_permille = dense_permille
        self._model_keep = None
        if model is not None:
            m = model if isinstance(model, S.sofa_model) else S.sofa_model.from_dict(model)
            self._model_keep = m
            opts.model = S.C.pointer(m)
        self.handle = S.sofa_build(series, self.n, self.len, l, alphabet, opts, stream)
        self.k_max = S.MAX_K
        self._host_bufs = {}

    def set_tuning(self, **fields):
        """Query-kernel tuning (sofa_set_tuning; include/sofa.h sofa_tuning): fields not given keep
        their defaults.  Changes the order of work only, never a result."""
        t = S.sofa_default_tuning()
        for kk, v in fields.items():
            if kk not in dict(t._fields_):
                raise KeyError(kk)
            setattr(t, kk, int(v))
        S.sofa_set_tuning(self.handle, t)

    # -------------------------------------------------------------------------------- queries
    def knn(self, queries: torch.Tensor, k: int = 1, bsf_init: torch.Tensor | None = None, stats: bool = False,
            out=None, stream=None):
        """Exact k-NN of a device batch (q x len float32).  Returns (dist, idx[, stats])."""
        q = queries.shape[0]
        if out is None:
            dist = torch.empty(q, k, dtype=torch.float32, device=queries.device)
            idx = torch.empty(q, k, dtype=torch.int64, device=queries.device)
        else:
            dist, idx = out
        st = S.sofa_knn_stats() if stats else None
        S.sofa_knn(self.handle, queries.contiguous(), q, k, bsf_init, dist, idx, st, stream)
        return (dist, idx, st.to_dict()) if stats else (dist, idx)

    def knn_host(self, queries: np.ndarray, k: int = 1, out=None, stream=None):
        """End-to-end path: host queries in, host results out (copies inside the C call)."""
        queries = np.ascontiguousarray(queries, dtype=np.float32)
        q = queries.shape[0]
        if out is None:
            out = (np.empty((q, k), dtype=np.float32), np.empty((q, k), dtype=np.int64))
        S.sofa_knn_host(self.handle, queries, q, k, out[0], out[1], None, stream)
        return out

    def knn_seed(self, queries: torch.Tensor, k: int = 1, stream=None) -> torch.Tensor:
        """(q,) float32: this index's seed bound on each query's k-th best squared distance (the
        k-th best of the rows its seed step refines; +inf if fewer).  Sharded search all-reduces
        the minimum over shards and passes it as `bsf_init` (distributed.ShardedSofa)."""
        out = torch.empty(queries.shape[0], dtype=torch.float32, device=queries.device)
        S.sofa_knn_seed(self.handle, queries.contiguous(), queries.shape[0], k, out, stream)
        return out

    def lower_bounds(self, queries: torch.Tensor, m: int, stream=None):
        """(lb2, ed2, rows): squared lower bounds and exact squared z-ED of each query against m index
        rows (sorted positions floor(j n / m)); TLB = sqrt(lb2 / ed2)."""
        q = queries.shape[0]
        lb2 = torch.empty(q, m, dtype=torch.float32, device=queries.device)
        ed2 = torch.empty(q, m, dtype=torch.float32, device=queries.device)
        rows = torch.empty(m, dtype=torch.int64, device=queries.device)
        S.sofa_lower_bounds(self.handle, queries.contiguous(), q, m, lb2, ed2, rows, stream)
        return lb2, ed2, rows

    def kernel_timing(self, enable: int = -1) -> tuple[dict, int]:
        """Live per-launch-group GPU times of knn calls: returns the totals recorded since the last
        (re)start ({front, dense, scan} ms, sub-batches), then starts (1), stops (0) or keeps (-1)
        timing.  CUDA events only, no synchronisation inside knn (include/sofa.h)."""
        return S.sofa_kernel_timing(self.handle, enable)

    # -------------------------------------------------------------------------------- introspection
    @property
    def model(self) -> dict:
        return S.sofa_get_model(self.handle).to_dict()

    @property
    def raw_model(self) -> S.sofa_model:
        return S.sofa_get_model(self.handle)

    @property
    def info(self) -> dict:
        i = S.sofa_get_info(self.handle)
        d = {f: int(getattr(i, f)) for f, _ in i._fields_ if f != "build_ms"}
        d["build_ms"] = dict(zip(("model", "transform", "sort", "gather_envelopes"), map(float, i.build_ms)))
        return d

    def export(self) -> dict:
        inf = self.info
        dev = self.series.device
        w = torch.empty(inf["n"], inf["word_stride"], dtype=torch.uint8, device=dev)
        p = torch.empty(inf["n"], dtype=torch.int32, device=dev)
        e = torch.empty(inf["n_blocks"], 2, inf["word_stride"], dtype=torch.uint8, device=dev)
        kk = torch.empty(inf["n_blocks"], dtype=torch.int64, device=dev)
        S.sofa_export_index(self.handle, w, p, e, kk)
        return {"words": w, "perm": p, "env": e, "block_keys": kk}

    def close(self):
        if getattr(self, "handle", None):
            S.sofa_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def merge_topk(dist: torch.Tensor, idx: torch.Tensor, stream=None):
    """a9: (P, q, k) per-shard sorted lists -> (q, k) global top-k (libsofa kernel)."""
    P, q, k = dist.shape
    od = torch.empty(q, k, dtype=torch.float32, device=dist.device)
    oi = torch.empty(q, k, dtype=torch.int64, device=dist.device)
    S.sofa_merge_topk(dist.contiguous(), idx.contiguous(), P, q, k, od, oi, stream)
    return od, oi


def transform(series: torch.Tensor, model, stream=None):
    """a1+a3 parity entry point: (values float64 n x l, words uint8 n x l) under `model`."""
    m = model if isinstance(model, S.sofa_model) else S.sofa_model.from_dict(model)
    n = series.shape[0]
    vals = torch.empty(n, m.l, dtype=torch.float64, device=series.device)
    words = torch.empty(n, m.l, dtype=torch.uint8, device=series.device)
    S.sofa_transform(series.contiguous(), n, m, vals, words, stream)
    return vals, words


def learn_model(sample: torch.Tensor, l: int, alphabet: int, binning: str = "equi-depth", candidate_limit: int = 0,
                stream=None) -> dict:
    opts = S.sofa_default_opts()
    opts.binning, opts.candidate_limit = S.BINNING[binning], candidate_limit
    m = S.sofa_learn_model(sample.contiguous(), sample.shape[0], sample.shape[1], l, alphabet, opts, stream)
    return m.to_dict()
