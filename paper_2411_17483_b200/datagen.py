"""Seeded synthetic workloads for the SOFA exact k-NN path (BASELINE.json configs).

This module is the ONLY code shared by the oracle side (tests, bench cpu leg) and the
CUDA side: it produces input bytes and holds none of the method's arithmetic (no DFT,
no binning, no lower bound, no distance).  The z-normalisation applied here is the
*input recipe* BASELINE.json states for every config ("z-normalized"), not the
method's step a1; the oracle and the kernels each re-normalise on their own.

Recipes (SURVEY.md 8(c) readings 20-23):
  * random walk  x_t = sum_{i<=t} eps_i, eps ~ N(0,1), t = 1..n       (BJ cfg1, reading 22)
  * high-freq    x_t = sum_{m=1..3} sin(2*pi*f_m*t/n + phi_m) + N(0, 0.5^2),
                 f_m ~ U(32,128) cycles/series (continuous), phi_m ~ U(0, 2*pi),
                 t = 0..n-1                                              (BJ cfg3, reading 21)
  * mixed        row i is random-walk if i is even, high-frequency if odd (BJ cfg5, reading 23)
  * noisy-member queries: dataset rows at seeded distinct indices + N(0, sigma^2), then
                 re-z-normalised; sigma fixed (cfg2: 0.1) or (0.01, 0.1, 1.0)[i mod 3] (cfg4)
All rows are z-normalised in float64 and stored as float32.

Data are generated in chunks of CHUNK_ROWS rows; chunk c of a dataset with seed s uses
its own torch generator seeded from (s, c), so any row range (a shard) can be produced
on any device independently of the number of GPUs.  CPU and CUDA generators produce
different (but each deterministic) streams; a consumer that needs the same bytes on both
sides generates once and copies.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

CHUNK_ROWS = 1 << 18


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config (index into BJ.configs in the docstring of each)."""

    name: str
    n_series: int
    length: int
    kind: str                 # "rw" | "hf" | "mixed"
    n_queries: int
    query_kind: str           # "independent" | "noisy"
    noise_sigmas: tuple = ()  # per-query sigma cycle for "noisy"
    l: int = 16
    alphabet: int = 256
    k: int = 1
    sample_size: int = 0      # 0 => round(1% N)
    seed: int = 1
    n_gpus: int = 1
    extra: dict = field(default_factory=dict)


# BJ configs[0..4]
WORKLOADS = {
    "cfg1": Workload("cfg1_rw100k_n256_l16_1nn", 100_000, 256, "rw", 100, "independent",
                     sample_size=10_000, seed=1),
    "cfg2": Workload("cfg2_rw10M_n256_l16_noisy0.1_1nn", 10_000_000, 256, "rw", 1000, "noisy",
                     noise_sigmas=(0.1,), seed=2),
    "cfg3": Workload("cfg3_hf10M_n256_l16_1nn", 10_000_000, 256, "hf", 1000, "independent", seed=3),
    "cfg4": Workload("cfg4_rw100M_n256_l16_noisymix_1nn", 100_000_000, 256, "rw", 1000, "noisy",
                     noise_sigmas=(0.01, 0.1, 1.0), seed=4, n_gpus=8),
    "cfg5": Workload("cfg5_mixed20M_n1024_l32_10nn", 20_000_000, 1024, "mixed", 1000, "independent",
                     l=32, k=10, seed=5, n_gpus=8),
}


def scaled(w: Workload, n_series: int, n_queries: int | None = None, **kw) -> Workload:
    """Same recipe at a smaller size (parity tests)."""
    d = dict(w.__dict__)
    d.update(n_series=n_series, n_queries=n_queries if n_queries is not None else w.n_queries)
    d.update(kw)
    return Workload(**d)


def default_sample_size(w: Workload) -> int:
    """Reading 6: cfg1 uses 10k; otherwise round(1% N), at least the alphabet size."""
    if w.sample_size:
        return min(w.sample_size, w.n_series)
    return min(w.n_series, max(w.alphabet, int(round(0.01 * w.n_series))))


def _gen(seed: int, stream: int, chunk: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((seed * 1_000_003 + stream * 7_919 + chunk) & 0x7FFF_FFFF_FFFF_FFFF)
    return g


def _znorm_rows(x64: torch.Tensor) -> torch.Tensor:
    mu = x64.mean(dim=1, keepdim=True)
    sd = (x64 - mu).pow(2).mean(dim=1, keepdim=True).sqrt()
    sd = torch.where(sd < 1e-12, torch.ones_like(sd), sd)
    return ((x64 - mu) / sd).to(torch.float32)


def _random_walk(rows: int, n: int, g: torch.Generator, device) -> torch.Tensor:
    eps = torch.randn(rows, n, generator=g, device=device, dtype=torch.float32)
    return torch.cumsum(eps.to(torch.float64), dim=1)


def _high_freq(rows: int, n: int, g: torch.Generator, device) -> torch.Tensor:
    f = 32.0 + 96.0 * torch.rand(rows, 3, 1, generator=g, device=device, dtype=torch.float64)
    phi = 2.0 * math.pi * torch.rand(rows, 3, 1, generator=g, device=device, dtype=torch.float64)
    t = torch.arange(n, device=device, dtype=torch.float64).view(1, 1, n)
    x = torch.sin(2.0 * math.pi * f * t / n + phi).sum(dim=1)
    noise = torch.randn(rows, n, generator=g, device=device, dtype=torch.float32)
    return x + 0.5 * noise.to(torch.float64)


def _chunk(kind: str, seed: int, c: int, rows: int, n: int, device, stream: int = 0) -> torch.Tensor:
    if kind == "rw":
        return _znorm_rows(_random_walk(rows, n, _gen(seed, stream, c, device), device))
    if kind == "hf":
        return _znorm_rows(_high_freq(rows, n, _gen(seed, stream + 1, c, device), device))
    if kind == "mixed":
        # row i (global) even -> random walk, odd -> high frequency (reading 23);
        # CHUNK_ROWS is even so parity of the global index == parity of the local one.
        out = torch.empty(rows, n, dtype=torch.float32, device=device)
        ne, no = (rows + 1) // 2, rows // 2
        out[0::2] = _znorm_rows(_random_walk(ne, n, _gen(seed, stream, c, device), device))
        if no:
            out[1::2] = _znorm_rows(_high_freq(no, n, _gen(seed, stream + 1, c, device), device))
        return out
    raise ValueError(kind)


def generate_rows(w: Workload, start: int, stop: int, device="cpu") -> torch.Tensor:
    """Rows [start, stop) of the dataset of workload w, float32 (stop-start) x n."""
    n = w.length
    out = torch.empty(max(0, stop - start), n, dtype=torch.float32, device=device)
    c0, c1 = start // CHUNK_ROWS, (stop - 1) // CHUNK_ROWS if stop > start else -1
    for c in range(c0, c1 + 1):
        lo, hi = c * CHUNK_ROWS, min((c + 1) * CHUNK_ROWS, w.n_series)
        chunk = _chunk(w.kind, w.seed, c, hi - lo, n, device)
        a, b = max(lo, start), min(hi, stop)
        out[a - start:b - start] = chunk[a - lo:b - lo]
        del chunk
    return out


def shard_range(n_series: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, as-equal-as-possible shards; the remainder goes to the last ranks."""
    base, rem = divmod(n_series, world)
    first_big = world - rem
    start = rank * base + max(0, rank - first_big)
    size = base + (1 if rank >= first_big else 0)
    return start, start + size


def query_sources(w: Workload) -> np.ndarray:
    """Seeded distinct dataset indices the noisy-member queries are drawn from."""
    rng = np.random.default_rng(w.seed * 31 + 7)
    return np.sort(rng.choice(w.n_series, size=w.n_queries, replace=False)).astype(np.int64)


def query_sigmas(w: Workload) -> np.ndarray:
    s = w.noise_sigmas or (0.0,)
    return np.array([s[i % len(s)] for i in range(w.n_queries)], dtype=np.float64)


def generate_queries(w: Workload, device="cpu", data: torch.Tensor | None = None,
                     data_offset: int = 0) -> torch.Tensor:
    """Query batch (Q x n float32).

    independent: fresh rows from the dataset generator on a separate stream.
    noisy: source rows (re-generated from their chunk seeds unless `data` holds them) plus
    N(0, sigma^2) noise, re-z-normalised.  For "mixed" independent queries, even query
    indices are random walks and odd ones high-frequency (reading 23).
    """
    n, q = w.length, w.n_queries
    if w.query_kind == "independent":
        g = _gen(w.seed, 101, 0, device)
        if w.kind == "mixed":
            out = torch.empty(q, n, dtype=torch.float32, device=device)
            out[0::2] = _znorm_rows(_random_walk((q + 1) // 2, n, g, device))
            if q // 2:
                out[1::2] = _znorm_rows(_high_freq(q // 2, n, g, device))
            return out
        if w.kind == "rw":
            return _znorm_rows(_random_walk(q, n, g, device))
        return _znorm_rows(_high_freq(q, n, g, device))
    src = query_sources(w)
    rows = torch.empty(q, n, dtype=torch.float32, device=device)
    if data is not None and data_offset <= int(src.min()) and int(src.max()) < data_offset + data.shape[0]:
        rows.copy_(data[torch.as_tensor(src - data_offset, device=data.device)].to(device))
    else:
        for c in np.unique(src // CHUNK_ROWS):
            lo, hi = int(c) * CHUNK_ROWS, min((int(c) + 1) * CHUNK_ROWS, w.n_series)
            chunk = _chunk(w.kind, w.seed, int(c), hi - lo, n, device)
            sel = np.nonzero((src >= lo) & (src < hi))[0]
            rows[torch.as_tensor(sel, device=device)] = chunk[torch.as_tensor(src[sel] - lo, device=device)]
            del chunk
    sig = torch.as_tensor(query_sigmas(w), dtype=torch.float64, device=device).view(q, 1)
    g = _gen(w.seed, 202, 0, device)
    noise = torch.randn(q, n, generator=g, device=device, dtype=torch.float32).to(torch.float64)
    return _znorm_rows(rows.to(torch.float64) + sig * noise)
