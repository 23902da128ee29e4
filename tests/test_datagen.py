"""Input recipe checks: determinism, shard independence, shapes."""
import numpy as np
import torch

from paper_2411_17483_b200 import datagen


def test_rows_deterministic_and_shard_independent():
    w = datagen.scaled(datagen.WORKLOADS["cfg1"], 3 * datagen.CHUNK_ROWS // 256, 4)
    full = datagen.generate_rows(w, 0, w.n_series)
    again = datagen.generate_rows(w, 0, w.n_series)
    assert torch.equal(full, again)
    for world in (2, 3):
        parts = [datagen.generate_rows(w, *datagen.shard_range(w.n_series, r, world)) for r in range(world)]
        assert torch.equal(torch.cat(parts), full)


def test_chunk_boundary_and_znorm():
    w = datagen.scaled(datagen.WORKLOADS["cfg3"], datagen.CHUNK_ROWS + 5, 3, length=32)
    a = datagen.generate_rows(w, datagen.CHUNK_ROWS - 3, datagen.CHUNK_ROWS + 5)
    b = datagen.generate_rows(w, datagen.CHUNK_ROWS - 3, datagen.CHUNK_ROWS)
    assert torch.equal(a[:3], b)
    x = a.double()
    assert x.mean(1).abs().max() < 1e-5 and ((x.std(1, unbiased=False) - 1).abs().max() < 1e-4)


def test_shard_range_covers():
    for N in (10, 11, 100_000_000):
        for P in (1, 2, 3, 8):
            r = [datagen.shard_range(N, i, P) for i in range(P)]
            assert r[0][0] == 0 and r[-1][1] == N
            assert all(r[i][1] == r[i + 1][0] for i in range(P - 1))
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1


def test_queries():
    w = datagen.scaled(datagen.WORKLOADS["cfg4"], 5000, 9)
    data = datagen.generate_rows(w, 0, w.n_series)
    q1 = datagen.generate_queries(w, data=data)
    q2 = datagen.generate_queries(w)             # regenerates source rows from chunk seeds
    assert torch.equal(q1, q2)
    assert list(datagen.query_sigmas(w)[:4]) == [0.01, 0.1, 1.0, 0.01]
    src = datagen.query_sources(w)
    assert len(np.unique(src)) == 9
    w5 = datagen.scaled(datagen.WORKLOADS["cfg5"], 64, 6, length=64)
    x = datagen.generate_rows(w5, 0, 64)
    assert x.shape == (64, 64)
    assert datagen.generate_queries(w5).shape == (6, 64)
