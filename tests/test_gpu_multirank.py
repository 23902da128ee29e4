"""The multi-GPU code path on a one-GPU box: 2 ranks (torch.distributed, gloo, both on cuda:0 — their
kernels never wait on each other) build shard indices with the GLOBAL model (strided sample
all-gather C1, model byte broadcast), answer the same queries, all-gather their local top-k (C4)
and min-merge with the libsofa kernel (a9).  The merged answer must equal a single index over all
rows, bit for bit.  On an 8-GPU box the same code runs over NCCL (bench.py --gpus N)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import os, sys, torch, numpy as np
import torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"])
from paper_2411_17483_b200 import datagen
from paper_2411_17483_b200.distributed import ShardedSofa
from paper_2411_17483_b200.index import SofaIndex
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group(os.environ.get("BACKEND", "gloo"))
w = datagen.scaled(datagen.WORKLOADS[os.environ["CFG"]], int(os.environ["N"]), 64, k=int(os.environ["K"]))
a, b = datagen.shard_range(w.n_series, rank, world)
shard = datagen.generate_rows(w, a, b, device="cuda")
q = datagen.generate_queries(w, device="cuda")
sh = ShardedSofa(shard, a, w.n_series, l=w.l, sample_size=4000)
d, i = sh.knn(q, w.k)
if rank == 0:
    x = datagen.generate_rows(w, 0, w.n_series, device="cuda")
    ref = SofaIndex(x, l=w.l, sample_size=4000)
    d0, i0 = ref.knn(q, w.k)
    same = torch.equal(i.cuda(), i0) and torch.equal(d.cuda(), d0)
    print("MERGED_EQUALS_SINGLE", same, flush=True)
dist.barrier()
dist.destroy_process_group()
"""


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("cfg,N,k", [("cfg1", 50_001, 1), ("cfg4", 60_000, 5), ("cfg3", 30_000, 3)])
def test_two_ranks_on_one_gpu_equal_single_index(cfg, N, k, tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, ROOT=ROOT, CFG=cfg, N=str(N), K=str(k))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", str(script)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "MERGED_EQUALS_SINGLE True" in r.stdout, r.stdout[-2000:]


@pytest.mark.parametrize("cfg,N,k", [("cfg1", 40_000, 1), ("cfg3", 30_000, 3)])
def test_nccl_path_on_one_rank(cfg, N, k, tmp_path):
    """the sharded pipeline over NCCL itself (one rank: this pool has one GPU per box): the model
    broadcast, the seed-bound all-reduce MIN, and the k = 1 packed-key all-reduce MIN / k > 1
    all-gather + min-merge run as real NCCL collectives on cuda:0; the answer equals a single index"""
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, ROOT=ROOT, CFG=cfg, N=str(N), K=str(k), BACKEND="nccl")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", str(script)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "MERGED_EQUALS_SINGLE True" in r.stdout, r.stdout[-2000:]
