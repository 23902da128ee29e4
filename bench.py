#!/usr/bin/env python
"""Benchmark of the B200-native SOFA exact k-NN path (BASELINE.json metric: exact k-NN queries/sec).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl sofa|reference]

With --gpus N > 1 and no torchrun environment (WORLD_SIZE unset), bench.py re-executes itself under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU) and fails if fewer than N GPUs
are visible (SOFA_DIST_BACKEND=gloo allows N ranks on fewer GPUs: a check of the multi-rank code path,
never a measurement).

A step = one exact k-NN batch (all Q queries of the config) through libsofa's query kernel
(a5-a8) on an index built over the synthetic dataset (a1-a4, timed separately as `build`), plus
the NCCL all-gather + merge kernel (a9) when N > 1.  Data and queries are resident in HBM when
the timed region starts; L2 is flushed (512 MB write) between timed steps; each step is timed with
CUDA events on the launching stream; max over ranks.  N > 1 shards the same dataset over the
ranks (strong scaling).  `e2e` repeats the measurement through the host-buffer C call
(sofa_knn_host: pinned host queries in, host results out).  `--impl reference` times the CPU
float64 oracle (the reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2411_17483_b200 import datagen  # noqa: E402

METRIC = "exact k-NN queries/sec"
UNIT = "queries/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    # default: BASELINE.json configs[3] (100M random walks, noisy-member mix, 1-NN) — the config the metric
    # "queries/sec at 1/2/4/8 B200" is quoted on; it fits one B200 (102.4 GB of rows + ~4 GB of index)
    p.add_argument("--config", default="cfg4", choices=sorted(datagen.WORKLOADS))
    p.add_argument("--impl", default="sofa", choices=["sofa", "reference"])
    p.add_argument("--n-series", type=int, default=0, help="override N (debug only; changes the workload)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-flush", action="store_true",
                   help="diagnostic: skip the L2 flush between timed steps (inputs are larger than L2 anyway)")
    return p.parse_args()


HBM_NOMINAL_GBS = 8000.0    # BASELINE.json north_star "roughly 8 TB/s" (DGX figure; HGX 7.7)


def lib_fingerprint() -> str | None:
    p = os.path.join(ROOT, "paper_2411_17483_b200", "lib", "libsofa.sha256")
    return open(p).read().strip() if os.path.exists(p) else None


def load_traffic(config: str) -> dict | None:
    """profiles/traffic_<config>.json: DRAM bytes per step of each kernel group from an ncu capture
    (tools/traffic.py), valid only for the library build it was captured on."""
    tp = os.path.join(ROOT, "profiles", f"traffic_{config}.json")
    if not os.path.exists(tp):
        return None
    d = json.load(open(tp))
    if d.get("lib_fingerprint") != lib_fingerprint():
        return None
    return d.get("groups")


def dense_roofline(st, km, rows, w, bf16, bf16_kind):
    """dense pass (f1): 2 * queries * rows * n flops of the bf16 screen GEMM (k_dense_screen: tcgen05
    kind::f16, fp32 accumulation in TMEM) over the screen's own time, against the measured bf16 rate;
    the exact refine of its candidates (k_dense_post) is reported beside it"""
    flops = 2.0 * st["dense_queries"] * rows * w.length
    ms = km.get("dense_screen") or km["dense"]
    dn = {"bound": "tensor", "achieved": flops / (ms / 1e3) / 1e12, "peak": bf16, "unit": "TFLOP/s",
          "kernel": "k_dense_screen (tcgen05 kind::f16, bf16 operands)", "group": "dense",
          "kernel_ms": ms, "dense_pass_ms": km["dense"], "refine_ms": km.get("dense_post"),
          "algorithmic_flops_per_launch": flops, "peak_note": f"{bf16_kind} {bf16:.1f} TFLOP/s",
          "peak_nominal": 2250.0}
    dn["frac"] = dn["achieved"] / bf16
    dn["frac_nominal"] = dn["achieved"] / 2250.0
    # the screen streams the rows' bf16 copy once per pass (2 n bytes per row; query groups share it)
    dn["stream_bytes"] = rows * w.length * 2
    dn["stream_gb_per_s"] = dn["stream_bytes"] / (ms / 1e3) / 1e9
    return dn


def build_report(index, build_ms, rows, w):
    """build (a1-a4) time and its phases (sofa_get_info.build_ms, CUDA events on the build stream); the
    transform (a1 + a3) reads the rows once and writes words, statistics and the bf16 row copy"""
    ph = index.info["build_ms"]
    series = rows * w.length * 4
    written = rows * (16 * ((w.l + 15) // 16) + 8 + 8 + 2 * w.length)
    return {"ms": build_ms, "gb_per_s_series_read": series / (build_ms / 1e3) / 1e9, "phases_ms": ph,
            "transform_gb_per_s": (series + written) / (ph["transform"] / 1e3) / 1e9 if ph["transform"] > 0 else None,
            "transform_bytes": series + written}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def tensor_peak():
    """bf16 dense TFLOP/s and which figure: the measured SUSTAINED rate (MEASURED_PEAKS.json) — the
    dense pass runs inside back-to-back steps of 10-60 ms, i.e. under the sustained power/clock
    regime, not alone — else the measured burst, else the guide's fallback."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        if "bf16_tflops_sustained" in d:
            return float(d["bf16_tflops_sustained"]), "measured bf16 sustained"
        return float(d["bf16_tflops"]), "measured bf16 burst"
    return 1590.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev, self.rows, self.proc = dev, [], None
        self.period_ms = int(os.environ.get("SOFA_BENCH_SMI_MS", "100"))

    def __enter__(self):
        try:
            if self.period_ms <= 0:  # diagnostic only (SOFA_BENCH_SMI_MS=0): no clock record
                return self
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.dev), "-lms", str(self.period_ms)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_sample(w, rows: int, nq: int, x_host: np.ndarray | None = None, q_host: np.ndarray | None = None):
    """Time the CPU oracle (brute force, float64) for nq queries over `rows` rows; returns (q/s
    extrapolated to the full N, seconds, sample description)."""
    from oracle import sofa_oracle as O
    if x_host is None:
        x_host = datagen.generate_rows(w, 0, rows).numpy()
    if q_host is None:
        q_host = datagen.generate_queries(datagen.scaled(w, w.n_series, nq)).numpy()[:nq]
    t0 = time.perf_counter()
    O.knn_bruteforce(x_host, q_host, w.k)
    dt = time.perf_counter() - t0
    per_query_full = dt / nq * (w.n_series / rows)
    return 1.0 / per_query_full, dt, f"{nq} queries x first {rows:,} of {w.n_series:,} rows, brute force float64, " \
                                     f"time extrapolated linearly in N"


def run_reference(a, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch as _t
    _t.set_num_threads(cores())
    rows = min(w.n_series, 250_000 if w.length <= 256 else 60_000)
    nq = 4
    x = datagen.generate_rows(w, 0, rows).numpy()
    qh = datagen.generate_queries(datagen.scaled(w, w.n_series, nq) if w.query_kind == "independent"
                                  else datagen.scaled(w, rows, nq), data=None).numpy()[:nq]
    vals = []
    for s in range(a.warmup + a.steps):
        v, dt, desc = oracle_sample(w, rows, nq, x, qh)
        if s >= a.warmup:
            vals.append((v, dt))
    v = statistics.median([x[0] for x in vals])
    ms = statistics.median([x[1] for x in vals]) * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "n_series": w.n_series, "length": w.length, "l": w.l, "alphabet": w.alphabet,
                       "k": w.k, "queries": w.n_queries},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores(), "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def flush_l2(buf):
    buf.zero_()


def self_launch(a):
    """--gpus N > 1 without a torchrun environment: re-exec under torch.distributed.run (N ranks)."""
    if a.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    if a.impl != "reference" and os.environ.get("SOFA_DIST_BACKEND", "nccl") == "nccl":
        have = torch.cuda.device_count()
        if have < a.gpus:
            sys.exit(f"bench.py: --gpus {a.gpus} needs {a.gpus} visible GPUs, found {have}")
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    a = parse()
    self_launch(a)
    w = datagen.WORKLOADS[a.config]
    if a.n_series:
        w = datagen.scaled(w, a.n_series, w.n_queries)
    if a.impl == "reference":
        run_reference(a, w)
        return

    from paper_2411_17483_b200 import sofa as S
    from paper_2411_17483_b200.index import SofaIndex

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local %= max(1, torch.cuda.device_count())  # one GPU per rank; a 1-GPU box can still run a smoke
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        import torch.distributed as dist
        # NCCL over NVLink; SOFA_DIST_BACKEND=gloo runs the same sharded path with several ranks on one
        # GPU (a check of the multi-rank code path, not a measurement)
        backend = os.environ.get("SOFA_DIST_BACKEND", "nccl")
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    lo, hi = datagen.shard_range(w.n_series, rank, world)

    # ---------------------------------------------------------------- data (resident in HBM)
    x = datagen.generate_rows(w, lo, hi, device=dev)
    q = datagen.generate_queries(w, device=dev, data=x if world == 1 else None, data_offset=lo)
    torch.cuda.synchronize()

    # ---------------------------------------------------------------- build (a1-a4), timed separately
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if world == 1:
        ix = SofaIndex(x, l=w.l, alphabet=w.alphabet, sample_size=datagen.default_sample_size(w))
        knn = lambda qq: ix.knn(qq, w.k)  # noqa: E731
        index = ix
    else:
        from paper_2411_17483_b200.distributed import ShardedSofa
        sh = ShardedSofa(x, lo, w.n_series, l=w.l, alphabet=w.alphabet, sample_size=datagen.default_sample_size(w))
        knn = lambda qq: sh.knn(qq, w.k)  # noqa: E731
        index = sh.index
    e1.record()
    torch.cuda.synchronize()
    build_ms = e0.elapsed_time(e1)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    l2 = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for _ in range(a.warmup):
        knn(q)
    torch.cuda.synchronize()
    # pruning statistics of this shard (same work as a step: with N > 1, under the exchanged bound)
    if world == 1:
        _, _, st = index.knn(q, w.k, stats=True)
    else:
        from paper_2411_17483_b200.distributed import exchange_bound
        _, _, st = index.knn(q, w.k, bsf_init=exchange_bound(index.knn_seed(q, w.k)), stats=True)

    # ---------------------------------------------------------------- timed steps
    times = []
    km_steps = []
    launches0 = S.sofa_launch_count()
    index.kernel_timing(1)  # per-kernel-group CUDA events inside every timed step (no sync)
    with Clocks(local) as clk:
        for s in range(a.steps):
            if not a.no_flush:
                flush_l2(l2)
            barrier()
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            d, i = knn(q)
            s1.record()
            torch.cuda.synchronize()
            barrier()
            times.append(s0.elapsed_time(s1))
            km_step, _ = index.kernel_timing(1)  # this step's groups (after the sync; restarts the totals)
            km_steps.append(km_step)
        launches = S.sofa_launch_count() - launches0
        index.kernel_timing(0)
        km_tot = {kk: sum(m[kk] for m in km_steps) for kk in km_steps[0]}
        # keep sampling clocks for a short sustained run of the same step (no timing taken)
        t_end = time.time() + 1.0
        while time.time() < t_end:
            knn(q)
        torch.cuda.synchronize()
    tot_ms = max_over_ranks(sum(times))
    ms_per_step = tot_ms / a.steps
    value = w.n_queries * a.steps / (tot_ms / 1e3)

    # ---------------------------------------------------------------- roofline of the dominant kernel
    # Per-kernel GPU times: the library's CUDA events on the launching stream, recorded inside every
    # timed step (sofa_kernel_timing) and averaged over the K steps: front (a5-a8 per query), dense
    # pass (tcgen05 TF32 screen + exact refine, f1) and scan (a7-a8 task pool).  The work counts
    # (words, refines, ...) come from the stats call before the timed region (same inputs).
    hbm, peak_kind = peaks()
    bf16, bf16_kind = tensor_peak()
    km = {kk: v / a.steps for kk, v in km_tot.items()}
    l_b, n_b = w.l, 4 * w.length
    # sparse path (front + scan): algorithmic bytes = envelope nodes (2l B) + words scanned (l B)
    # + rows refined (4n B) + query rows (4n B)  (SURVEY 8(d) unit costs)
    sparse_bytes = (st["env_nodes"] * 2 * l_b + st["words_scanned"] * l_b + st["refined"] * n_b
                    + st["queries"] * n_b)
    sparse_ms = km["front"] + km["scan"]
    sparse = {"bound": "hbm", "achieved": sparse_bytes / (sparse_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
              "kernel": "k_query front + scan (a5-a8)", "group": "sparse", "kernel_ms": sparse_ms,
              "algorithmic_bytes_per_launch": sparse_bytes}
    sparse["frac"] = sparse["achieved"] / hbm
    # report against both the measured copy rate and the north star's ~8 TB/s nominal
    sparse["peak_nominal"] = HBM_NOMINAL_GBS
    sparse["frac_nominal"] = sparse["achieved"] / HBM_NOMINAL_GBS
    rooflines = [sparse]
    if st["dense_queries"] > 0 and km["dense"] > 0:
        rooflines.append(dense_roofline(st, km, hi - lo, w, bf16, bf16_kind))
    # DRAM bytes per step of each group, from the ncu capture of THIS build (the library fingerprint
    # must match, else the number is from other kernels and is not reported)
    traffic = load_traffic(a.config)
    for r in rooflines:
        tb = traffic.get(r["group"]) if traffic else None
        r["dram_bytes_per_launch"] = tb
        if tb:
            r["dram_gbs"] = tb / (r["kernel_ms"] / 1e3) / 1e9
            r["dram_frac"] = r["dram_gbs"] / hbm
            r["dram_frac_nominal"] = r["dram_gbs"] / HBM_NOMINAL_GBS
    dominant = max(rooflines, key=lambda r: r["kernel_ms"])
    roofline = dict(dominant, traffic=dominant.get("dram_bytes_per_launch"), peak_kind=peak_kind,
                    share_of_step=dominant["kernel_ms"] / (km["front"] + km["dense"] + km["scan"]))

    # ---------------------------------------------------------------- e2e through the host C call
    e2e = None
    if not a.no_e2e:
        qh = torch.empty(q.shape, dtype=torch.float32, pin_memory=True)
        qh.copy_(q)
        qhn = qh.numpy()
        od = torch.empty(w.n_queries, w.k, dtype=torch.float32, pin_memory=True).numpy()
        oi = torch.empty(w.n_queries, w.k, dtype=torch.int64, pin_memory=True).numpy()
        et = []
        for s in range(a.warmup + a.steps):
            flush_l2(l2)
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if world == 1:
                index.knn_host(qhn, w.k, out=(od, oi))
            else:
                qd = qh.to(dev, non_blocking=True)
                dd, ii = knn(qd)
                dd.cpu(), ii.cpu()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            barrier()
            if s >= a.warmup:
                et.append(dt)
        e_tot = max_over_ranks(sum(et))
        e2e = {"value": w.n_queries * a.steps / e_tot, "unit": UNIT,
               "h2d_bytes_per_step": int(w.n_queries * w.length * 4),
               "d2h_bytes_per_step": int(w.n_queries * w.k * 12)}

    # ---------------------------------------------------------------- cpu brute-force scan (UCR Suite-P style)
    # BASELINE.json north_star: "a multithreaded CPU brute-force scan, timed on the box's host cores in
    # the same run"; rank 0, N=1; a bounded sample (8 queries over up to 10M rows), extrapolated in N
    cpu_scan_line = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        import cpu_scan
        rows = min(w.n_series, 10_000_000 if w.length <= 256 else 2_500_000)
        xs = x[:rows].cpu().numpy()
        qs = q[:8].cpu().numpy()
        stats_h = cpu_scan.row_stats(xs)
        cpu_scan.knn(xs, stats_h, qs[:1], w.k, threads=cores())  # warm-up (page faults, threads)
        t0 = time.perf_counter()
        cpu_scan.knn(xs, stats_h, qs, w.k, threads=cores())
        dt = time.perf_counter() - t0
        per_q = dt / len(qs) * (w.n_series / rows)
        cpu_scan_line = {"value": 1.0 / per_q, "unit": UNIT, "cores": cores(), "kind": "ucr-suite-p-style OpenMP "
                         "float32 brute force, early abandoning (cpu_scan/)", "seconds": dt,
                         "sample": f"{len(qs)} queries x first {rows:,} of {w.n_series:,} rows, time extrapolated "
                                   "linearly in N"}
        del xs

    # ---------------------------------------------------------------- cpu baseline (oracle), rank 0, N=1
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        torch.set_num_threads(cores())
        # ~10 s of host work on 16 cores: the oracle's cost is per row (float64 z-normalisation + GEMM),
        # so the sample is sized in rows; 3M x 256 needs ~20 GB of host memory in float64 copies
        import psutil
        big = psutil.virtual_memory().available > 96e9
        rows = min(w.n_series, (3_000_000 if big else 1_000_000) * 256 // max(256, w.length))
        nq = 16
        xs = x[:rows].cpu().numpy()
        qs = q[:nq].cpu().numpy()
        v, dt, desc = oracle_sample(w, rows, nq, xs, qs)
        cpu = {"value": v, "unit": UNIT, "cores": cores(), "kind": "oracle", "sample": desc, "seconds": dt}

    if rank == 0:
        N = w.n_series
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": w.name, "n_series": N, "length": w.length, "l": w.l, "alphabet": w.alphabet,
                       "k": w.k, "queries": w.n_queries, "block_size": 256,
                       "sample_size": datagen.default_sample_size(w),
                       "l2": "not flushed (inputs larger than L2)" if a.no_flush else "flushed between timed steps (512 MB write)", "parallelism": f"shard{world}"},
            "prune": {"series": 1.0 - st["refined"] / (st["queries"] * (hi - lo)),
                      "block": 1.0 - st["blocks_survived"] / max(1, st["blocks_total"]),
                      "refined_per_query": st["refined"] / st["queries"],
                      "words_scanned_per_query": st["words_scanned"] / st["queries"]},
            "knn_stats": st,
            "build": build_report(index, build_ms, hi - lo, w),
            "roofline": roofline, "roofline_all": rooflines, "kernel_ms": km, "step_ms": [round(t, 4) for t in times],
            "kernel_ms_steps": {kk: [round(m[kk], 4) for m in km_steps] for kk in km},
            "cpu_baseline": cpu, "cpu_scan": cpu_scan_line, "e2e": e2e, "clocks": clk.summary(), "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    index.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
