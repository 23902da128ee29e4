"""Build-side sweeps on one GPU, synthetic analogs of the paper's
  * build-time split (Fig. 7): GPU time of model learning, transform, sort, envelopes;
  * sampling rate (Table 4): sample fraction vs build time, mean TLB, query throughput;
  * leaf size (Fig. 11): block size B vs query throughput and pruning.
The paper's datasets are not available; BASELINE.json's configs[1] (10M random walks, 1000
noisy-member queries) and configs[2] (10M high-frequency, 1000 random queries) stand in.
python tools/build_sweeps.py [N] > profiles/r02_build_sweeps.md"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17483_b200 import datagen  # noqa: E402
from paper_2411_17483_b200.index import SofaIndex  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000


def time_knn(ix, q, k, reps=9):
    ix.knn(q, k)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ix.knn(q, k)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def mean_tlb(ix, q, m=10_000):
    lb2, ed2, _ = ix.lower_bounds(q[:50], m)
    ok = ed2 > 0
    return float(torch.sqrt(lb2[ok].double() / ed2[ok].double()).mean())


out = {"N": N, "split": {}, "sampling": {}, "leaf_size": {}}
for kind in ("cfg2", "cfg3"):
    w = datagen.scaled(datagen.WORKLOADS[kind], N, 1000)
    x = datagen.generate_rows(w, 0, N, device="cuda")
    q = datagen.generate_queries(w, device="cuda", data=x)
    torch.cuda.synchronize()
    print(f"## {w.name} (N = {N:,}, 1000 queries, k = {w.k})\n")
    # build-time split at the default sampling rate (1%): the fastest of 3 builds (the first one
    # pays module loading and allocator growth)
    splits = []
    for _ in range(3):
        ix = SofaIndex(x, sample_size=datagen.default_sample_size(w))
        splits.append(ix.info["build_ms"])
        ix.close()
    bm = min(splits, key=lambda b: sum(b.values()))
    out["split"][kind] = bm
    tot = sum(bm.values())
    print("Build-time split (Fig. 7 analog), GPU ms: " + ", ".join(f"{k} {v:.2f} ({v / tot:.0%})" for k, v in bm.items())
          + f"; total {tot:.2f} ms = {N * w.length * 4 / (tot / 1e3) / 1e9:.0f} GB/s of rows\n")
    # sampling rate (Table 4 analog)
    print("| sample | rows | model ms | build ms | mean TLB | query ms (1000 q) | q/s | refined/query |")
    print("|---|---|---|---|---|---|---|---|")
    out["sampling"][kind] = []
    for frac in (0.001, 0.005, 0.01, 0.05, 0.1, 0.2):
        S = max(256, int(round(frac * N)))
        ix = SofaIndex(x, sample_size=S)
        bm = ix.info["build_ms"]
        ms = time_knn(ix, q, w.k)
        _, _, st = ix.knn(q, w.k, stats=True)
        tl = mean_tlb(ix, q)
        row = {"frac": frac, "S": S, "model_ms": bm["model"], "build_ms": sum(bm.values()), "tlb": tl, "knn_ms": ms,
               "qps": 1000 / (ms / 1e3), "refined_per_query": st["refined"] / 1000}
        out["sampling"][kind].append(row)
        print(f"| {frac:.1%} | {S:,} | {bm['model']:.2f} | {row['build_ms']:.2f} | {tl:.3f} | {ms:.3f} | {row['qps']:,.0f} | "
              f"{row['refined_per_query']:.1f} |")
        ix.close()
    print()
    # leaf size (Fig. 11 analog)
    print("| block size B | query ms (1000 q) | q/s | leaves scanned/query | words/query | refined/query | dense |")
    print("|---|---|---|---|---|---|---|")
    out["leaf_size"][kind] = []
    for B in (64, 128, 256, 512, 1024, 2048, 4096):
        ix = SofaIndex(x, sample_size=datagen.default_sample_size(w), block_size=B)
        ms = time_knn(ix, q, w.k)
        _, _, st = ix.knn(q, w.k, stats=True)
        row = {"B": B, "knn_ms": ms, "qps": 1000 / (ms / 1e3), "leaves": st["blocks_survived"] / 1000,
               "words": st["words_scanned"] / 1000, "refined": st["refined"] / 1000, "dense": st["dense_queries"]}
        out["leaf_size"][kind].append(row)
        print(f"| {B} | {ms:.3f} | {row['qps']:,.0f} | {row['leaves']:.1f} | {row['words']:.0f} | {row['refined']:.1f} | "
              f"{row['dense']} |")
        ix.close()
    print()
    del x, q
    torch.cuda.empty_cache()
print("```json\n" + json.dumps(out) + "\n```")
