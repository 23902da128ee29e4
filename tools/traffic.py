"""DRAM bytes per step of each kernel group (bench.py `roofline.traffic`), from one ncu pass over a
bench step of THIS library build: `python tools/traffic.py cfg4` (on the GPU box) writes
profiles/traffic_cfg4.json with the library fingerprint bench.py checks before using it.

The last bench step's launches are used (front k_query, k_dense_screen, k_dense_post, scan k_query);
ncu serialises the launches and flushes caches between them, so these are cold-cache bytes."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
metrics = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
cmd = ["ncu", "--metrics", metrics, "--clock-control", "none", "--csv", "-k", "regex:k_query|k_dense_screen|k_dense_post",
       sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", "1", "--warmup", "3",
       "--no-cpu-baseline", "--no-e2e"]
out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT).stdout
rows = [r for r in csv.reader(io.StringIO(out[out.index('"ID"'):]))]
hdr = rows[0]
iK, iM, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
iID = hdr.index("ID")
launches = {}
for r in rows[1:]:
    if len(r) <= iV:
        continue
    d = launches.setdefault(int(r[iID]), {"kernel": r[iK]})
    unit_scale = 1.0
    v = float(r[iV].replace(",", ""))
    d[r[iM]] = v
ids = sorted(launches)
# the last step: the last 4 launches (front, screen, post, scan)
step = [launches[i] for i in ids[-4:]]
assert "k_query" in step[0]["kernel"] and "k_dense_screen" in step[1]["kernel"] and "k_query" in step[3]["kernel"], \
    [s["kernel"] for s in step]
units = {}
for r in rows[1:]:
    if len(r) > iV and r[iM] == "dram__bytes_read.sum":
        units["dram"] = r[hdr.index("Metric Unit")]
    if len(r) > iV and r[iM] == "gpu__time_duration.sum":
        units["time"] = r[hdr.index("Metric Unit")]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units.get("dram", "byte")]


def b(s):
    return (s["dram__bytes_read.sum"] + s["dram__bytes_write.sum"]) * scale


lib_fp = open(os.path.join(ROOT, "paper_2411_17483_b200", "lib", "libsofa.sha256")).read().strip()
res = {"config": cfg, "lib_fingerprint": lib_fp,
       "groups": {"sparse": b(step[0]) + b(step[3]), "dense": b(step[1])},
       "launches": [{"kernel": s["kernel"][:60], "dram_bytes": b(s),
                     "ncu_duration": f'{s["gpu__time_duration.sum"]:.0f} {units.get("time", "")}'} for s in step],
       "note": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum on the last bench step (cold cache, serialised)"}
json.dump(res, open(os.path.join(ROOT, "profiles", f"traffic_{cfg}.json"), "w"), indent=1)
print(json.dumps(res, indent=1))
