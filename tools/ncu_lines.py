"""Summarise an ncu --set full report: per-source-line warp-stall samples (needs -lineinfo) and key
raw metrics.  Usage: python tools/ncu_lines.py report.ncu-rep [kernel-regex] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else "k_query"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25


def run(args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv", "-k", f"regex:{kern}"]))))
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
if len(raw) > 2:
    h, u = raw[0], raw[1]
    for row in raw[2:]:
        print("--", row[h.index("Kernel Name")][:80])
        for n in want:
            if n in h:
                print(f"   {n:60s} {row[h.index(n)]:>16s} {u[h.index(n)]}")
rows = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source=cuda,sass", "-k",
                                        f"regex:{kern}"]))))
cur_file = cur_line = cur_src = None
agg = {}
stall_cols = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        stall_cols = [i for i, n in enumerate(hdr) if n.startswith("stall_") and "Not Issued" not in n]
        continue
    if len(r) < 5:
        continue
    if r[0].isdigit():
        cur_line, cur_src = int(r[0]), r[1]
        continue
    if r[0] == "" and r[2].startswith("0x"):
        try:
            smp = float(r[4] or 0)
        except ValueError:
            continue
        a = agg.setdefault((cur_file, cur_line), [0.0, cur_src, {}])
        a[0] += smp
        for i in stall_cols or []:
            a[2][hdr[i]] = a[2].get(hdr[i], 0) + float(r[i] or 0)
tot = sum(v[0] for v in agg.values()) or 1
print(f"-- warp-stall samples by source line (total {tot:.0f})")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    st = sorted(v[2].items(), key=lambda x: -x[1])[:2]
    st = ", ".join(f"{n[6:]} {c / max(v[0], 1) * 100:.0f}%" for n, c in st)
    print(f"{v[0] / tot * 100:5.1f}%  {k[0]}:{k[1]:<5} {v[1].strip()[:90]:90s} [{st}]")
