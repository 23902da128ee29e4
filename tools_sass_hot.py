import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = sum(float(r[si] or 0) for r in data)
print("total samples", tot)
agg = {}
for r in data:
    for i in stall_cols:
        agg[h[i]] = agg.get(h[i], 0) + float(r[i] or 0)
print(sorted(agg.items(), key=lambda x: -x[1])[:8])
top = sorted(range(len(data)), key=lambda i: -float(data[i][si] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for i in sorted(top):
    r = data[i]
    st = sorted(((float(r[c] or 0), h[c]) for c in stall_cols), reverse=True)[:2]
    print(f"{i:5d} {r[0]:>6} {float(r[si])/tot*100:5.1f}%  {r[1][:60]:60s} {st}")
