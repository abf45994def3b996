"""Summarise an ncu --metrics gpu__time_duration.sum CSV into per-kernel shares."""
import csv, sys
path, out, title = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
agg = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    agg.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")) * scale[r[ui]])
tot = sum(sum(v) for v in agg.values())
with open(out, "w") as fh:
    fh.write(title + "\n")
    fh.write(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'mean_us':>10s} {'share':>7s}\n")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        fh.write(f"{k[:60]:60s} {len(v):8d} {sum(v):12.1f} {sum(v)/len(v):10.1f} {sum(v)/tot:7.1%}\n")
print(open(out).read())
