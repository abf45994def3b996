"""Summarise the ncu launch list of `bench.py --steps K` (gpu__time_duration.sum):
the last K steps' launches (router x3 + replay x groups per step), their shares."""
import csv, sys, collections
path, steps, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui, ii, gi = (h.index(x) for x in ("Kernel Name", "Metric Value", "Metric Unit", "ID", "Grid Size"))
sc = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
launches = [(r[ki].split("(")[0], r[gi], float(r[vi].replace(",", "")) * sc[r[ui]]) for r in rows[hi + 1:]
            if len(r) > vi and "at::" not in r[ki]]
# the timed steps are the tail: each step starts with classify_kernel (the batched router)
starts = [i for i, l in enumerate(launches) if "classify" in l[0]]
tail = launches[starts[-steps]:]
agg = collections.defaultdict(lambda: [0, 0.0])
for k, g, t in tail:
    agg[k][0] += 1
    agg[k][1] += t
tot = sum(v[1] for v in agg.values())
with open(out, "w") as f:
    f.write(f"ncu --metrics gpu__time_duration.sum --clock-control none: python bench.py --steps {steps} --warmup 1 "
            f"--no-e2e --no-layer-step\n(last {steps} steps; cold-cache, serialised launches: the SHARES compare with "
            f"the bench's kernel_ms, the absolutes do not: the bench runs the replay groups concurrently)\n")
    f.write(f"{'kernel':48s} {'launches':>8s} {'total_us':>11s} {'mean_us':>10s} {'share':>7s}\n")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        f.write(f"{k[:48]:48s} {n:8d} {t:11.1f} {t / n:10.1f} {t / tot:7.1%}\n")
print(open(out).read())
