"""Per-point start/end SM clocks -> utilisation of warp slots over the replay launch."""
import sys, torch, numpy as np
sys.path.insert(0, ".")
from bench import make_traces
from paper_2602_03921_b200.sweep import DeviceSweep, c5_points
cfgs, trs = c5_points(make_traces(list(range(1, 49))))
ds = DeviceSweep(cfgs, trs)
ds.step(); torch.cuda.synchronize()
ds.tune_order(); ds.step(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); ds.replay(); e1.record(); torch.cuda.synchronize()
res = ds.results()
st = np.array([r.counters.pad[0] for r in res], np.int64)
en = np.array([r.counters.pad[1] for r in res], np.int64)
sm = np.array([r.counters.pad[2] for r in res])
dur = (en - st) / 1e6       # globaltimer ns -> ms
ms = e0.elapsed_time(e1)
print(f"replay {ms:.1f} ms, points {len(res)}, mean point {dur.mean():.1f} ms, max {dur.max():.1f} ms")
print("point-ms sum / (148 SM * 8 warps * kernel ms) =", dur.sum() / (148 * 8 * ms))
for m in ("olmoe", "mixtral", "qwen15moe", "phi35moe"):
    idx = [i for i, c in enumerate(cfgs) if c.model.name == m]
    print(m, f"mean {dur[idx].mean():.1f} max {dur[idx].max():.1f} ms", "accesses/point", np.mean([res[i].counters.totals[0] for i in idx]))
for ev in ("lru", "lfu", "ls"):
    idx = [i for i, c in enumerate(cfgs) if c.eviction == ev]
    print(ev, f"mean {dur[idx].mean():.1f} ms")
for cap in (0.01, 0.05, 0.25):
    idx = [i for i, c in enumerate(cfgs) if c.hardware.capacity_fraction == cap]
    print(cap, f"mean {dur[idx].mean():.1f} ms")
# concurrency timeline: running points per 1 ms bin
t0 = st.min()
T = int((en.max() - t0) / 1e6) + 1
run = np.zeros(T)
for a, b in zip((st - t0) / 1e6, (en - t0) / 1e6):
    run[int(a):int(b) + 1] += 1
print("running points per ms:", " ".join(str(int(x)) for x in run))
# per-SM busy: sum of durations per SM
busy = np.bincount(sm, weights=dur, minlength=148)
print("per-SM busy ms: min %.1f mean %.1f max %.1f" % (busy.min(), busy.mean(), busy.max()))
print("model cap bw -> mean ms")
for m in ("qwen15moe", "olmoe", "mixtral", "phi35moe"):
    row = []
    for cap in (0.01, 0.05, 0.25):
        for bw in (1e9, 5e9, 25e9):
            idx = [i for i, c in enumerate(cfgs) if c.model.name == m and c.hardware.capacity_fraction == cap
                   and c.hardware.bandwidth_bytes_per_sec == bw]
            row.append(f"{dur[idx].mean():5.1f}")
    print(m, " ".join(row))
import json
rows = []
for i, c in enumerate(cfgs):
    r = res[i].counters
    rows.append(dict(start_ms=float((st[i] - st.min()) / 1e6), sm=int(sm[i]), model=c.model.name, cap=c.hardware.capacity_fraction, bw=c.hardware.bandwidth_bytes_per_sec,
                     ev=c.eviction, seed=trs[i].seed if hasattr(trs[i], "seed") else 0, ms=float(dur[i]),
                     totals=[int(x) for x in r.totals], pf_pred=int(r.pf_pred_total), pf_dem=int(r.pf_dem_total),
                     n_recs=int(r.n_recs), ttft=int(r.ttft_us), total_us=int(r.total_us), passes=int(r.passes)))
import os
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open("gpurun_out/sched_points.json", "w"))
# per-group start times (launch order) and host enqueue time of one replay()
import time
torch.cuda.synchronize()
h0 = time.perf_counter(); ds.replay(); h1 = time.perf_counter(); torch.cuda.synchronize()
print(f"host enqueue of replay(): {(h1 - h0) * 1e3:.2f} ms for {len(ds.batch.groups)} groups")
res = ds.results()
st = np.array([r.counters.pad[0] for r in res], np.int64)
t0 = st.min()
for gi, g in enumerate(ds.batch.groups):
    idx = list(g)
    c = cfgs[idx[0]]
    print(f"group {gi}: {c.model.name:10s} {c.eviction:4s} n={len(g)} first start {(st[idx].min() - t0) / 1e6:.2f} ms, median start {(np.median(st[idx]) - t0) / 1e6:.2f} ms")
