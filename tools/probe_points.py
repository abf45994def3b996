"""Per-point replay times of the C5 x S step (globaltimer stamps the replay
kernel writes into EsimCounters.pad): max vs mean per launch group, the
slowest configurations, and the per-launch span -- the inputs to the replay
kernel's critical-path work. Usage: python tools/probe_points.py [seeds]"""
import collections
import ctypes as C
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from bench import make_traces
from paper_2602_03921_b200 import _abi
from paper_2602_03921_b200.sweep import DeviceSweep, c5_points

S = int(sys.argv[1]) if len(sys.argv) > 1 else 48
cfgs, trs = c5_points(make_traces(list(range(1, S + 1))))
ds = DeviceSweep(cfgs, trs)
for _ in range(3):
    ds.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ds.step()
e1.record()
torch.cuda.synchronize()
raw = ds.batch.counters.cpu().numpy().tobytes()
sz = C.sizeof(_abi.EsimCounters)
b = ds.batch
rows = []
for pos in range(len(b.ccfg)):
    c = _abi.EsimCounters.from_buffer_copy(raw[pos * sz:(pos + 1) * sz])
    i = b.order[pos]
    cfg = cfgs[i]
    rows.append(dict(pos=pos, ev=cfg.eviction, model=cfg.model.name, cap=cfg.hardware.capacity_fraction,
                     bw=cfg.hardware.bandwidth_bytes_per_sec / 1e9, t0=int(c.pad[0]), t1=int(c.pad[1]),
                     sm=int(c.pad[2]), dem=int(c.totals[0]), recs=int(c.n_recs)))
t00 = min(r["t0"] for r in rows)
out = {"seeds": S, "points": len(rows), "step_ms": e0.elapsed_time(e1)}
by = collections.defaultdict(list)
for r in rows:
    by[r["ev"]].append(r)
out["groups"] = {}
for ev, rs in by.items():
    d = np.array([(r["t1"] - r["t0"]) / 1e6 for r in rs])
    out["groups"][ev] = {"n": len(rs), "start_ms": (min(r["t0"] for r in rs) - t00) / 1e6,
                         "end_ms": (max(r["t1"] for r in rs) - t00) / 1e6, "point_ms_max": d.max(),
                         "point_ms_mean": d.mean(), "point_ms_p50": float(np.median(d))}
cfgk = collections.defaultdict(list)
for r in rows:
    cfgk[(r["ev"], r["model"], r["cap"], r["bw"])].append(((r["t1"] - r["t0"]) / 1e6, r["recs"], r["dem"]))
slow = sorted(((np.mean([x[0] for x in v]), k, np.mean([x[1] for x in v]), np.mean([x[2] for x in v]))
               for k, v in cfgk.items()), reverse=True)
out["slowest_configs"] = [{"cfg": list(k), "ms": m, "recs": rc, "demanded": dm, "ns_per_rec": m * 1e6 / rc}
                          for m, k, rc, dm in slow[:15]]
out["all_configs"] = [{"cfg": list(k), "ms": m, "recs": rc, "demanded": dm} for m, k, rc, dm in slow]
out["fastest_configs"] = [{"cfg": list(k), "ms": m, "recs": rc, "demanded": dm} for m, k, rc, dm in slow[-5:]]
# occupancy: points in flight over the step (per SM group of each policy launch)
t_end = max(r["t1"] for r in rows)
span = (t_end - t00) / 1e6
busy = sum((r["t1"] - r["t0"]) for r in rows) / 1e6
slots = len(set(r["sm"] for r in rows)) * 12
grid_t = np.linspace(0, span, 201)
act = [sum(1 for r in rows if (r["t0"] - t00) / 1e6 <= t < (r["t1"] - t00) / 1e6) for t in grid_t]
full = 0.9 * slots
tail_start = next((grid_t[i] for i in range(len(act)) if i > 10 and act[i] < full), span)
out["occupancy"] = {"span_ms": span, "warp_ms_busy": busy, "warp_slots": slots,
                    "utilisation": busy / (span * slots), "tail_from_ms": tail_start,
                    "active_points_at_pct": {str(p): act[int(p * 2)] for p in (10, 25, 50, 75, 90, 95, 99)}}
print(json.dumps(out, indent=1, default=float))
