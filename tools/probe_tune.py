"""Replay step time: grouping (geometry x policy vs policy only) x point order (heuristic vs measured)."""
import os, sys, torch
sys.path.insert(0, ".")
from bench import make_traces
from paper_2602_03921_b200.sweep import DeviceSweep, c5_points
cfgs, trs = c5_points(make_traces(list(range(1, 49))))
ds = DeviceSweep(cfgs, trs)
ds.step(); torch.cuda.synchronize()
def t():
    ts = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ds.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(round(e0.elapsed_time(e1), 2))
    return ts
g = "policy" if os.environ.get("ESIM_GROUP_BY_POLICY") else "geometry x policy"
print(g, "heuristic order", t(), len(ds.batch.groups), "launches", flush=True)
d0 = [int(r.counters.digest) for r in ds.results()]
ds.tune_order()
print(g, "measured order", t(), flush=True)
print("digests equal", d0 == [int(r.counters.digest) for r in ds.results()])
