"""Replay step time vs warps per CTA (occupancy granularity), after tune_order."""
import sys, torch
sys.path.insert(0, ".")
from bench import make_traces
from paper_2602_03921_b200.sweep import DeviceSweep, c5_points
cfgs, trs = c5_points(make_traces(list(range(1, 49))))
ds = DeviceSweep(cfgs, trs)
ds.step(); torch.cuda.synchronize()
ds.tune_order(); ds.step(); torch.cuda.synchronize()
d0 = [int(r.counters.digest) for r in ds.results()]
for w in (4, 1, 2, 3, 4):
    ts = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ds.batch.launch(warps_per_cta=w); e1.record(); torch.cuda.synchronize()
        ts.append(round(e0.elapsed_time(e1), 2))
    ok = [int(r.counters.digest) for r in ds.results()] == d0
    print("warps/CTA", w, ts, "digests ok" if ok else "DIGEST MISMATCH", flush=True)
