"""Time the batched router (C5 x S seeds) and the replay with CUDA events."""
import sys
sys.path.insert(0, ".")
import torch
from bench import make_traces
from paper_2602_03921_b200.sweep import DeviceSweep, c5_points
S = int(sys.argv[1]) if len(sys.argv) > 1 else 48
cfgs, trs = c5_points(make_traces(list(range(1, S + 1))))
ds = DeviceSweep(cfgs, trs)
ds.step(); torch.cuda.synchronize()
ds.tune_order(); ds.step(); torch.cuda.synchronize()
for name, fn in (("route", ds.route), ("replay", ds.replay)):
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(name, "ms", [round(t, 3) for t in ts], flush=True)
