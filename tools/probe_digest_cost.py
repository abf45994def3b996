import sys, torch
sys.path.insert(0, ".")
from bench import make_traces
from paper_2602_03921_b200.sweep import DeviceSweep, c5_points
cfgs, trs = c5_points(make_traces(list(range(1, 49))))
for dg in (True, False):
    ds = DeviceSweep(cfgs, trs, digest=dg)
    ds.step(); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ds.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print("digest", dg, [round(t, 1) for t in ts], flush=True)
