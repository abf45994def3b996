"""Small workload for ncu: C5 grid x S seeds, warmup step then one profiled step."""
import sys
sys.path.insert(0, ".")
import torch
from bench import make_traces
from paper_2602_03921_b200.sweep import DeviceSweep, c5_points
S = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfgs, trs = c5_points(make_traces(list(range(1, S + 1))))
ds = DeviceSweep(cfgs, trs)
ds.step(); torch.cuda.synchronize()
ds.step(); torch.cuda.synchronize()
print("done", len(cfgs))
