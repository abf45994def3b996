"""One replay launch of a single (model, policy) group for ncu source-level capture.
usage: python tools/ncu_one.py MODEL POLICY SEEDS"""
import sys
sys.path.insert(0, ".")
import torch
from bench import make_traces
from paper_2602_03921_b200.sweep import DeviceSweep, c5_points
model, pol, S = sys.argv[1], sys.argv[2], int(sys.argv[3])
trs = make_traces(list(range(1, S + 1)))
cfgs, traces = c5_points({model: trs[model]})
keep = [i for i, c in enumerate(cfgs) if c.eviction == pol]
ds = DeviceSweep([cfgs[i] for i in keep], [traces[i] for i in keep])
ds.step(); torch.cuda.synchronize()
print("points", len(keep))
