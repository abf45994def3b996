"""ncu workload: the C5 grid of ONE model (argv[1]) x S seeds (argv[2]); warm-up step, then one profiled step."""
import sys
sys.path.insert(0, ".")
import torch
from bench import make_traces
from paper_2602_03921_b200.sweep import DeviceSweep, c5_points
model, S = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 16
tr = {m: v for m, v in make_traces(list(range(1, S + 1))).items() if m == model}
cfgs, trs = c5_points(tr)
ds = DeviceSweep(cfgs, trs)
ds.step(); torch.cuda.synchronize()
ds.step(); torch.cuda.synchronize()
print("done", len(cfgs))
