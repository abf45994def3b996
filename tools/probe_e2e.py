"""e2e (C-ABI sweep plan, host buffers) step-time distribution: synchronous
runs vs the pipelined submit/wait path, against the device-resident step."""
import sys, time, json, statistics
sys.path.insert(0, ".")
import torch
from bench import make_traces
from paper_2602_03921_b200.sweep import HostGrid, DeviceSweep, c5_points, pin_traces
S = int(sys.argv[1]) if len(sys.argv) > 1 else 48
cfgs, trs = c5_points(make_traces(list(range(1, S + 1))))
pin_traces(trs)
g = HostGrid(cfgs, trs)
for _ in range(3):
    g.run()
sync = []
for _ in range(10):
    t = time.perf_counter(); g.run(); sync.append(1e3 * (time.perf_counter() - t))
g.submit(); g.submit(); g.wait(); g.wait()
pipe = []
t0 = time.perf_counter()
g.submit()
for _ in range(20):
    g.submit(); g.wait(); pipe.append(time.perf_counter())
g.wait()
steps = [1e3 * (b - a) for a, b in zip([t0] + pipe[:-1], pipe)]
ds = DeviceSweep(cfgs, trs)
for _ in range(3):
    ds.step()
torch.cuda.synchronize()
dev = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ds.step(); e1.record(); torch.cuda.synchronize(); dev.append(e0.elapsed_time(e1))
print(json.dumps({"sync_ms": sync, "pipelined_step_ms": steps, "device_step_ms": dev,
                  "median": {"sync": statistics.median(sync), "pipelined": statistics.median(steps[2:]),
                             "device": statistics.median(dev)}}, indent=1))
