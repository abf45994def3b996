import sys, torch
sys.path.insert(0, ".")
from bench import make_traces
from paper_2602_03921_b200.sweep import DeviceSweep, c5_points
cfgs, trs = c5_points(make_traces(list(range(1, 49))))
ds = DeviceSweep(cfgs, trs)
ds.step(); torch.cuda.synchronize()
ds.tune_order(); ds.step(); torch.cuda.synchronize()
for mode in ("concurrent", "serial", "concurrent"):
    ts = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if mode == "serial":
            ds.batch.launch(stream=torch.cuda.current_stream().cuda_stream)
        else:
            ds.batch.launch()
        e1.record(); torch.cuda.synchronize()
        ts.append(round(e0.elapsed_time(e1), 2))
    print(mode, ts, flush=True)
