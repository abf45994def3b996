import sys, torch
sys.path.insert(0, ".")
from bench import make_traces
from paper_2602_03921_b200.sweep import DeviceSweep, c5_points
cfgs, trs = c5_points(make_traces(list(range(1, 49))))
ds = DeviceSweep(cfgs, trs)
ds.route()
for wpc in (4, 3, 2, 1, 4):
    ds.batch.launch(warps_per_cta=wpc); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ds.batch.launch(warps_per_cta=wpc); e1.record(); torch.cuda.synchronize()
    res = ds.results()
    acc = sum(r.counters.totals[0] for r in res)
    print(f"wpc={wpc} replay_ms={e0.elapsed_time(e1):.1f} acc/s={acc/(e0.elapsed_time(e1)/1e3)/1e6:.1f}M", flush=True)
