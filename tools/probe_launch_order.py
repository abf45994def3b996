"""Replay step time vs the order of the per-policy launches (after tune_order)."""
import itertools, sys, torch
sys.path.insert(0, ".")
from bench import make_traces
from paper_2602_03921_b200.sweep import DeviceSweep, c5_points
cfgs, trs = c5_points(make_traces(list(range(1, 49))))
ds = DeviceSweep(cfgs, trs)
ds.step(); torch.cuda.synchronize()
ds.tune_order(); ds.step(); torch.cuda.synchronize()
b = ds.batch
base_groups = list(b.groups)
name = {0: "lru", 1: "lfu", 5: "ls"}
for perm in itertools.permutations(range(len(base_groups))):
    b.groups = [base_groups[i] for i in perm]
    b.order = [i for g in b.groups for i in g]
    import ctypes as C
    from paper_2602_03921_b200 import _abi
    harr = (_abi.EsimConfig * len(b.ccfg))(*[b.ccfg[i] for i in b.order])
    b.h_cfg = harr
    b.d_cfg.copy_(torch.frombuffer(bytearray(harr), dtype=torch.uint8))
    if hasattr(b, "_streams"):
        del b._streams
    ts = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.launch(); e1.record(); torch.cuda.synchronize()
        ts.append(round(e0.elapsed_time(e1), 2))
    print([name.get(b.ccfg[g[0]].eviction, "?") for g in b.groups], ts, flush=True)
