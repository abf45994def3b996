"""One-off probe of the GPU box: host cores, CPU flags, pinned H2D / D2D bandwidth."""
import os, subprocess, json, time
import numpy as np
import torch
out = {}
out["nproc"] = os.cpu_count()
try:
    out["sched_affinity"] = len(os.sched_getaffinity(0))
except Exception:
    pass
lscpu = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
out["cpu_model"] = [l for l in lscpu.splitlines() if "Model name" in l]
out["avx512f"] = "avx512f" in lscpu
out["avx2"] = " avx2" in lscpu
out["numpy"] = np.__version__
dev = torch.device("cuda:0")
print(torch.cuda.get_device_name(0), flush=True)
for mb in (12.582912, 64, 256, 1024):
    n = int(mb * 1e6)
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
    s.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = max(3, int(2000 / mb))
    with torch.cuda.stream(s):
        e0.record()
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
        e1.record()
    s.synchronize()
    ms = e0.elapsed_time(e1)
    out[f"h2d_gbs_{mb}MB"] = n * reps / ms / 1e6
    with torch.cuda.stream(s):
        e0.record()
        for _ in range(reps):
            h.copy_(d, non_blocking=True)
        e1.record()
    s.synchronize()
    out[f"d2h_gbs_{mb}MB"] = n * reps / e0.elapsed_time(e1) / 1e6
# two streams concurrently
n = int(64e6)
hs = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
ds = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(2)]
ss = [torch.cuda.Stream() for _ in range(2)]
torch.cuda.synchronize()
t0 = time.perf_counter()
for r in range(20):
    for i in range(2):
        with torch.cuda.stream(ss[i]):
            ds[i].copy_(hs[i], non_blocking=True)
torch.cuda.synchronize()
out["h2d_2streams_gbs"] = 2 * 20 * n / (time.perf_counter() - t0) / 1e9
t0 = time.perf_counter()
big = torch.empty(int(12.9e9), dtype=torch.uint8, pin_memory=True)
out["pin_alloc_12.9GB_s"] = time.perf_counter() - t0
free, total = torch.cuda.mem_get_info()
out["gpu_mem_free_gb"] = free / 1e9
meminfo = open("/proc/meminfo").read().splitlines()[:3]
out["meminfo"] = meminfo
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
