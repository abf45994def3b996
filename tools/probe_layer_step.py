import sys, time, json
sys.path.insert(0, ".")
import torch
from paper_2602_03921_b200 import HardwareSpec, SimConfig, builtin_spec, generate_synthetic
from paper_2602_03921_b200.layer_step import LayerStepEngine
spec = builtin_spec("olmoe")
out = {}
tr = generate_synthetic(spec, seed=1, prefill_tokens=64, decode_tokens=64)
g = torch.Generator().manual_seed(0)
x0 = torch.randn(64, 2048, generator=g).to(torch.bfloat16).pin_memory()
xd = torch.randn(64, 2048, generator=g).to(torch.bfloat16).pin_memory()
t0 = time.time()
cfg = SimConfig(model=spec, hardware=HardwareSpec(capacity_bytes=614_400_000), working_precision="fp16",
                eviction="ls", prefetch="score", percentile=80.0, miss="fetch")
eng = LayerStepEngine(cfg, 2048, 1024, max_tokens=64)
out["create_s"] = time.time() - t0
t0 = time.time(); eng.init_weights(seed=0); out["init_s"] = time.time() - t0
for ev in ("ls", "lru"):
    eng.cfg = SimConfig(model=spec, hardware=HardwareSpec(capacity_bytes=614_400_000), working_precision="fp16",
                        eviction=ev, prefetch="score", percentile=80.0, miss="fetch")
    for rep in range(2):
        r = eng.run(tr, x0, xd)
    d = {k: getattr(r, k) for k in ("ttft_ms", "total_ms", "decode_tokens_per_sec", "h2d_gbs", "n_copies",
                                    "n_demand_copies", "n_prefetch_copies", "n_cancelled", "n_ffn_batches",
                                    "host_enqueue_ms")}
    d["hit_rate"] = r.report["rates"]["hit_rate"]
    d["logical_ttft_us"] = r.report["timing"]["ttft_us"]
    out[ev] = d
    print(ev, d, flush=True)
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/probe_layer_step.json", "w"), indent=1)
