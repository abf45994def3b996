"""Physical layer step on other BASELINE configs (bf16 random-init experts in a
pinned tile-major store, HBM slots, copy engine + tcgen05 FFN), e.g. configs[3]:
Qwen1.5-MoE-A2.7B shape (24 x 60, top-4, H=2048, I=1408 -> 17,301,504 B/expert)
at 5 % capacity with expert substitution. Decisions are checked against the C
oracle (test infrastructure) for the same config; TTFT / decode tok/s / host
link measured with CUDA events.
usage: python tools/layer_step_models.py [model] [miss] [capacity_fraction or bytes,...] [policies] [decode_tokens] [fp16|int8|int4|int2]
Mixtral (configs[2]): 32 x 8 top-2, H=4096, I=14336, 352,321,536 B/expert -> a 90 GB pinned store."""
import json, sys, time
sys.path.insert(0, ".")
import torch
from paper_2602_03921_b200 import HardwareSpec, SimConfig, builtin_spec, generate_synthetic
from paper_2602_03921_b200.layer_step import LayerStepEngine
from oracle import oracle

model = sys.argv[1] if len(sys.argv) > 1 else "qwen15moe"
miss = sys.argv[2] if len(sys.argv) > 2 else "subst"
fracs = [float(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "0.05").split(",")]
pols = (sys.argv[4] if len(sys.argv) > 4 else "ls,lru").split(",")
n_dec = int(sys.argv[5]) if len(sys.argv) > 5 else 64
prec = sys.argv[6] if len(sys.argv) > 6 else "fp16"          # fp16 (bf16 store) or int8
H, I = {"qwen15moe": (2048, 1408), "olmoe": (2048, 1024), "mixtral": (4096, 14336)}[model]
spec = builtin_spec(model)
tr = generate_synthetic(spec, seed=1, prefill_tokens=64, decode_tokens=n_dec)
g = torch.Generator().manual_seed(0)
x0 = torch.randn(64, H, generator=g).to(torch.bfloat16).pin_memory()
xd = torch.randn(n_dec, H, generator=g).to(torch.bfloat16).pin_memory()
out = {"model": model, "H": H, "I": I, "expert_bytes_bf16": 3 * H * I * 2, "miss": miss,
       "trace": f"64 prefill + {n_dec} decode tokens, seed 1"}
eng = None
t0 = time.time()
runs = 2 if model != "mixtral" else 1
for frac in fracs:
  for ev in pols:
    hw = HardwareSpec(capacity_bytes=int(frac)) if frac > 1 else HardwareSpec(capacity_fraction=frac)
    cfg = SimConfig(model=spec, hardware=hw, working_precision=prec,
                    eviction=ev, prefetch="score", percentile=80.0, miss=miss, subst_tolerance=0.05)
    if eng is None:
        # slots for the largest capacity; smaller ones use a prefix (the decisions bound the live slots)
        bf = max(fracs)
        big = SimConfig(model=spec, hardware=HardwareSpec(capacity_bytes=int(bf)) if bf > 1 else
                        HardwareSpec(capacity_fraction=bf), working_precision=prec,
                        eviction=ev, prefetch="score", percentile=80.0, miss=miss)
        eng = LayerStepEngine(big, H, I, max_tokens=64)
        eng.init_weights(seed=0)
        out["n_slots_allocated"] = eng.n_slots
        out["store_gb"] = eng.store_bytes.numel() / 1e9
        out["store_precisions"] = list(eng.precisions)
        out["init_s"] = time.time() - t0
    eng.cfg = cfg
    best = None
    for _ in range(runs):
        r = eng.run(tr, x0, xd)
        best = r if best is None or r.total_ms < best.total_ms else best
    ref = oracle.run(cfg, tr, full_log=False).report
    out[f"{ev}@{frac}"] = {"n_slots": cfg.capacity_bytes() // spec.expert_bytes(prec), "precision": prec,
               "copy_bytes": eng.expert_bytes, "ttft_ms": best.ttft_ms, "decode_tok_s": best.decode_tokens_per_sec, "total_ms": best.total_ms,
               "host_link_gbs": best.h2d_gbs, "h2d_gb": best.h2d_bytes / 1e9, "copies": best.n_copies, "ffn_batches": best.n_ffn_batches,
               "logical_hit_rate": best.report["rates"]["hit_rate"],
               "substituted": best.report["totals"].get("substituted"),
               "decisions_match_oracle": json.dumps(ref) == json.dumps(best.report)}
    print(ev, frac, out[f"{ev}@{frac}"], flush=True)
eng.close()
json.dump(out, open(f"gpurun_out/layer_step_{model}_{miss}_{prec}.json", "w"), indent=1)
print(json.dumps(out))
