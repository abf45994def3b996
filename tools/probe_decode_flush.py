"""Decode FFN timing under different L2 preparations (int4 / bf16, 8 experts x 1 token):
memset flush (dirty L2), read flush (clean L2), no flush with rotating expert sets,
and back-to-back launches. Separates the kernels' own time from L2 write-back."""
import sys, json
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2602_03921_b200.ffn import ExpertSlots, routing_tables
H, I = 2048, 1024
slots = ExpertSlots(64, H, I, max_tokens=8, max_exec=64)
slots.buf.copy_((torch.randn(slots.buf.numel(), device="cuda") * 0.02).to(torch.bfloat16))
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
nq, ns = 3 * H * I, 2 * I + H
bits = 4
per = nq * bits // 8 + 4 * ns
sb = (per + 255) // 256 * 256
qbuf = torch.randint(0, 256, (64 * sb,), device="cuda", dtype=torch.int32).to(torch.uint8)
qbuf.view(64, sb)[:, nq * bits // 8:per] = torch.full((64, ns), 0.01, device="cuda").view(torch.uint8).view(64, ns * 4)
row_sel = np.arange(8, dtype=np.int32).reshape(1, 8)
ti, tw = routing_tables(row_sel, np.full((1, 8), 0.1, np.float32), {e: (e, e) for e in range(8)}, 16)
ti, tw = torch.from_numpy(ti).cuda(), torch.from_numpy(tw).cuda()
x = torch.randn(1, H, device="cuda").to(torch.bfloat16)
sets = [torch.arange(8 * s, 8 * s + 8, dtype=torch.int32, device="cuda") for s in range(8)]
def run(kind, impl, es):
    if kind == "q4":
        slots.run_layer_quant(qbuf, sb, 4, x, es, ti, tw, decode=impl, max_tok=1)
    else:
        slots.run_layer(x, es, ti, tw, 16, residual=False, max_tok=1, decode=impl)
out = {}
for kind in ("q4", "bf16"):
    for impl in ("tc", "gemv"):
        for _ in range(3):
            run(kind, impl, sets[0])
        res = {}
        for prep in ("memset", "read", "none_rotate"):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(24)]
            for i in range(24):
                if prep == "memset":
                    flush.zero_()
                elif prep == "read":
                    flush.view(torch.int64).sum()
                ev[i][0].record()
                run(kind, impl, sets[i % 8])
                ev[i][1].record()
            torch.cuda.synchronize()
            res[prep] = float(np.median([a.elapsed_time(b) for a, b in ev])) * 1000
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.view(torch.int64).sum()
        a.record()
        for i in range(40):
            run(kind, impl, sets[i % 8])
        b.record()
        torch.cuda.synchronize()
        res["back_to_back_avg"] = a.elapsed_time(b) * 1000 / 40
        out[f"{kind}_{impl}_us"] = res
        print(kind, impl, res, flush=True)
json.dump(out, open("gpurun_out/probe_decode_flush.json", "w"), indent=1)
