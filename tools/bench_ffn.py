"""FFN kernel microbenchmark (enqueue-ahead, per-iteration CUDA events, L2 flushed between
iterations): a prefill-64 layer (28 experts, ~18 tokens each), decode (8 experts x 1 token),
all 64 experts. Algorithmic bytes = 12,582,912 B weights per executed expert."""
import sys, json
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2602_03921_b200.ffn import ExpertSlots, npad_for, routing_tables
H, I = 2048, 1024
out = {}
slots = ExpertSlots(64, H, I, max_tokens=1024, max_exec=64)
slots.buf.copy_((torch.randn(slots.buf.numel(), device="cuda") * 0.02).to(torch.bfloat16))
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6650.0
for name, T, K, n_exp in (("prefill64", 64, 8, 28), ("decode", 1, 8, 8), ("prefill64_all64", 64, 8, 64),
                          ("prefill1024_128tok_all64", 1024, 8, 64)):
    rng = np.random.default_rng(0)
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    if T * K == 128 * n_exp:       # every expert exactly 128 tokens (the largest tile, N = 128)
        row_sel = (np.arange(T * K) % n_exp).reshape(T, K).astype(np.int32)
    else:
        row_sel = np.stack([rng.choice(n_exp, size=K, replace=False) for _ in range(T)]).astype(np.int32)
    row_w = rng.uniform(0.01, 0.3, size=(T, K)).astype(np.float32)
    mt = int(np.bincount(row_sel.ravel()).max())
    npad = npad_for(mt)
    ti, tw = routing_tables(row_sel, row_w, {e: (e, e) for e in range(n_exp)}, npad)
    ti, tw = torch.from_numpy(ti).cuda(), torch.from_numpy(tw).cuda()
    es = torch.arange(n_exp, dtype=torch.int32, device="cuda")
    for impl in (("tc", "gemv") if mt <= 4 else ("tc",)):
        for _ in range(3):
            slots.run_layer(x, es, ti, tw, npad, residual=False, max_tok=mt, decode=impl)
        torch.cuda.synchronize()
        n = 30
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for i in range(n):
            flush.zero_()
            ev[i][0].record()
            slots.run_layer(x, es, ti, tw, npad, residual=False, max_tok=mt, decode=impl)
            ev[i][1].record()
        torch.cuda.synchronize()
        ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
        byt = n_exp * 3 * H * I * 2
        flops = 2 * 3 * H * I * int(row_sel.size)
        key = name if impl == "tc" else name + "_gemv"
        out[key] = {"ms": ms, "npad": npad, "n_exec": n_exp, "weight_gbs": byt / ms / 1e6,
                    "frac_of_hbm_peak": byt / ms / 1e6 / peak, "tflops": flops / ms / 1e9}
        print(key, out[key], flush=True)
# decode over quantised slots (ffn_decode_q_kernel, dequantisation fused into the
# A operand): algorithmic bytes = codes + fp32 row scales per executed expert
for bits in (8, 4, 2):
    nq, ns = 3 * H * I, 2 * I + H
    per = nq * bits // 8 + 4 * ns
    sb = (per + 255) // 256 * 256
    qbuf = torch.randint(0, 256, (64 * sb,), device="cuda", dtype=torch.int32).to(torch.uint8)
    qv = qbuf.view(64, sb)
    qv[:, nq * bits // 8:per] = torch.full((64, ns), 0.01, device="cuda").view(torch.uint8).view(64, ns * 4)
    for n_exp in (8, 64):
        rng = np.random.default_rng(0)
        row_sel = rng.choice(n_exp, size=8, replace=False).astype(np.int32).reshape(1, 8) if n_exp >= 8 else None
        T = 1 if n_exp == 8 else 8
        if n_exp == 64:
            row_sel = np.arange(64, dtype=np.int32).reshape(8, 8)
        row_w = rng.uniform(0.01, 0.3, size=row_sel.shape).astype(np.float32)
        ti, tw = routing_tables(row_sel, row_w, {e: (e, e) for e in range(n_exp)}, 16)
        ti, tw = torch.from_numpy(ti).cuda(), torch.from_numpy(tw).cuda()
        x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
        es = torch.arange(n_exp, dtype=torch.int32, device="cuda")
        for impl in ("tc", "gemv"):
            for _ in range(3):
                slots.run_layer_quant(qbuf, sb, bits, x, es, ti, tw, decode=impl, max_tok=1)
            torch.cuda.synchronize()
            n = 30
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
            for i in range(n):
                flush.zero_()
                ev[i][0].record()
                slots.run_layer_quant(qbuf, sb, bits, x, es, ti, tw, decode=impl, max_tok=1)
                ev[i][1].record()
            torch.cuda.synchronize()
            ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
            byt = n_exp * per
            name = f"decode_int{bits}_{n_exp}experts" + ("_gemv" if impl == "gemv" else "")
            out[name] = {"ms": ms, "n_exec": n_exp, "quant_bytes_per_expert": per, "quant_gbs": byt / ms / 1e6,
                         "frac_of_hbm_peak": byt / ms / 1e6 / peak,
                         "bf16_equivalent_gbs": n_exp * 3 * H * I * 2 / ms / 1e6}
            print(name, out[name], flush=True)
json.dump(out, open("gpurun_out/bench_ffn.json", "w"), indent=1)
