"""Decode GEMV ring-size variants (standalone builds of csrc/ffn_gemv.cu with
-DGEMV_STAGES / -DGEMV_CHUNK, loaded with ctypes): CUDA-event time of one
decode layer (8 and 64 experts x 1 token, bf16 / int4 / int2 slots),
L2 cleaned by a read pass between iterations. Usage: probe_gemv_variants.py lib.so..."""
import sys, json, ctypes as C
sys.path.insert(0, ".")
import numpy as np, torch
H, I = 2048, 1024
nq, ns = 3 * H * I, 2 * I + H
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
bufs = {}
for bits in (16, 4, 2):
    per = nq * 2 if bits == 16 else nq * bits // 8 + 4 * ns
    sb = (per + 255) // 256 * 256
    q = torch.randint(0, 256, (64 * sb,), device="cuda", dtype=torch.int32).to(torch.uint8)
    if bits == 16:
        q.view(torch.bfloat16).copy_((torch.randn(64 * sb // 2, device="cuda") * 0.02).to(torch.bfloat16))
    else:
        q.view(64, sb)[:, nq * bits // 8:per] = torch.full((64, ns), 0.01, device="cuda").view(torch.uint8).view(64, ns * 4)
    bufs[bits] = (q, sb, per)
x = torch.randn(8, H, device="cuda").to(torch.bfloat16)
out = {}
for path in sys.argv[1:]:
    L = C.CDLL(path)
    vp, i32 = C.c_void_p, C.c_int32
    L.esim_ffn_experts_gemv.argtypes = [vp, C.c_int64, i32, vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, vp]
    res = {}
    for bits in (16, 4, 2):
        q, sb, per = bufs[bits]
        for n_exp in (8, 64):
            ti = torch.full((n_exp, 16), -1, dtype=torch.int32, device="cuda")
            ti[:, 0] = torch.arange(n_exp, device="cuda", dtype=torch.int32) % 8
            tw = torch.full((n_exp, 16), 0.1, dtype=torch.float32, device="cuda")
            es = torch.arange(n_exp, dtype=torch.int32, device="cuda")
            y = torch.zeros(8 * H, device="cuda")
            call = lambda: L.esim_ffn_experts_gemv(q.data_ptr(), sb, bits, x.data_ptr(), es.data_ptr(), ti.data_ptr(),
                                                   tw.data_ptr(), y.data_ptr(), n_exp, 16, 1, I, H, None)
            for _ in range(3):
                assert call() == 0
            torch.cuda.synchronize()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
            for i in range(20):
                flush.view(torch.int64).sum()
                ev[i][0].record()
                call()
                ev[i][1].record()
            torch.cuda.synchronize()
            us = float(np.median([a.elapsed_time(b) for a, b in ev])) * 1000
            a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.view(torch.int64).sum()
            a0.record()
            for i in range(20):
                call()
            b0.record()
            torch.cuda.synchronize()
            b2b = a0.elapsed_time(b0) * 1000 / 20
            res[f"b{bits}_e{n_exp}"] = {"us": round(us, 2), "gbs": round(n_exp * per / us / 1e3, 1),
                                        "back_to_back_us": round(b2b, 2)}
    out[path] = res
    print(path, res, flush=True)
json.dump(out, open("gpurun_out/probe_gemv_variants.json", "w"), indent=1)
