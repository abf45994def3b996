"""Per-unit timeline of one FFN launch (globaltimer stamps) for the decode and prefill-64 cases."""
import sys, json, ctypes as C
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2602_03921_b200.ffn import ExpertSlots, npad_for, routing_tables
from paper_2602_03921_b200._device import lib
H, I = 2048, 1024
slots = ExpertSlots(64, H, I, max_tokens=64, max_exec=64)
slots.buf.copy_((torch.randn(slots.buf.numel(), device="cuda") * 0.02).to(torch.bfloat16))
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
tr = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")
lib().esim_ffn_set_trace.argtypes = [C.c_void_p]
for name, T, K, n_exp in (("prefill64", 64, 8, 28),):
    rng = np.random.default_rng(0)
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    row_sel = np.stack([rng.choice(n_exp, size=K, replace=False) for _ in range(T)]).astype(np.int32)
    row_w = rng.uniform(0.01, 0.3, size=(T, K)).astype(np.float32)
    npad = npad_for(int(np.bincount(row_sel.ravel()).max()))
    ti, tw = routing_tables(row_sel, row_w, {e: (e, e) for e in range(n_exp)}, npad)
    ti, tw = torch.from_numpy(ti).cuda(), torch.from_numpy(tw).cuda()
    es = torch.arange(n_exp, dtype=torch.int32, device="cuda")
    for _ in range(3):
        slots.run_layer(x, es, ti, tw, npad, residual=False)
    flush.zero_(); torch.cuda.synchronize()
    tr.zero_()
    lib().esim_ffn_set_trace(tr.data_ptr())
    slots.run_layer(x, es, ti, tw, npad, residual=False)
    torch.cuda.synchronize()
    lib().esim_ffn_set_trace(None)
    a = tr.view(-1, 8).cpu().numpy()
    n1 = n_exp * (I // 64)
    used = a[:, 0] > 0
    a = a[used]
    t0 = a[:, 0].min()
    rel = (a[:, :4] - t0) / 1000.0
    print(f"== {name}: units {len(a)} (gemm1 {n1}), span {(a[:, 3].max() - t0) / 1000:.1f} us")
    g1, g2 = rel[:n1], rel[n1:]
    for lab, r in (("gemm1", g1), ("gemm2", g2)):
        if len(r):
            print(f"  {lab}: mma start [{r[:,0].min():.1f},{r[:,0].max():.1f}] "
                  f"acc ready [{r[:,2].min():.1f},{r[:,2].max():.1f}] epi end [{r[:,3].min():.1f},{r[:,3].max():.1f}] "
                  f"mean: mma {np.mean(r[:,2]-r[:,0]):.2f} epi {np.mean(r[:,3]-r[:,2]):.2f} us")
    np.save(f"gpurun_out/ffn_timeline_{name}.npy", a)
