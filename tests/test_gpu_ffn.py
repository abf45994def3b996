"""tcgen05 grouped SwiGLU expert FFN vs a plain PyTorch fp32 reference of the
same op (same bf16 weights/activations; the kernel keeps the intermediate
activation in bf16, so the reference rounds it too). Tolerance: max error
<= 1e-2 of max |y| (BASELINE.json north star: bf16 tolerance 1e-2)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

H, I = 2048, 1024
TOL = 1e-2


def _case(T, K, n_exp, npad_expected, seed, fused, H=H, I=I, decode="tc"):
    import torch
    from paper_2602_03921_b200.ffn import ExpertSlots, expert_matrices, npad_for, routing_tables
    g = torch.Generator(device="cuda").manual_seed(seed)
    n_slots = n_exp + 2
    slots = ExpertSlots(n_slots, H, I, max_tokens=T, max_exec=n_exp)
    slots.buf.copy_((torch.randn(slots.buf.numel(), generator=g, device="cuda") * 0.02).to(torch.bfloat16))
    x = torch.randn(T, H, generator=g, device="cuda").to(torch.bfloat16)
    rng = np.random.default_rng(seed)
    row_sel = np.stack([rng.choice(n_exp, size=K, replace=False) for _ in range(T)]).astype(np.int32)
    row_w = rng.uniform(0.01, 0.3, size=(T, K)).astype(np.float32)
    slot_of = rng.permutation(n_slots)[:n_exp]
    executed = {e: (e, e) for e in range(n_exp)}
    counts = np.bincount(row_sel.ravel(), minlength=n_exp)
    npad = npad_for(int(counts.max()))
    assert npad == npad_expected
    ti, tw = routing_tables(row_sel, row_w, executed, npad)
    exec_slot = torch.tensor(slot_of, dtype=torch.int32, device="cuda")
    slots.y.zero_()
    mt = int(counts.max()) if fused else None          # <= 4 tokens: fused decode kernel
    slots.run_layer(x, exec_slot, torch.from_numpy(ti).cuda(), torch.from_numpy(tw).cuda(), npad, residual=False,
                    max_tok=mt, decode=decode)
    torch.cuda.synchronize()
    y = slots.y[:T * H].view(T, H).float()
    ref = torch.zeros(T, H, device="cuda")
    xf = x.float()
    for e in range(n_exp):
        w = slots.slot_view(int(slot_of[e])).float()
        w1, wd = expert_matrices(w, H, I)
        gate, up = xf @ w1[:I].T, xf @ w1[I:].T
        act = (torch.nn.functional.silu(gate) * up).to(torch.bfloat16).float()
        out = act @ wd.T
        for t in range(T):
            for j in range(K):
                if row_sel[t, j] == e:
                    ref[t] += float(row_w[t, j]) * out[t]
    err = (y - ref).abs().max().item() / ref.abs().max().item()
    assert err <= TOL, f"max rel err {err:.3e}"
    # residual path: x += y
    x2 = x.clone()
    slots.run_layer(x2, exec_slot, torch.from_numpy(ti).cuda(), torch.from_numpy(tw).cuda(), npad, max_tok=mt,
                    decode=decode)
    torch.cuda.synchronize()
    assert torch.isfinite(x2.float()).all()
    return err


@pytest.mark.parametrize("T,K,n_exp,npad,seed", [(1, 8, 8, 16, 0), (16, 2, 8, 16, 1), (64, 8, 28, 32, 2),
                                                  (64, 8, 8, 64, 3), (128, 4, 8, 128, 4)])
def test_ffn_matches_torch_fp32(T, K, n_exp, npad, seed):
    """The two-phase kernel (gemm1 tiles -> split-K gemm2 units)."""
    _case(T, K, n_exp, npad, seed, fused=False)


@pytest.mark.parametrize("decode", ["tc", "gemv"])
@pytest.mark.parametrize("T,K,n_exp,seed", [(1, 8, 8, 10), (1, 8, 64, 11), (3, 4, 8, 12), (4, 2, 3, 13),
                                            (2, 8, 8, 14)])
def test_ffn_decode_kernel_matches_torch_fp32(T, K, n_exp, seed, decode):
    """Decode layers (<= 4 tokens per expert): the fused per-slice tcgen05
    kernel ("tc") and the streaming GEMV over the slots ("gemv")."""
    _case(T, K, n_exp, 16, seed, fused=True, decode=decode)


# BASELINE.json configs[2]: Mixtral-8x7B experts, H=4096, I=14336 (352 MB bf16
# per expert). Decode takes ffn_fused_kernel<16> (H/BM = 32 > 16 rows of
# output tiles per unit: the split-K n_kc = 4 path, ffn_gemm.cu), prefill the
# persistent two-phase kernel; top-2 of 8 experts.
@pytest.mark.parametrize("T,K,n_exp,npad,seed,fused", [(1, 2, 2, 16, 30, True), (2, 2, 4, 16, 31, True),
                                                       (64, 2, 8, 32, 32, False), (16, 2, 8, 16, 33, False)])
def test_ffn_mixtral_shape_matches_torch_fp32(T, K, n_exp, npad, seed, fused):
    _case(T, K, n_exp, npad, seed, fused=fused, H=4096, I=14336)


@pytest.mark.parametrize("T,K,n_exp,seed,H_,I_", [(1, 2, 2, 34, 4096, 14336), (2, 2, 4, 35, 4096, 14336),
                                                  (1, 4, 4, 44, 2048, 1408), (1, 1, 1, 45, 2048, 5632)])
def test_ffn_gemv_decode_other_shapes(T, K, n_exp, seed, H_, I_):
    """The GEMV decode kernel at the Mixtral (configs[2]) and Qwen (configs[3])
    expert shapes."""
    _case(T, K, n_exp, 16, seed, fused=True, H=H_, I=I_, decode="gemv")


# configs[3]: Qwen1.5-MoE routed experts (I = 1408) and its shared expert (I = 5632)
@pytest.mark.parametrize("T,K,n_exp,npad,seed,fused,inter", [(1, 4, 4, 16, 40, True, 1408), (64, 4, 24, 32, 41, False, 1408),
                                                             (1, 1, 1, 16, 42, True, 5632), (64, 1, 1, 64, 43, False, 5632)])
def test_ffn_qwen_shapes_match_torch_fp32(T, K, n_exp, npad, seed, fused, inter):
    _case(T, K, n_exp, npad, seed, fused=fused, H=2048, I=inter)


@pytest.mark.parametrize("decode", ["tc", "gemv"])
@pytest.mark.parametrize("bits,T,K,n_exp,seed", [(8, 1, 8, 8, 20), (4, 1, 8, 64, 21), (2, 3, 4, 16, 22),
                                                 (4, 4, 8, 40, 23), (2, 1, 8, 8, 24), (8, 2, 8, 8, 25)])
def test_ffn_quantised_decode_kernel_matches_torch_fp32(bits, T, K, n_exp, seed, decode):
    """ffn_decode_q_kernel: quantised slots (codes + fp32 row scales), the
    dequantisation fused into the A operand; 64 experts x 16 units puts
    several units on every CTA (ring phases wrap across units)."""
    import torch
    from paper_2602_03921_b200.ffn import ExpertSlots, routing_tables
    from paper_2602_03921_b200.layer_step import dequant_expert
    g = torch.Generator(device="cuda").manual_seed(seed)
    n_slots = n_exp + 3
    nq, ns = 3 * H * I, 2 * I + H
    per = nq * bits // 8 + 4 * ns
    slot_bytes = (per + 255) // 256 * 256
    q = torch.zeros(n_slots, slot_bytes, dtype=torch.uint8, device="cuda")
    q[:, :nq * bits // 8] = torch.randint(0, 256, (n_slots, nq * bits // 8), generator=g, device="cuda",
                                          dtype=torch.int32).to(torch.uint8)
    qmax = {8: 127, 4: 7, 2: 1}[bits]
    sc = (0.5 + torch.rand(n_slots, ns, generator=g, device="cuda")) * (0.02 / qmax)
    q[:, nq * bits // 8:per] = sc.view(torch.uint8).view(n_slots, ns * 4)
    slots = ExpertSlots(1, H, I, max_tokens=T, max_exec=n_exp)
    x = torch.randn(T, H, generator=g, device="cuda").to(torch.bfloat16)
    rng = np.random.default_rng(seed)
    row_sel = np.stack([rng.choice(n_exp, size=K, replace=False) for _ in range(T)]).astype(np.int32)
    row_w = rng.uniform(0.01, 0.3, size=(T, K)).astype(np.float32)
    slot_of = rng.permutation(n_slots)[:n_exp]
    mt = int(np.bincount(row_sel.ravel()).max())
    assert mt <= 4
    ti, tw = routing_tables(row_sel, row_w, {e: (e, e) for e in range(n_exp)}, 16)
    slots.y.zero_()
    slots.run_layer_quant(q, slot_bytes, bits, x, torch.tensor(slot_of, dtype=torch.int32, device="cuda"),
                          torch.from_numpy(ti).cuda(), torch.from_numpy(tw).cuda(), decode=decode, max_tok=mt)
    torch.cuda.synchronize()
    y = slots.y[:T * H].view(T, H).float()
    ref = torch.zeros(T, H, device="cuda")
    xf = x.float()
    for e in range(n_exp):
        w1, wd = dequant_expert(q[int(slot_of[e])], bits, H, I)
        act = (torch.nn.functional.silu(xf @ w1[:I].T) * (xf @ w1[I:].T)).to(torch.bfloat16).float()
        out = act @ wd.T
        for t in range(T):
            for j in range(K):
                if row_sel[t, j] == e:
                    ref[t] += float(row_w[t, j]) * out[t]
    err = (y - ref).abs().max().item() / ref.abs().max().item()
    assert err <= TOL, f"max rel err {err:.3e}"


def _gemv_reference(q_or_w, bits, H, I, x, row_sel, row_w, slot_of, n_exp):
    import torch
    from paper_2602_03921_b200.ffn import expert_matrices
    from paper_2602_03921_b200.layer_step import dequant_expert
    T = x.shape[0]
    ref = torch.zeros(T, H, device="cuda")
    xf = x.float()
    for e in range(n_exp):
        if bits == 16:
            w1, wd = expert_matrices(q_or_w[int(slot_of[e])].float(), H, I)
        else:
            w1, wd = dequant_expert(q_or_w[int(slot_of[e])], bits, H, I)
        out = (torch.nn.functional.silu(xf @ w1[:I].T) * (xf @ w1[I:].T)) @ wd.T
        for t in range(T):
            for j in range(row_sel.shape[1]):
                if row_sel[t, j] == e:
                    ref[t] += float(row_w[t, j]) * out[t]
    return ref


@pytest.mark.parametrize("case", range(16))
def test_ffn_gemv_random_geometries(case):
    """The decode GEMV over random shapes (H a multiple of 128 from 128 to
    4096, I a multiple of 64 from 64 to 3008, 1-64 experts, 1-4 tokens per
    expert, bf16 / int8 / int4 / int2 slots): partial ring chunks, single-tile
    blocks, CTA-pair and single-CTA units, against fp32 torch (1e-2 of max |y|)."""
    import torch
    from paper_2602_03921_b200.ffn import ExpertSlots, routing_tables
    rng = np.random.default_rng(1000 + case)
    H_ = int(rng.integers(1, 33)) * 128
    I_ = int(rng.integers(1, 48)) * 64
    bits = int(rng.choice([16, 8, 4, 2]))
    n_exp = int(rng.integers(1, 65))
    K = int(rng.integers(1, min(n_exp, 8) + 1))
    T = int(rng.integers(1, 5))
    g = torch.Generator(device="cuda").manual_seed(case)
    n_slots = n_exp + 1
    nq, ns = 3 * H_ * I_, 2 * I_ + H_
    if bits == 16:
        sb = nq * 2
        buf = (torch.randn(n_slots, nq, generator=g, device="cuda") * 0.02).to(torch.bfloat16)
        flat = buf.view(torch.uint8).view(-1)
        refw = buf
    else:
        per = nq * bits // 8 + 4 * ns
        sb = (per + 255) // 256 * 256
        q = torch.zeros(n_slots, sb, dtype=torch.uint8, device="cuda")
        q[:, :nq * bits // 8] = torch.randint(0, 256, (n_slots, nq * bits // 8), generator=g, device="cuda",
                                              dtype=torch.int32).to(torch.uint8)
        qmax = {8: 127, 4: 7, 2: 1}[bits]
        sc = (0.5 + torch.rand(n_slots, ns, generator=g, device="cuda")) * (0.02 / qmax)
        q[:, nq * bits // 8:per] = sc.view(torch.uint8).view(n_slots, ns * 4)
        flat = q.view(-1)
        refw = q
    x = torch.randn(T, H_, generator=g, device="cuda").to(torch.bfloat16)
    row_sel = np.stack([rng.choice(n_exp, size=K, replace=False) for _ in range(T)]).astype(np.int32)
    row_w = rng.uniform(0.01, 0.3, size=(T, K)).astype(np.float32)
    slot_of = rng.permutation(n_slots)[:n_exp]
    mt = int(np.bincount(row_sel.ravel()).max())
    ti, tw = routing_tables(row_sel, row_w, {e: (e, e) for e in range(n_exp)}, 16)
    slots = ExpertSlots(1, H_, I_, max_tokens=T, max_exec=n_exp)
    slots.y.zero_()
    slots.run_layer_quant(flat, sb, bits, x, torch.tensor(slot_of, dtype=torch.int32, device="cuda"),
                          torch.from_numpy(ti).cuda(), torch.from_numpy(tw).cuda(), decode="gemv", max_tok=mt)
    torch.cuda.synchronize()
    y = slots.y[:T * H_].view(T, H_).float()
    ref = _gemv_reference(refw, bits, H_, I_, x, row_sel, row_w, slot_of, n_exp)
    err = (y - ref).abs().max().item() / ref.abs().max().item()
    assert err <= TOL, f"H={H_} I={I_} bits={bits} experts={n_exp} K={K} T={T}: max rel err {err:.3e}"
