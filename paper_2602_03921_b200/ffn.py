"""Physical expert FFN: HBM cache slots + the tcgen05 grouped SwiGLU GEMMs.

Each cache slot holds one expert in the TILE-MAJOR layout the kernels stream
with TMA (every TMA box is one contiguous run of HBM, so weight streaming is
sequential 16 KB bursts instead of 128-byte pieces of 4 KB-strided rows):
    w1 = [gate; up] (logical [2*I, H], K = H) as tiles [I/64][H/64][128][64]:
         tile (m, k) = gate rows 64m..64m+63 then up rows 64m..64m+63, K cols 64k..
    w2 = down       (logical [H, I],   K = I) as tiles [I/64][H/128][128][64]
3*H*I*2 bytes (12,582,912 B for OLMoE-1B-7B: H=2048, I=1024), the same bytes
a host->HBM fetch moves (the pinned store uses the same layout; the tiling is
a property of the expert store, like a checkpoint converted once at load).
`expert_matrices` maps a slot back to the logical matrices. One TMA
descriptor per slot per matrix is built once; kernels pick the descriptor of
the slot an expert lives in.
Layer semantics (no renormalisation, original-softmax weights, matching
the reference's dual-logit routing, routing.py:93-99):
    x <- x + sum_e w[t,e] * down_e(silu(gate_e x) * up_e x)
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._device import _check, _stream, _torch, lib

NPADS = (16, 32, 64, 128)


def npad_for(max_tokens_per_expert: int) -> int:
    for n in NPADS:
        if max_tokens_per_expert <= n:
            return n
    raise ValueError(f"{max_tokens_per_expert} tokens per expert exceeds the largest tile ({NPADS[-1]})")


def tmap(base_ptr: int, rows: int, cols: int, box_rows: int) -> bytes:
    buf = (C.c_uint8 * 128)()
    rc = lib().esim_tmap_bf16(C.addressof(buf), base_ptr, rows, cols, box_rows)
    if rc != 0:
        raise RuntimeError(f"cuTensorMapEncodeTiled failed ({rc})")
    return bytes(buf)


class ExpertSlots:
    """n_slots expert-sized HBM buffers + their TMA descriptors."""

    def __init__(self, n_slots: int, hidden: int, inter: int, max_tokens: int, max_exec: int):
        torch = _torch()
        self.n_slots, self.H, self.I = n_slots, hidden, inter
        self.expert_elems = 3 * hidden * inter
        self.expert_bytes = 2 * self.expert_elems
        self.buf = torch.empty(n_slots * self.expert_elems, dtype=torch.bfloat16, device="cuda")
        base = self.buf.data_ptr()
        w1 = b"".join(tmap(base + s * self.expert_bytes, 2 * inter * hidden // 64, 64, 128) for s in range(n_slots))
        w2 = b"".join(tmap(base + s * self.expert_bytes + 2 * 2 * inter * hidden, inter * hidden // 64, 64, 128)
                      for s in range(n_slots))
        self.w1_maps = torch.frombuffer(bytearray(w1), dtype=torch.uint8).cuda()
        self.w2_maps = torch.frombuffer(bytearray(w2), dtype=torch.uint8).cuda()
        # activation staging, one descriptor pair per token-tile width
        self.max_exec = max_exec
        self.xg = torch.empty(max_exec * NPADS[-1] * hidden, dtype=torch.bfloat16, device="cuda")
        self.act = torch.empty(max_exec * NPADS[-1] * inter, dtype=torch.bfloat16, device="cuda")
        self.x_maps, self.act_maps = {}, {}
        for n in NPADS:
            self.x_maps[n] = torch.frombuffer(bytearray(tmap(self.xg.data_ptr(), max_exec * n, hidden, n)),
                                              dtype=torch.uint8).cuda()
            self.act_maps[n] = torch.frombuffer(bytearray(tmap(self.act.data_ptr(), max_exec * n, inter, n)),
                                                dtype=torch.uint8).cuda()
        self.y = torch.zeros(max_tokens * hidden, dtype=torch.float32, device="cuda")

    def slot_ptr(self, slot: int) -> int:
        return self.buf.data_ptr() + slot * self.expert_bytes

    def slot_view(self, slot: int):
        return self.buf[slot * self.expert_elems:(slot + 1) * self.expert_elems]

    def run_layer(self, x, exec_slot, tok_index, tok_weight, npad: int, stream=None, residual: bool = True,
                  max_tok: int | None = None, decode: str = "gemv") -> None:
        """x[T,H] bf16 (device, updated in place: x += MoE(x)). exec_slot int32
        [n_exec] (device), tok_index int32 [n_exec*npad], tok_weight f32 (device).
        max_tok: the largest token count of an executed expert; <= 4 is a decode
        layer: decode="gemv" streams it straight from the slots (ffn_gemv.cu),
        "tc" runs the fused tcgen05 decode kernel; None = npad (the two-phase
        tcgen05 kernel)."""
        n_exec = int(exec_slot.numel())
        if n_exec > self.max_exec:
            raise ValueError("more executed experts than staged")
        if decode not in ("gemv", "tc"):
            raise ValueError(f"unknown decode kernel {decode!r}")
        st = stream or _stream()
        L = lib()
        if decode == "gemv" and max_tok is not None and 1 <= max_tok <= 4:
            _check(L.esim_ffn_experts_gemv(self.buf.data_ptr(), self.expert_bytes, 16, x.data_ptr(),
                                           exec_slot.data_ptr(), tok_index.data_ptr(), tok_weight.data_ptr(),
                                           self.y.data_ptr(), n_exec, npad, max_tok, self.I, self.H, st),
                   "gemv ffn experts")
        else:
            _check(L.esim_ffn_gather(x.data_ptr(), tok_index.data_ptr(), self.xg.data_ptr(), n_exec, npad, self.H,
                                     st), "gather")
            _check(L.esim_ffn_experts_ex(self.w1_maps.data_ptr(), self.w2_maps.data_ptr(),
                                         self.x_maps[npad].data_ptr(), self.act_maps[npad].data_ptr(),
                                         exec_slot.data_ptr(), tok_index.data_ptr(), tok_weight.data_ptr(),
                                         self.act.data_ptr(), self.y.data_ptr(), n_exec, npad, self.I, self.H,
                                         npad if max_tok is None else max_tok, st), "ffn experts")
        if residual:
            T = x.numel() // self.H
            _check(L.esim_ffn_residual(x.data_ptr(), self.y.data_ptr(), T * self.H, st), "residual")

    def run_layer_quant(self, qslots, slot_bytes: int, bits: int, x, exec_slot, tok_index, tok_weight,
                        stream=None, decode: str = "gemv", max_tok: int = 4) -> None:
        """Decode-like layer (<= 4 tokens per expert, npad 16) over quantised
        slots: qslots uint8 (device) holding tile-major codes of `bits` then
        fp32 row scales per slot (slot_bytes apart, layer_step.cu's format);
        y += MoE(x) with the dequantisation fused into the FFN: decode="gemv"
        (ffn_gemv.cu, codes converted in registers) or "tc"
        (ffn_decode_q_kernel, codes converted into the tcgen05 A operand).
        No residual."""
        n_exec = int(exec_slot.numel())
        if n_exec > self.max_exec:
            raise ValueError("more executed experts than staged")
        if decode not in ("gemv", "tc"):
            raise ValueError(f"unknown decode kernel {decode!r}")
        st = stream or _stream()
        L = lib()
        if decode == "gemv":
            _check(L.esim_ffn_experts_gemv(qslots.data_ptr(), slot_bytes, bits, x.data_ptr(), exec_slot.data_ptr(),
                                           tok_index.data_ptr(), tok_weight.data_ptr(), self.y.data_ptr(), n_exec,
                                           16, max_tok, self.I, self.H, st), "gemv quantised ffn experts")
            return
        _check(L.esim_ffn_gather(x.data_ptr(), tok_index.data_ptr(), self.xg.data_ptr(), n_exec, 16, self.H, st),
               "gather")
        _check(L.esim_ffn_experts_q(qslots.data_ptr(), slot_bytes, bits, self.x_maps[16].data_ptr(),
                                    exec_slot.data_ptr(), tok_index.data_ptr(), tok_weight.data_ptr(),
                                    self.y.data_ptr(), n_exec, self.I, self.H, st), "quantised ffn experts")


def expert_matrices(flat, hidden: int, inter: int):
    """Logical (w1 [2I, H], wd [H, I]) views-turned-copies of one expert stored
    tile-major (see the module docstring); `flat` is the expert's 3*H*I elements."""
    H, I = hidden, inter
    t = flat[:2 * I * H].reshape(I // 64, H // 64, 2, 64, 64)          # [m][k][gate/up][row][col]
    w1 = t.permute(2, 0, 3, 1, 4).reshape(2 * I, H)
    wd = flat[2 * I * H:].reshape(I // 64, H // 128, 128, 64).permute(1, 2, 0, 3).reshape(H, I)
    return w1, wd


def pack_expert(w1, wd, hidden: int, inter: int):
    """Inverse of expert_matrices: logical w1 [2I, H] and wd [H, I] -> the
    expert's tile-major flat 3*H*I elements."""
    H, I = hidden, inter
    t1 = w1.reshape(2, I // 64, 64, H // 64, 64).permute(1, 3, 0, 2, 4).reshape(-1)
    t2 = wd.reshape(H // 128, 128, I // 64, 64).permute(2, 0, 1, 3).reshape(-1)
    import torch                     # layout helper on caller tensors (any device), not a compute path
    return torch.cat([t1, t2])


def routing_tables(row_sel: np.ndarray, row_w: np.ndarray, executed: dict, npad: int):
    """Per executed expert token lists: executed maps expert -> (position, substitute-or-self).
    Returns tok_index [n_exec*npad] (-1 pad) and tok_weight [n_exec*npad]."""
    n_exec = len({v[0] for v in executed.values()})
    ti = np.full((n_exec, npad), -1, np.int32)
    tw = np.zeros((n_exec, npad), np.float32)
    fill = np.zeros(n_exec, np.int32)
    T, K = row_sel.shape
    for t in range(T):
        for j in range(K):
            e = int(row_sel[t, j])
            if e not in executed:
                continue
            pos = executed[e][0]
            ti[pos, fill[pos]] = t
            tw[pos, fill[pos]] = row_w[t, j]
            fill[pos] += 1
    return ti.ravel(), tw.ravel()
