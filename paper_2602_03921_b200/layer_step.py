"""Physical expert-cached MoE layer step (BASELINE.json configs[1]).

OLMoE-1B-7B shape (16 layers x 64 experts, top-8, H=2048, I=1024 SwiGLU,
12,582,912 B per bf16 expert) with the expert store in pinned host memory,
a capacity-bounded pool of HBM cache slots, and the reference's decision
semantics (SimConfig: eviction / prefetch / miss policy, logical clock)
driving real host->HBM copies and real tcgen05 expert FFNs. The decisions
come from the replay kernel (bit-exact with the reference for `cfg`); the
native runtime in csrc/layer_step.cu executes them.

Measured: TTFT (end of the prefill pass) and decode tokens/s with CUDA
events, host-link bytes and achieved GB/s.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from ._device import DeviceTrace, _check, _torch, lib
from .metrics import report_from_counters
from .models import ConfigError


class EsimLSParams(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("num_layers", "experts", "top_k", "hidden", "inter", "n_slots",
                                         "max_tokens", "weight_format", "prec_mask")]


# physical expert format per logical precision (models.PRECISION_CODE): bf16
# for fp16 (the reference's "fp16" sizes), int8 / int4 / int2 codes + per-row
# fp32 scales
WEIGHT_FORMAT = {"fp16": 0, "int8": 1, "int4": 2, "int2": 3}
_QBITS = {0: 0, 1: 8, 2: 4, 3: 2}
_QMAX = {8: 127, 4: 7, 2: 1}
_MIXED_MISS = ("fetch_low", "fetch_priority")


class EsimLSResult(C.Structure):
    _fields_ = [("ttft_ms", C.c_double), ("total_ms", C.c_double), ("decode_ms", C.c_double),
                ("host_enqueue_ms", C.c_double)] + \
               [(n, C.c_int64) for n in ("h2d_bytes", "n_copies", "n_demand_copies", "n_prefetch_copies",
                                         "n_cancelled", "n_ffn_batches", "n_exec_experts", "n_records", "status")]


def _bind():
    L = lib()
    if not hasattr(L, "_ls_bound"):
        vp = C.c_void_p
        L.esim_ls_create.argtypes = [vp, vp]
        L.esim_ls_store.argtypes = [vp]
        L.esim_ls_store.restype = vp
        L.esim_ls_expert_bytes.argtypes = [vp]
        L.esim_ls_expert_bytes.restype = C.c_int64
        L.esim_ls_format.argtypes = [vp, C.c_int32, vp]
        L.esim_ls_format.restype = C.c_int64
        L.esim_ls_store_bytes.argtypes = [vp]
        L.esim_ls_store_bytes.restype = C.c_int64
        L.esim_ls_route_rows.argtypes = [vp, vp, vp, C.c_int64]
        L.esim_ls_slots.argtypes = [vp]
        L.esim_ls_slots.restype = vp
        L.esim_ls_destroy.argtypes = [vp]
        L.esim_ls_last_error.restype = C.c_char_p
        L.esim_ls_run.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.esim_ls_shared_expert.argtypes = [vp, vp, vp, C.c_int32]
        L.esim_ls_capture_layers.argtypes = [vp, vp, C.c_int64]
        L._ls_bound = True
    return L


@dataclass
class LayerStepResult:
    ttft_ms: float
    total_ms: float
    decode_ms: float
    decode_tokens_per_sec: float
    h2d_bytes: int
    h2d_gbs: float
    n_copies: int
    n_demand_copies: int
    n_prefetch_copies: int
    n_cancelled: int
    n_ffn_batches: int
    n_exec_experts: int
    host_enqueue_ms: float
    report: dict                 # the decision stream's reference-format report (logical timeline)
    out: object = None           # last-layer hidden states of every pass (host bf16)
    layers: object = None        # every layer's output per (pass, layer) event (keep_layers)


def code_positions(bits: int) -> list:
    """Bit position (in units of `bits`) of element i of each 32-bit code word
    (int4 / int2): even elements fill the low half-word, odd ones the high
    half-word, pair j at positions (j, PER/2 + j) -- so one shift + one
    LOP3 with 0x000F000F (int4) / 0x00030003 (int2) puts elements (2j, 2j+1)
    into the two halves of a bf16x2 register (ffn_decode_q_kernel)."""
    per = 32 // bits
    return [i // 2 if i % 2 == 0 else per // 2 + i // 2 for i in range(per)]


def pack_codes(q, bits: int):
    """int codes [..., n] (two's complement in `bits`) -> uint8 bytes of the
    slot format: int8 one per byte; int4 / int2 word-interleaved
    (code_positions) in little-endian 32-bit words."""
    import torch
    if bits == 8:
        return q.to(torch.int8).view(torch.uint8)
    per = 32 // bits
    u = (q.to(torch.int64) & ((1 << bits) - 1)).reshape(*q.shape[:-1], q.shape[-1] // per, per)
    w = torch.zeros(u.shape[:-1], dtype=torch.int64, device=q.device)
    for i, pos in enumerate(code_positions(bits)):
        w |= u[..., i] << (bits * pos)
    return _words_to_bytes(w).reshape(*q.shape[:-1], q.shape[-1] * bits // 8)


def _words_to_bytes(w):
    import torch
    w = w & 0xFFFFFFFF
    b = torch.stack([(w >> (8 * k)) & 0xFF for k in range(4)], dim=-1)
    return b.to(torch.uint8)


def unpack_codes(raw, bits: int, n: int):
    """Inverse of pack_codes: the first n codes of `raw` (uint8) as float."""
    import torch
    if bits == 8:
        return raw[:n].view(torch.int8).float()
    per = 32 // bits
    b = raw[:n * bits // 8].to(torch.int64).view(-1, 4)
    w = b[:, 0] | (b[:, 1] << 8) | (b[:, 2] << 16) | (b[:, 3] << 24)
    cols = []
    for i, pos in enumerate(code_positions(bits)):
        c = (w >> (bits * pos)) & ((1 << bits) - 1)
        cols.append(torch.where(c >= (1 << (bits - 1)), c - (1 << bits), c))
    return torch.stack(cols, dim=1).reshape(-1).float()


def dequant_expert(raw, bits: int, hidden: int, inter: int):
    """One quantised expert's bytes (tile-major codes of `bits`, lowest bits
    first, two's complement, then fp32 row scales: 2I gate/up rows, H down
    rows) -> logical (w1 [2I, H], wd [H, I]) = bf16(q * scale) as fp32, on
    raw's device (the test reference / weight inspection; the device path
    dequantises in dequant_kernel / ffn_decode_q_kernel)."""
    from .ffn import expert_matrices
    import torch
    H, I = hidden, inter
    nq = 3 * H * I
    q = unpack_codes(raw, bits, nq)
    sc = raw[nq * bits // 8:nq * bits // 8 + 4 * (2 * I + H)].view(torch.float32)
    w1q, wdq = expert_matrices(q, H, I)
    w1 = (w1q * sc[:2 * I, None]).to(torch.bfloat16).float()
    wd = (wdq * sc[2 * I:, None]).to(torch.bfloat16).float()
    return w1, wd


class LayerStepEngine:
    """Pinned expert store + HBM slots + copy/compute streams for one model.

    The store holds the working precision, or -- for the mixed-precision miss
    policies (fetch_low / fetch_priority, miss.py) -- every rung of the
    model's precision ladder; each HBM slot then holds whichever precision
    the decision stream fetched into it and the FFN dequantises per slot."""

    def __init__(self, cfg, hidden: int = 2048, inter: int = 1024, max_tokens: int = 64):
        from ._device import ensure_host_semantics
        ensure_host_semantics()
        torch = _torch()
        m = cfg.model
        self.cfg, self.H, self.I = cfg, hidden, inter
        if cfg.working_precision not in WEIGHT_FORMAT:
            raise ConfigError(f"physical layer step stores fp16 (bf16), int8, int4 or int2 experts, not "
                              f"{cfg.working_precision}")
        self.weight_format = WEIGHT_FORMAT[cfg.working_precision]
        self.precisions = tuple(m.precisions) if cfg.miss in _MIXED_MISS else (cfg.working_precision,)
        self.prec_mask = sum(1 << WEIGHT_FORMAT[q] for q in set(self.precisions) | {cfg.working_precision})
        lowest = min(m.expert_bytes(q) for q in self.precisions + (cfg.working_precision,))
        self.n_slots = min(cfg.capacity_bytes() // lowest, m.num_layers * m.experts_per_layer)
        p = EsimLSParams(m.num_layers, m.experts_per_layer, m.top_k, hidden, inter, self.n_slots, max_tokens,
                         self.weight_format, self.prec_mask)
        self._h = C.c_void_p()
        L = _bind()
        rc = L.esim_ls_create(C.addressof(p), C.addressof(self._h))
        if rc:
            raise RuntimeError(f"esim_ls_create failed ({rc}): {L.esim_ls_last_error().decode()}")
        self.expert_bytes = L.esim_ls_expert_bytes(self._h)
        self.n_experts_total = m.num_layers * m.experts_per_layer
        self.formats = {}                                # precision code -> (bytes per expert, store offset)
        for code in range(4):
            off = C.c_int64()
            nb = L.esim_ls_format(self._h, code, C.addressof(off))
            if nb:
                self.formats[code] = (nb, off.value)
        nbytes = L.esim_ls_store_bytes(self._h)
        buf = (C.c_uint8 * nbytes).from_address(L.esim_ls_store(self._h))
        self.store_bytes = torch.frombuffer(buf, dtype=torch.uint8)  # pinned host view
        self.torch = torch

    def _row_of_element(self):
        """Scale row (0..2I+H) of every element of a tile-major expert."""
        from .ffn import pack_expert
        torch, H, I = self.torch, self.H, self.I
        r1 = torch.arange(2 * I, device="cuda", dtype=torch.int64)[:, None].expand(2 * I, H)
        r2 = (2 * I + torch.arange(H, device="cuda", dtype=torch.int64))[:, None].expand(H, I)
        return pack_expert(r1, r2, H, I)

    def init_weights(self, seed: int = 0, std: float = 0.02) -> None:
        """Random-init experts, generated on the GPU in chunks and copied into
        the pinned store: bf16 masters N(0, std); every quantised precision
        in the store is the per-row quantisation of the same master
        (int8 / int4: symmetric absmax scales; int2: ternary codes with the
        row's mean |w| as scale), so all rungs of one expert agree."""
        torch = self.torch
        H, I = self.H, self.I
        nq, ns = 3 * H * I, 2 * I + H
        g = torch.Generator(device="cuda").manual_seed(seed)
        chunk = max(1, min(32, (1 << 30) // (nq * 4)))
        rows = self._row_of_element() if any(c for c in self.formats) else None
        for e0 in range(0, self.n_experts_total, chunk):
            n = min(chunk, self.n_experts_total - e0)
            w = (torch.randn(n, nq, generator=g, device="cuda") * std).to(torch.bfloat16)
            for code, (nb, off) in self.formats.items():
                dst = self.store_bytes[off + e0 * nb:off + (e0 + n) * nb]
                if code == 0:
                    dst.copy_(w.view(torch.uint8).reshape(-1))
                    continue
                bits = _QBITS[code]
                qmax = _QMAX[bits]
                wf = w.float()
                idx = rows.expand(n, nq)
                if bits == 2:
                    sc = torch.zeros(n, ns, device="cuda").scatter_add_(1, idx, wf.abs()) / \
                        torch.bincount(rows, minlength=ns).float()
                else:
                    sc = torch.zeros(n, ns, device="cuda").scatter_reduce_(1, idx, wf.abs(), "amax") / qmax
                sc = torch.clamp(sc, min=1e-12)
                q = torch.clamp(torch.round(wf / torch.gather(sc, 1, idx)), -qmax, qmax).to(torch.int32)
                codes = pack_codes(q, bits)              # int8 bytes / word-interleaved int4, int2
                blob = torch.cat([codes, sc.contiguous().view(torch.uint8).view(n, ns * 4)], dim=1)
                dst.copy_(blob.reshape(-1))
        torch.cuda.synchronize()

    def attach_shared_expert(self, inter: int, seed: int = 1, std: float = 0.02) -> None:
        """Always-resident shared expert per layer (Qwen1.5-MoE-A2.7B: I = 5632,
        BASELINE.json configs[3]), random-init bf16 N(0, std) in HBM, outside the
        expert cache (the reference sizes only routed experts).
        Each layer adds sigmoid(x . gate_l) * SwiGLU_l(x) before the residual."""
        torch = self.torch
        L, H = self.cfg.model.num_layers, self.H
        g = torch.Generator(device="cuda").manual_seed(seed)
        self.shared_inter = inter
        self.shared_w = (torch.randn(L, 3 * H * inter, generator=g, device="cuda") * std).to(torch.bfloat16)
        self.shared_gate = (torch.randn(L, H, generator=g, device="cuda") * std).to(torch.bfloat16)
        rc = _bind().esim_ls_shared_expert(self._h, self.shared_w.data_ptr(), self.shared_gate.data_ptr(), inter)
        if rc:
            raise RuntimeError(f"esim_ls_shared_expert failed ({rc}): {_bind().esim_ls_last_error().decode()}")

    @property
    def shared_bytes(self) -> int:
        return 0 if not getattr(self, "shared_inter", 0) else self.shared_w.numel() * 2 + self.shared_gate.numel() * 2

    def shared_matrices(self, layer: int):
        """(w1 [2Is, H], wd [H, Is], gate [H]) of the layer's shared expert, fp32."""
        from .ffn import expert_matrices
        w1, wd = expert_matrices(self.shared_w[layer], self.H, self.shared_inter)
        return w1.float(), wd.float(), self.shared_gate[layer].float()

    def expert_weights(self, layer: int, expert: int, precision: str | None = None):
        """The expert's stored bytes at `precision` (default: working):
        bf16 elements, or raw codes + scale bytes."""
        code = WEIGHT_FORMAT[precision or self.cfg.working_precision]
        nb, off = self.formats[code]
        i = layer * self.cfg.model.experts_per_layer + expert
        raw = self.store_bytes[off + i * nb:off + (i + 1) * nb]
        return raw.view(self.torch.bfloat16) if code == 0 else raw

    def expert_matrices(self, layer: int, expert: int, precision: str | None = None):
        """Logical (w1 [2I, H], wd [H, I]) as the FFN sees them (quantised:
        bf16(q * scale)), fp32, on the GPU."""
        from .ffn import expert_matrices
        H, I = self.H, self.I
        code = WEIGHT_FORMAT[precision or self.cfg.working_precision]
        raw = self.expert_weights(layer, expert, precision).cuda()
        if code == 0:
            w1, wd = expert_matrices(raw, H, I)
            return w1.float(), wd.float()
        return dequant_expert(raw, _QBITS[code], H, I)

    def run(self, trace, x_prefill, x_decode, keep_outputs: bool = False,
            keep_layers: bool = False) -> LayerStepResult:
        """One request. keep_outputs: the last layer's hidden states of every
        pass (res.out); keep_layers: every layer's (res.layers, [events] list of
        [T, H] bf16 host tensors, events in (pass, layer) order)."""
        from .engine import check_geometry
        check_geometry(self.cfg, trace)
        torch = self.torch
        pk = trace.packed()
        cap = None
        if keep_layers:
            cap = torch.empty(int(pk.pass_tokens.sum()) * self.cfg.model.num_layers * self.H,
                              dtype=torch.bfloat16).pin_memory()
            _bind().esim_ls_capture_layers(self._h, cap.data_ptr(), cap.numel() // self.H)
        dt = DeviceTrace(pk)
        ctoks = np.ascontiguousarray(pk.pass_tokens, np.int32)
        c = self.cfg.to_c(0, True)
        rows = int(pk.pass_tokens.sum())
        out = torch.empty(rows * self.H, dtype=torch.bfloat16).pin_memory()
        counters = _abi.EsimCounters()
        per_layer = np.zeros((self.cfg.model.num_layers, _abi.ESIM_PL_FIELDS), np.int64)
        res = EsimLSResult()
        L = _bind()
        torch.cuda.synchronize()
        rc = L.esim_ls_run(self._h, C.addressof(dt.desc), ctoks.ctypes.data, C.addressof(c), x_prefill.data_ptr(),
                           x_decode.data_ptr(), out.data_ptr(), C.addressof(counters), per_layer.ctypes.data,
                           C.addressof(res))
        if keep_layers:
            L.esim_ls_capture_layers(self._h, None, 0)
        if rc:
            raise RuntimeError(f"esim_ls_run failed ({rc}): {L.esim_ls_last_error().decode()}")
        layers = None
        if keep_layers:
            layers, r0 = [], 0
            for p in range(pk.n_passes):
                T = int(pk.pass_tokens[p])
                for _ in range(self.cfg.model.num_layers):
                    layers.append(cap[r0 * self.H:(r0 + T) * self.H].view(T, self.H))
                    r0 += T
        rep = report_from_counters(self.cfg.echo(), self.cfg.model.num_layers,
                                   self.cfg.hardware.per_layer_compute_us, counters, per_layer)
        decode_passes = int((pk.pass_kind == 1).sum())
        return LayerStepResult(
            ttft_ms=res.ttft_ms, total_ms=res.total_ms, decode_ms=res.decode_ms,
            decode_tokens_per_sec=decode_passes / (res.decode_ms / 1e3) if res.decode_ms > 0 else 0.0,
            h2d_bytes=res.h2d_bytes, h2d_gbs=res.h2d_bytes / (res.total_ms / 1e3) / 1e9,
            n_copies=res.n_copies, n_demand_copies=res.n_demand_copies, n_prefetch_copies=res.n_prefetch_copies,
            n_cancelled=res.n_cancelled, n_ffn_batches=res.n_ffn_batches, n_exec_experts=res.n_exec_experts,
            host_enqueue_ms=res.host_enqueue_ms, report=rep, out=out if keep_outputs else None, layers=layers)

    def route_rows(self, rows: int):
        """The last run's executed routing: (sel int16 [rows, K], w float32 [rows, K])."""
        K = self.cfg.model.top_k
        sel = np.zeros((rows, K), np.int16)
        w = np.zeros((rows, K), np.float32)
        rc = _bind().esim_ls_route_rows(self._h, sel.ctypes.data, w.ctypes.data, rows)
        if rc:
            raise RuntimeError(f"esim_ls_route_rows failed ({rc}): {_bind().esim_ls_last_error().decode()}")
        return sel, w

    def close(self) -> None:
        if self._h:
            _bind().esim_ls_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
