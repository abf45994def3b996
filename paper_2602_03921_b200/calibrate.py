"""HardwareSpec calibrated to the box it runs on.

The reference's logical clock (models.py:126-145) charges `transfer_us =
ceil(bytes * 1e6 / bandwidth)` per fetch and a constant
`per_layer_compute_us` per layer; its defaults (5 GB/s, 2000 us) model a
PCIe-attached consumer GPU. Here both come from this B200: the pinned
host -> HBM copy bandwidth measured on a copy stream, and the grouped expert
FFN's measured per-layer time (CUDA events, L2 flushed between layers) for
the run's own shapes -- a prefill layer of the trace's first pass and a
decode layer, weighted by how many passes of each kind the trace has. The
decisions made at these ratios are still bit-exact with the reference run
with the same HardwareSpec (only the integers in the config change).
"""
from __future__ import annotations

import math

import numpy as np

from .models import HardwareSpec


def measure_link_gbs(nbytes: int = 1 << 30, reps: int = 5, trials: int = 3) -> float:
    """Pinned host -> HBM copy bandwidth (GB/s) on a side stream: the best of
    `trials` timings of `reps` back-to-back 1 GiB copies (the link's peak, not
    an average over whatever else the host was doing)."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        d.copy_(h, non_blocking=True)
    s.synchronize()
    best = 0.0
    for _ in range(trials):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record()
            for _ in range(reps):
                d.copy_(h, non_blocking=True)
            e1.record()
        s.synchronize()
        best = max(best, nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


def _routing(tokens: int, top_k: int, experts: int, rng):
    row_sel = np.stack([rng.choice(experts, size=top_k, replace=False) for _ in range(tokens)]).astype(np.int32)
    row_w = rng.uniform(0.01, 0.3, size=(tokens, top_k)).astype(np.float32)
    return row_sel, row_w


def measure_layer_us(hidden: int, inter: int, experts: int, top_k: int, tokens: int, precision: str = "fp16",
                     iters: int = 20, seed: int = 0) -> float:
    """Median per-layer time (us) of the grouped expert FFN for `tokens` rows
    routed top-k over `experts` experts (the layer step's kernels: bf16
    tcgen05 two-phase / fused decode; quantised decode with the dequant
    fused into the operand path). Quantised prefills are timed on the bf16
    kernel (the engine dequantises to bf16 scratch first, so this is their
    lower bound)."""
    import torch
    from .ffn import ExpertSlots, npad_for, routing_tables
    rng = np.random.default_rng(seed)
    row_sel, row_w = _routing(tokens, top_k, experts, rng)
    used = np.unique(row_sel)
    remap = {int(e): i for i, e in enumerate(used)}
    row_sel = np.vectorize(remap.get)(row_sel).astype(np.int32)
    n_exec = len(used)
    mt = int(np.bincount(row_sel.ravel()).max())
    quant = precision != "fp16" and mt <= 4
    npad = 16 if quant else npad_for(mt)
    slots = ExpertSlots(n_exec, hidden, inter, max_tokens=max(tokens, 1), max_exec=n_exec)
    slots.buf.copy_((torch.randn(slots.buf.numel(), device="cuda") * 0.02).to(torch.bfloat16))
    ti, tw = routing_tables(row_sel, row_w, {e: (e, e) for e in range(n_exec)}, npad)
    ti, tw = torch.from_numpy(ti).cuda(), torch.from_numpy(tw).cuda()
    es = torch.arange(n_exec, dtype=torch.int32, device="cuda")
    x = torch.randn(tokens, hidden, device="cuda").to(torch.bfloat16)
    if quant:
        bits = {"int8": 8, "int4": 4, "int2": 2}[precision]
        nq, ns = 3 * hidden * inter, 2 * inter + hidden
        per = nq * bits // 8 + 4 * ns
        sb = (per + 255) // 256 * 256
        qbuf = torch.randint(0, 256, (n_exec * sb,), device="cuda", dtype=torch.int32).to(torch.uint8)
        qv = qbuf.view(n_exec, sb)
        qv[:, nq * bits // 8:per] = torch.full((n_exec, ns), 0.01, device="cuda").view(torch.uint8).view(n_exec, ns * 4)

        def run():
            slots.run_layer_quant(qbuf, sb, bits, x, es, ti, tw)
    else:
        def run():
            slots.run_layer(x, es, ti, tw, npad, residual=False, max_tok=mt)
    flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for a, b in ev:
        flush.zero_()
        a.record()
        run()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3


def calibrated_hardware(spec, trace, hidden: int, inter: int, precision: str, capacity_bytes: int,
                        link_gbs: float | None = None) -> tuple[HardwareSpec, dict]:
    """HardwareSpec(capacity_bytes, measured link bytes/s, measured per-layer us)
    for `trace`'s pass mix, plus the measurements."""
    link = measure_link_gbs() if link_gbs is None else link_gbs
    pk = trace.packed()
    prefill_tokens = int(pk.pass_tokens[pk.pass_kind == 0].max()) if (pk.pass_kind == 0).any() else 1
    n_pre, n_dec = int((pk.pass_kind == 0).sum()), int((pk.pass_kind == 1).sum())
    pre_us = measure_layer_us(hidden, inter, spec.experts_per_layer, spec.top_k, prefill_tokens, precision)
    dec_us = measure_layer_us(hidden, inter, spec.experts_per_layer, spec.top_k, 1, precision)
    per_layer = max(1, int(round((n_pre * pre_us + n_dec * dec_us) / max(1, n_pre + n_dec))))
    hw = HardwareSpec(capacity_bytes=capacity_bytes, bandwidth_bytes_per_sec=int(math.floor(link * 1e9)),
                      per_layer_compute_us=per_layer)
    return hw, {"link_gbs": link, "prefill_layer_us": pre_us, "decode_layer_us": dec_us,
                "per_layer_compute_us": per_layer, "bandwidth_bytes_per_sec": hw.bandwidth_bytes_per_sec,
                "passes": {"prefill": n_pre, "decode": n_dec}}
