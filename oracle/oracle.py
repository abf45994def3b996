"""ctypes wrapper of the C oracle (oracle/esim_oracle.c).

TEST INFRASTRUCTURE: used by tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline / reference legs only, as the checker. It returns results in
the same shapes as the device path (EsimCounters, per-layer counters,
decoded records) so tests compare the two directly.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import subprocess
from dataclasses import dataclass

import numpy as np

from paper_2602_03921_b200 import _abi
from paper_2602_03921_b200.metrics import report_from_counters
from paper_2602_03921_b200.prefetch import PREFETCH_CODE, apply_prediction_noise
from paper_2602_03921_b200.records import REC_DTYPE, decode_records

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libesim_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.esim_oracle_set_host_sum(1 if sys.version_info >= (3, 12) else 0)   # this interpreter's sum()
        vp = C.c_void_p
        L.esim_oracle_run.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_int64, vp, C.c_int64]
        L.esim_oracle_run_batch.argtypes = [vp, C.c_int, vp, C.c_int, vp, vp, C.c_int]
        L.esim_oracle_predict.argtypes = [vp, C.c_int, C.c_double, C.c_double, vp, vp, vp, vp]
        L.esim_oracle_softmax.argtypes = [vp, C.c_int, C.c_int, vp]
        L.esim_oracle_row_sum_f64.argtypes = [vp, C.c_int]
        L.esim_oracle_row_sum_f64.restype = C.c_double
        L.esim_oracle_row_sum_f32.argtypes = [vp, C.c_int]
        L.esim_oracle_row_sum_f32.restype = C.c_float
        L.esim_oracle_expf_array.argtypes = [vp, C.c_long, vp]
        L.esim_oracle_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data


def softmax(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    if x.ndim == 1:
        x = x[None]
    out = np.empty_like(x)
    lib().esim_oracle_softmax(_p(x), x.shape[0], x.shape[1], _p(out))
    return out


def expf(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty_like(x)
    lib().esim_oracle_expf_array(_p(x), x.size, _p(out))
    return out


def predictions(pk, mode: int, overfetch: float, percentile: float):
    n = pk.n_events
    off = np.zeros(n + 1, np.int32)
    ex = np.zeros(n * pk.experts, np.int32)
    sc = np.zeros(n * pk.experts, np.float32)
    cl = np.zeros(n, np.int32)
    desc, keep = _abi.trace_desc_host(pk)
    lib().esim_oracle_predict(C.addressof(desc), mode, overfetch, percentile, _p(off), _p(ex), _p(sc), _p(cl))
    return off, ex, sc, cl


def noised_prediction_stream(offsets, experts, scores, clamped, num_layers: int, n_passes: int,
                             num_experts: int, noise: float, seed: int):
    """Apply prediction noise to a whole trace's prediction stream.

    Inputs are the per-event predictions (event = pass*L + layer, each event
    as a TARGET layer). The reference draws noise in submission order --
    pass by pass, layer 0..L-2 predicting layer+1 -- from one
    default_rng(seed) (engine.py:413, 653-666); this replays that order and
    returns new (offsets, experts, scores, clamped) arrays.
    """
    rng = np.random.default_rng(seed)
    n_events = num_layers * n_passes
    out_e, out_s = [], []
    new_off = np.zeros(n_events + 1, np.int32)
    lists: dict = {}
    for p in range(n_passes):
        for layer in range(num_layers - 1):
            ev = p * num_layers + layer + 1
            a, b = int(offsets[ev]), int(offsets[ev + 1])
            preds = [(int(experts[i]), float(scores[i])) for i in range(a, b)]
            lists[ev] = apply_prediction_noise(preds, num_experts, noise, rng)
    pos = 0
    for ev in range(n_events):
        new_off[ev] = pos
        for e, s in lists.get(ev, []):
            out_e.append(e)
            out_s.append(s)
            pos += 1
    new_off[n_events] = pos
    return (new_off, np.asarray(out_e, np.int32), np.asarray(out_s, np.float32),
            np.asarray(clamped, np.int32).copy())


@dataclass
class OracleResult:
    counters: object
    per_layer: np.ndarray
    log: list | None
    report: dict


def run(cfg, trace, full_log: bool = True, rec_cap: int | None = None) -> OracleResult:
    """One reference-equivalent run on the CPU oracle."""
    pk = trace.packed()
    desc, keep = _abi.trace_desc_host(pk)
    c = cfg.to_c(0, full_log)
    po = [None] * 4
    if cfg.prefetch != "none" and cfg.prefetch_noise > 0.0:
        off, ex, sc, cl = predictions(pk, PREFETCH_CODE[cfg.prefetch], cfg.overfetch, cfg.percentile)
        po = noised_prediction_stream(off, ex, sc, cl, pk.num_layers, pk.n_passes, pk.experts,
                                      cfg.prefetch_noise, cfg.seed)
    L = cfg.model.num_layers
    counters = _abi.EsimCounters()
    per_layer = np.zeros((L, _abi.ESIM_PL_FIELDS), np.int64)
    if rec_cap is None:
        rows = int(pk.row_offset[-1])
        rec_cap = 64 + pk.n_events * (6 + 12 * pk.experts) + rows * pk.top_k * 2
    recs = np.zeros(rec_cap if full_log else 0, REC_DTYPE)
    pexp = np.zeros(pk.n_events * pk.experts if full_log else 0, np.int32)
    ptrs = [None if a is None else _p(a) for a in po]
    rc = lib().esim_oracle_run(C.addressof(c), C.addressof(desc), *ptrs, C.addressof(counters),
                               _p(per_layer), _p(recs) if full_log else None, rec_cap,
                               _p(pexp) if full_log else None, pexp.shape[0])
    if rc != 0:
        raise RuntimeError(f"oracle run failed ({rc}): {lib().esim_oracle_last_error().decode()}")
    log = decode_records(recs[:counters.n_recs], pexp) if full_log else None
    report = report_from_counters(cfg.echo(), L, cfg.hardware.per_layer_compute_us, counters, per_layer)
    return OracleResult(counters, per_layer, log, report)


def run_batch(cfgs, traces_by_id, nthreads: int):
    """Many runs (no logs, no noise) on nthreads host threads; returns counters + per-layer."""
    packs = [t.packed() for t in traces_by_id]
    descs, keeps = zip(*[_abi.trace_desc_host(pk) for pk in packs])
    darr = (_abi.EsimTraceDesc * len(descs))(*descs)
    carr = (_abi.EsimConfig * len(cfgs))(*cfgs)
    maxL = max(c.num_layers for c in cfgs)
    counters = (_abi.EsimCounters * len(cfgs))()
    per_layer = np.zeros((len(cfgs), maxL, _abi.ESIM_PL_FIELDS), np.int64)
    rc = lib().esim_oracle_run_batch(C.addressof(carr), len(cfgs), C.addressof(darr), nthreads,
                                     C.addressof(counters), _p(per_layer), maxL)
    if rc != 0:
        raise RuntimeError(f"oracle batch failed ({rc}): {lib().esim_oracle_last_error().decode()}")
    return list(counters), per_layer


def set_host_sum(neumaier: bool) -> None:
    """Reproduce CPython >= 3.12 (True) or <= 3.11 (False) builtin sum()."""
    lib().esim_oracle_set_host_sum(1 if neumaier else 0)
