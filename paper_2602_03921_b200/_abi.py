"""ctypes mirrors of the structs in include/specmd_b200.h (plain C ABI)."""
from __future__ import annotations

import ctypes as C

import numpy as np

ESIM_FLAG_FULL_LOG = 1
ESIM_FLAG_NO_DIGEST = 2
ESIM_FLAG_TIME32 = 4
ESIM_PL_FIELDS = 10
ESIM_MAX_E = 256
ESIM_MAX_K = 16


class EsimConfig(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("experts", C.c_int32), ("top_k", C.c_int32),
                ("n_precisions", C.c_int32), ("precisions", C.c_int32 * 4),
                ("expert_bytes", C.c_int64 * 4), ("capacity_bytes", C.c_int64),
                ("bandwidth", C.c_int64), ("compute_us", C.c_int64),
                ("working_prec", C.c_int32), ("routing", C.c_int32), ("lam", C.c_double),
                ("eviction", C.c_int32), ("prefetch", C.c_int32),
                ("sb_decay", C.c_double), ("overfetch", C.c_double), ("percentile", C.c_double),
                ("miss", C.c_int32), ("drop_rank_threshold", C.c_int32),
                ("subst_tolerance", C.c_double), ("degrade_percentile", C.c_double),
                ("flags", C.c_int32), ("trace_id", C.c_int32),
                ("prefetch_noise", C.c_double), ("seed", C.c_uint64)]


class EsimCounters(C.Structure):
    _fields_ = [("totals", C.c_int64 * 15),
                ("ttft_us", C.c_int64), ("total_us", C.c_int64), ("decode_us", C.c_int64),
                ("sync_overhead_us", C.c_int64), ("passes", C.c_int64), ("decode_passes", C.c_int64),
                ("rows_total", C.c_int64), ("faithful_rows", C.c_int64), ("modified_rows", C.c_int64),
                ("pf_tp", C.c_int64), ("pf_pred_total", C.c_int64), ("pf_dem_total", C.c_int64),
                ("pf_records", C.c_int64), ("pf_empty", C.c_int64), ("pf_prec_parts", C.c_int64),
                ("pf_rec_parts", C.c_int64),
                ("ls_forced", C.c_int64), ("ls_unforced", C.c_int64), ("ls_refusals", C.c_int64),
                ("n_recs", C.c_int64), ("n_pred_experts", C.c_int64), ("digest", C.c_uint64),
                ("original_mass", C.c_double), ("executed_mass", C.c_double),
                ("pf_prec_sum", C.c_double), ("pf_rec_sum", C.c_double),
                ("status", C.c_int64), ("pad", C.c_int64 * 3)]


class EsimTraceDesc(C.Structure):
    _fields_ = [("n_passes", C.c_int32), ("num_layers", C.c_int32), ("experts", C.c_int32),
                ("top_k", C.c_int32), ("n_events", C.c_int64), ("n_rows_total", C.c_int64),
                ("pass_tokens", C.c_void_p), ("pass_kind", C.c_void_p),
                ("row_offset", C.c_void_p), ("logits", C.c_void_p)]


class EsimRouterOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "n_dem", "dem_expert", "dem_rank", "dem_gate", "dem_summed", "dem_tokens", "sel_mass",
        "row_sel", "row_w", "n_pred", "pred_expert", "pred_score", "pred_clamped",
        "route_mix", "pred_mix", "layer_pred", "summary")]


class EsimRouteSummary(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("pf_tp", "pf_pred", "pf_dem", "pf_records", "pf_prec_parts", "pf_empty",
                                        "pf_rec_parts", "rows_total")] + \
               [(n, C.c_double) for n in ("orig_f", "orig_c", "prec_f", "prec_c", "rec_f", "rec_c")]


assert C.sizeof(EsimConfig) == 184, C.sizeof(EsimConfig)
assert C.sizeof(EsimCounters) == 360, C.sizeof(EsimCounters)
assert C.sizeof(EsimRouteSummary) == 112, C.sizeof(EsimRouteSummary)
COUNTERS_DTYPE = np.dtype((np.void, C.sizeof(EsimCounters)))


def counters_from_bytes(buf: bytes) -> EsimCounters:
    return EsimCounters.from_buffer_copy(buf)


def trace_desc_host(pk) -> tuple[EsimTraceDesc, list]:
    """EsimTraceDesc over host numpy arrays of a PackedTrace (keeps refs alive)."""
    keep = [np.ascontiguousarray(pk.pass_tokens, np.int32), np.ascontiguousarray(pk.pass_kind, np.int32),
            np.ascontiguousarray(pk.row_offset, np.int64), np.ascontiguousarray(pk.logits, np.float32)]
    d = EsimTraceDesc(pk.n_passes, pk.num_layers, pk.experts, pk.top_k, pk.n_events,
                      int(pk.row_offset[-1]), keep[0].ctypes.data, keep[1].ctypes.data,
                      keep[2].ctypes.data, keep[3].ctypes.data)
    return d, keep


class EsimPolicyOp(C.Structure):
    _fields_ = [("op", C.c_int32), ("key", C.c_int32), ("layer", C.c_int32), ("prec", C.c_int32),
                ("forced", C.c_int32), ("pad", C.c_int32), ("gate", C.c_double)]


class EsimPolicyState(C.Structure):
    _fields_ = [("policy", C.c_int32), ("num_layers", C.c_int32), ("highest_prec", C.c_int32),
                ("n_keys", C.c_int32), ("decay", C.c_double)] + \
               [(n, C.c_void_p) for n in ("seq", "counters", "flags", "key", "count", "signal", "layer", "expert")]


assert C.sizeof(EsimPolicyOp) == 32


class EsimMissQuery(C.Structure):
    _fields_ = [("policy", C.c_int32), ("rank", C.c_int32), ("drop_rank_threshold", C.c_int32),
                ("n_scores", C.c_int32), ("n_residents", C.c_int32), ("ladder_len", C.c_int32),
                ("pct_rank", C.c_int32), ("pad", C.c_int32), ("gate_score", C.c_double),
                ("subst_tolerance", C.c_double)]


class EsimMissDecision(C.Structure):
    _fields_ = [("kind", C.c_int32), ("substitute", C.c_int32), ("fetch", C.c_int32), ("start", C.c_int32)]
