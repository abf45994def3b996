"""Event-log records: the parity artefact of the layer step.

The reference appends six record kinds to `Simulation.log`
(`expertsim/metrics.py:62-128`): AccessRec, EvictRec, PrefetchRec,
PredictionRec, RouteRec, PassRec. The device replay emits the same stream
as fixed 64-byte structs (`EsimRec` in include/specmd_b200.h); this module
defines

* the record dataclasses the host API hands back (same field names and
  meanings as the reference, so report code and user code read alike),
* the canonical tuple form both sides are hashed in (floats as
  `float.hex()`, enums as their reference strings), and
* the struct <-> record decoding of the device stream.

Parity is "identical canonical tuple sequence", checked by digest and, on
small cases, record by record.
"""
from __future__ import annotations

import hashlib
import json
import struct
from dataclasses import dataclass

import numpy as np

# enum tables shared with the C ABI (include/specmd_b200.h)
PRECISIONS = ("fp16", "int8", "int4", "int2")          # code 0..3, -1 = None
OUTCOMES = ("hit", "fetch", "wait", "drop", "subst")     # AccessRec.outcome
MISS_CLASSES = ("compulsory", "collision", "capacity")   # -1 = None
CAUSES = ("demand", "prefetch")
PF_EVENTS = ("submitted", "started", "completed", "skipped", "dropped")
PF_REASONS = ("", "resident", "in_flight", "no_space", "superseded")
PASS_KINDS = ("prefill", "decode")

REC_ACCESS, REC_EVICT, REC_PREFETCH, REC_PREDICTION, REC_ROUTE, REC_PASS = 1, 2, 3, 4, 5, 6


@dataclass
class AccessRec:
    pass_id: int
    layer: int
    expert: int
    tokens: int
    rank: int
    outcome: str
    miss_class: str | None
    blocked_us: int
    weight_delta: float
    precision: str | None
    substitute: int | None = None


@dataclass
class EvictRec:
    pass_id: int
    layer: int
    victim_layer: int
    victim_expert: int
    precision: str
    cause: str
    forced: bool


@dataclass
class PrefetchRec:
    event: str
    pass_id: int
    layer: int
    target_layer: int
    expert: int
    time_us: int
    score: float = 0.0
    reason: str = ""


@dataclass
class PredictionRec:
    pass_id: int
    layer: int
    target_layer: int
    experts: tuple
    clamped: bool


@dataclass
class RouteRec:
    pass_id: int
    layer: int
    rows: int
    faithful_rows: int
    modified_rows: int
    selected_mass: float
    original_mass: float
    executed_mass: float


@dataclass
class PassRec:
    pass_id: int
    kind: str
    tokens: int
    start_us: int
    end_us: int
    blocked_us: int


def _h(x: float) -> str:
    return float(x).hex()


def canon_reference_record(r) -> tuple:
    """Canonical tuple of one record (reference dataclass or ours: the field
    names are the same, so this works on both)."""
    name = type(r).__name__
    if name == "AccessRec":
        return ("A", r.pass_id, r.layer, r.expert, r.tokens, r.rank, r.outcome,
                r.miss_class or "", int(r.blocked_us), _h(r.weight_delta),
                r.precision or "", -1 if r.substitute is None else int(r.substitute))
    if name == "EvictRec":
        return ("E", r.pass_id, r.layer, r.victim_layer, r.victim_expert, r.precision,
                r.cause, int(bool(r.forced)))
    if name == "PrefetchRec":
        return ("F", r.event, r.pass_id, r.layer, r.target_layer, r.expert, int(r.time_us),
                _h(r.score), r.reason)
    if name == "PredictionRec":
        return ("P", r.pass_id, r.layer, r.target_layer, [int(e) for e in r.experts],
                int(bool(r.clamped)))
    if name == "RouteRec":
        return ("R", r.pass_id, r.layer, r.rows, r.faithful_rows, r.modified_rows,
                _h(r.selected_mass), _h(r.original_mass), _h(r.executed_mass))
    if name == "PassRec":
        return ("S", r.pass_id, r.kind, r.tokens, int(r.start_us), int(r.end_us), int(r.blocked_us))
    raise TypeError(f"not a log record: {r!r}")


def digest_records(canon: list) -> str:
    """sha256 over the JSON lines of canonical tuples."""
    h = hashlib.sha256()
    for t in canon:
        h.update(json.dumps(t, separators=(",", ":")).encode())
        h.update(b"\n")
    return h.hexdigest()


# ---------------------------------------------------------------------------
# device stream decoding
# ---------------------------------------------------------------------------
# struct EsimRec { int32 kind, pass_id, layer, i0, i1, i2, i3, i4;
#                  int64 t0, t1, t2; double x0; }   -- 64 bytes
REC_DTYPE = np.dtype([("kind", "<i4"), ("pass_id", "<i4"), ("layer", "<i4"),
                      ("i0", "<i4"), ("i1", "<i4"), ("i2", "<i4"), ("i3", "<i4"), ("i4", "<i4"),
                      ("t0", "<i8"), ("t1", "<i8"), ("t2", "<i8"), ("x0", "<f8")])
assert REC_DTYPE.itemsize == 64


def _bits_to_f64(v: int) -> float:
    return struct.unpack("<d", struct.pack("<q", int(v)))[0]


def _prec(code: int):
    return None if code < 0 else PRECISIONS[code]


def decode_records(arr: np.ndarray, pred_experts: np.ndarray) -> list:
    """Decode an EsimRec array (REC_DTYPE) into record dataclasses.

    Field mapping (must match csrc/replay.cu and oracle/esim_oracle.c):
      ACCESS     i0=expert i1=tokens i2=rank i3=outcome|miss_class<<8|(prec+1)<<16
                 i4=substitute(-1) t0=blocked x0=weight_delta
      EVICT      i0=victim_layer i1=victim_expert i2=prec i3=cause i4=forced
      PREFETCH   i0=event i1=target_layer i2=expert i3=reason t0=time x0=score
      PREDICTION i0=target_layer i1=count i2=clamped t0=offset into pred_experts
      ROUTE      i0=rows i1=faithful i2=modified x0=selected t1=bits(original) t2=bits(executed)
      PASS       i0=kind i1=tokens t0=start t1=end t2=blocked
    """
    out = []
    for r in arr.tolist():
        kind, p, layer, i0, i1, i2, i3, i4, t0, t1, t2, x0 = r
        if kind == REC_ACCESS:
            oc, mc, pc = i3 & 0xFF, (i3 >> 8) & 0xFF, ((i3 >> 16) & 0xFF) - 1
            out.append(AccessRec(p, layer, i0, i1, i2, OUTCOMES[oc],
                                 None if mc == 0xFF else MISS_CLASSES[mc], t0, x0,
                                 _prec(pc), None if i4 < 0 else i4))
        elif kind == REC_EVICT:
            out.append(EvictRec(p, layer, i0, i1, PRECISIONS[i2], CAUSES[i3], bool(i4)))
        elif kind == REC_PREFETCH:
            out.append(PrefetchRec(PF_EVENTS[i0], p, layer, i1, i2, t0, x0, PF_REASONS[i3]))
        elif kind == REC_PREDICTION:
            ex = tuple(int(e) for e in pred_experts[t0:t0 + i1])
            out.append(PredictionRec(p, layer, i0, ex, bool(i2)))
        elif kind == REC_ROUTE:
            out.append(RouteRec(p, layer, i0, i1, i2, x0, _bits_to_f64(t1), _bits_to_f64(t2)))
        elif kind == REC_PASS:
            out.append(PassRec(p, PASS_KINDS[i0], i1, t0, t1, t2))
        else:
            raise ValueError(f"bad record kind {kind}")
    return out
