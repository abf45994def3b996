"""Miss-handler plug-in surface (mirror of expertsim/miss.py:1-140).

Inside a run the decision (fetch / fetch_low / fetch_priority cascade /
drop:rank / subst:tolerance) is taken by the replay kernel (csrc/replay.cu)
with the reference's exact tie-breaks and float64 comparisons. The
standalone plug-ins below keep the reference's signatures for callers with
their own engine: `find_substitute` and the decision part of
`resolve_miss` run as a one-warp device kernel (csrc/policy.cu,
esim_miss_decide); the fetch cascade then calls the caller's `fetch_fn`
(the engine's own make-space / transfer / block step, miss.py:61-63).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Callable

from .models import ConfigError

FETCH = "fetch"
FETCH_LOW = "fetch_low"
FETCH_PRIORITY = "fetch_priority"
DROP = "drop"
SUBST = "subst"
MISS_NAMES = (FETCH, FETCH_LOW, FETCH_PRIORITY, DROP, SUBST)
MISS_CODE = {n: i for i, n in enumerate(MISS_NAMES)}

FETCHED, DROPPED, SUBSTITUTED = "fetch", "drop", "subst"


@dataclass(frozen=True)
class MissConfig:
    policy: str = FETCH
    drop_rank_threshold: int = 2
    subst_tolerance: float = 0.05
    degrade_percentile: float = 60.0

    def __post_init__(self) -> None:
        if self.policy not in MISS_NAMES:
            raise ConfigError(f"unknown miss policy {self.policy!r}; expected one of {', '.join(MISS_NAMES)}")
        if self.drop_rank_threshold < 1:
            raise ConfigError("drop_rank_threshold must be >= 1")
        if self.subst_tolerance < 0:
            raise ConfigError("subst_tolerance must be >= 0")
        if not 0.0 <= self.degrade_percentile < 100.0:
            raise ConfigError("degrade_percentile must be in [0, 100)")


@dataclass
class MissOutcome:
    kind: str
    blocked_us: int = 0
    weight_delta: float = 0.0
    precision: str | None = None
    substitute: int | None = None


# fetch_fn(precision, final) -> blocked_us, or None when a non-final probe
# cannot make space without forcing (miss.py:61-63)
FetchFn = Callable[[str, bool], "int | None"]


def _decide(policy: str, rank: int, drop_rank_threshold: int, gate_score: float, subst_tolerance: float,
            layer_scores, layer_residents, ladder_len: int, degrade_percentile: float):
    from . import _abi
    from ._device import lib
    import numpy as np
    scores = np.ascontiguousarray(np.asarray(list(layer_scores), dtype=np.float64))
    res = list(layer_residents)
    rexp = np.ascontiguousarray([int(e) for e, _ in res], dtype=np.int32)
    rrec = np.ascontiguousarray([float(r) for _, r in res], dtype=np.float64)
    pct_rank = max(1, math.ceil(degrade_percentile / 100.0 * len(scores))) if len(scores) else 1
    q = _abi.EsimMissQuery(MISS_CODE[policy], int(rank), int(drop_rank_threshold), len(scores), len(res),
                           int(ladder_len), pct_rank, 0, float(gate_score), float(subst_tolerance))
    d = _abi.EsimMissDecision()
    rc = lib().esim_miss_decide(C.byref(q), scores.ctypes.data, rexp.ctypes.data, rrec.ctypes.data, C.byref(d))
    if rc != 0:
        raise RuntimeError(f"esim_miss_decide failed ({rc})")
    return d


def find_substitute(layer_residents, gate_score: float, tolerance: float):
    """The same-layer resident whose recorded score is nearest gate_score,
    within `tolerance`, ties to the lower expert; None if none qualifies
    (miss.py:66-79). Decided on the device."""
    d = _decide(SUBST, 1, 1, gate_score, tolerance, (), layer_residents, 1, 0.0)
    return int(d.substitute) if d.kind == _OUT_SUBST else None


_OUT_FETCH, _OUT_DROP, _OUT_SUBST = 0, 1, 2
_FETCH_WORKING, _FETCH_LOWEST, _FETCH_CASCADE = 0, 1, 2


def resolve_miss(cfg: MissConfig, spec, working_precision: str, rank: int, gate_score: float,
                 summed_weight: float, layer_scores, layer_residents, fetch_fn: FetchFn) -> MissOutcome:
    """Resolve one demand miss (miss.py:82-140): the policy decision on the
    device (esim_miss_decide), then the fetch through the caller's fetch_fn --
    the working precision, the lowest (fetch_low), or the ladder cascade
    (fetch_priority: non-final probes may return None, the last rung is
    final)."""
    d = _decide(cfg.policy, rank, cfg.drop_rank_threshold, gate_score, cfg.subst_tolerance, layer_scores,
                layer_residents, len(spec.precisions), cfg.degrade_percentile)
    if d.kind == _OUT_DROP:
        return MissOutcome(DROPPED, weight_delta=-summed_weight)
    if d.kind == _OUT_SUBST:
        return MissOutcome(SUBSTITUTED, weight_delta=-summed_weight, substitute=int(d.substitute))
    if d.fetch == _FETCH_LOWEST:
        return MissOutcome(FETCHED, fetch_fn(spec.lowest_precision, True), precision=spec.lowest_precision)
    if d.fetch == _FETCH_CASCADE:
        ladder = spec.precisions
        for i in range(int(d.start), len(ladder)):
            blocked = fetch_fn(ladder[i], i == len(ladder) - 1)
            if blocked is not None:
                return MissOutcome(FETCHED, blocked, precision=ladder[i])
        raise RuntimeError("fetch cascade exhausted without a forced level")
    return MissOutcome(FETCHED, fetch_fn(working_precision, True), precision=working_precision)
