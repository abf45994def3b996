"""Miss-handler plug-in surface (mirror of expertsim/miss.py:1-140).

The decision (fetch / fetch_low / fetch_priority cascade / drop:rank /
subst:tolerance) is taken by the replay kernel (csrc/replay.cu,
`resolve_miss`), with the reference's exact tie-breaks and float64
comparisons. This module keeps the config object and the names.
"""
from __future__ import annotations

from dataclasses import dataclass

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
