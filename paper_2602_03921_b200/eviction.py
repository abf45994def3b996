"""Eviction-policy plug-in surface (mirror of expertsim/eviction.py:1-318).

The six built-in policies are executed by the on-device directory inside
the replay kernel (csrc/replay.cu), each as an argmin over a flat per-slot
key -- no deques or ordered dicts on the device:

    lru  argmin stamp                      (stamp = counter++ on access/admit)
    lfu  argmin (count, touch, layer, e)   counts persist per (layer, expert)
    lhu  lfu counting only highest-precision accesses
    fld  argmin (-((l-c) mod L), e, l)
    sb   argmin (signal, layer, e), fp64 signal, *decay per pass
    ls   argmin gen over stale, else (forced only) over current

The policy objects below carry the name and parameters the device needs.
Custom Python subclasses cannot run on the device and are rejected by
SimConfig (the north star forbids a CPU path).
"""
from __future__ import annotations

from typing import NamedTuple

from .models import ConfigError

EVICTION_NAMES = ("lru", "lfu", "lhu", "fld", "sb", "ls")
EVICTION_CODE = {n: i for i, n in enumerate(EVICTION_NAMES)}


class AccessContext(NamedTuple):
    layer: int
    pass_id: int
    gate_score: float | None = None
    precision: str | None = None


class EvictionPolicy:
    """Descriptor of a device-executed eviction policy."""

    name = "base"

    @property
    def code(self) -> int:
        return EVICTION_CODE[self.name]


class LRUPolicy(EvictionPolicy):
    name = "lru"


class LFUPolicy(EvictionPolicy):
    name = "lfu"


class LHUPolicy(LFUPolicy):
    name = "lhu"

    def __init__(self, highest_precision: str = "fp16") -> None:
        self.highest_precision = highest_precision


class FLDPolicy(EvictionPolicy):
    name = "fld"

    def __init__(self, num_layers: int = 1) -> None:
        self.num_layers = num_layers


class SBPolicy(EvictionPolicy):
    name = "sb"

    def __init__(self, decay: float = 0.9) -> None:
        if not 0.0 < decay <= 1.0:
            raise ConfigError(f"sb decay must be in (0, 1], got {decay}")
        self.decay = decay


class LSPolicy(EvictionPolicy):
    name = "ls"


def make_eviction_policy(name: str, num_layers: int, highest_precision: str, sb_decay: float = 0.9):
    """Policy descriptor by config token (eviction.py:300-318)."""
    if name == "lhu":
        return LHUPolicy(highest_precision)
    if name == "fld":
        return FLDPolicy(num_layers)
    if name == "sb":
        return SBPolicy(sb_decay)
    simple = {"lru": LRUPolicy, "lfu": LFUPolicy, "ls": LSPolicy}.get(name)
    if simple is None:
        raise ConfigError(f"unknown eviction policy {name!r}; expected one of {', '.join(EVICTION_NAMES)}")
    return simple()
