"""Eviction-policy plug-in objects (mirror of expertsim/eviction.py:1-318).

Two uses:
* inside a run, SimConfig names the policy and the replay kernel executes it
  as a flat per-slot key + warp argmin (csrc/replay.cu);
* as standalone objects (`make_eviction_policy`, `LRUPolicy()`, ...), with
  the reference's methods. Each object owns a small device state; note_*
  calls are queued and flushed to a one-warp op kernel (csrc/policy.cu) with
  every select_victim, which returns the victim key. There is no host
  implementation: without a GPU the first flush raises.

Orders (all total, ties to the lower (layer, expert)):
    lru  oldest stamp            lfu  (count, last touch)     lhu  lfu counting top-precision hits
    fld  (-((l-c) mod L), e, l)  sb   (decayed gate signal)   ls   stale by generation, else
                                                                   (forced only) current
"""
from __future__ import annotations

import ctypes as C
import math
from typing import NamedTuple

import numpy as np

from .models import PRECISION_CODE, ConfigError

EVICTION_NAMES = ("lru", "lfu", "lhu", "fld", "sb", "ls")
EVICTION_CODE = {n: i for i, n in enumerate(EVICTION_NAMES)}
_OP_BEGIN, _OP_ACCESS, _OP_ADMIT, _OP_PREFETCH_HIT, _OP_SELECT = range(5)


class AccessContext(NamedTuple):
    layer: int
    pass_id: int
    gate_score: float | None = None
    precision: str | None = None


class EvictionPolicy:
    """Base class: queued ops, device state, reference method surface."""

    name = "base"

    def __init__(self) -> None:
        self._last_pass: int | None = None
        self._ops: list = []
        self._index: dict = {}
        self._keys: list = []
        self._dev = None
        self._cap = 0

    # -- reference API (eviction.py:37-62) ------------------------------------
    @property
    def code(self) -> int:
        return EVICTION_CODE[self.name]

    def begin_pass(self, pass_id: int) -> None:
        if self._last_pass is not None and pass_id <= self._last_pass:
            raise RuntimeError(f"begin_pass ids must strictly increase: {self._last_pass} -> {pass_id}")
        self._last_pass = pass_id
        self._ops.append((_OP_BEGIN, 0, 0, -1, 0, math.nan))

    def note_access(self, key, ctx: AccessContext) -> None:
        self._queue(_OP_ACCESS, key, ctx)

    def note_admit(self, key, ctx: AccessContext) -> None:
        self._queue(_OP_ADMIT, key, ctx)

    def note_prefetch_hit(self, key, ctx: AccessContext) -> None:
        self._queue(_OP_PREFETCH_HIT, key, ctx)

    def select_victim(self, ctx: AccessContext, forced: bool):
        self._ops.append((_OP_SELECT, 0, int(ctx.layer), -1, int(bool(forced)), math.nan))
        res = self._flush()
        v = int(res[-1])
        return None if v < 0 else self._keys[v]

    # -- device plumbing -------------------------------------------------------
    def _params(self) -> tuple:
        return (0, "fp16", 0.9)          # num_layers, highest precision, sb decay

    def _queue(self, op, key, ctx) -> None:
        key = (int(key[0]), int(key[1]))
        idx = self._index.get(key)
        if idx is None:
            idx = self._index[key] = len(self._keys)
            self._keys.append(key)
        gate = math.nan if ctx.gate_score is None else float(ctx.gate_score)
        prec = PRECISION_CODE.get(ctx.precision, -1) if ctx.precision is not None else -1
        self._ops.append((op, idx, int(ctx.layer), prec, 0, gate))

    def _ensure(self):
        from ._device import _torch
        torch = _torch()
        n = len(self._keys)
        if self._dev is None or n > self._cap:
            cap = max(64, 1 << max(0, n - 1).bit_length())
            new = {
                "flags": torch.zeros(cap, dtype=torch.uint8, device="cuda"),
                "key": torch.zeros(cap, dtype=torch.int64, device="cuda"),
                "count": torch.zeros(cap, dtype=torch.int32, device="cuda"),
                "signal": torch.zeros(cap, dtype=torch.float64, device="cuda"),
                "layer": torch.zeros(cap, dtype=torch.int32, device="cuda"),
                "expert": torch.zeros(cap, dtype=torch.int32, device="cuda"),
            }
            if self._dev is None:
                new["seq"] = torch.zeros(1, dtype=torch.int64, device="cuda")
                new["counters"] = torch.zeros(2, dtype=torch.int64, device="cuda")
            else:
                for k in ("flags", "key", "count", "signal", "layer", "expert"):
                    new[k][:self._cap].copy_(self._dev[k][:self._cap])
                new["seq"], new["counters"] = self._dev["seq"], self._dev["counters"]
            self._dev, self._cap = new, cap
        if n:
            ks = np.asarray(self._keys, np.int32)
            self._dev["layer"][:n].copy_(torch.from_numpy(ks[:, 0].copy()))
            self._dev["expert"][:n].copy_(torch.from_numpy(ks[:, 1].copy()))
        return torch

    def _flush(self):
        from . import _abi
        from ._device import _check, _stream, lib
        torch = self._ensure()
        L, highest, decay = self._params()
        st = _abi.EsimPolicyState(self.code, L, PRECISION_CODE[highest], len(self._keys), float(decay),
                                  *[self._dev[k].data_ptr() for k in ("seq", "counters", "flags", "key", "count",
                                                                     "signal", "layer", "expert")])
        arr = (_abi.EsimPolicyOp * len(self._ops))(*[_abi.EsimPolicyOp(o, k, l, p, f, 0, g)
                                                       for o, k, l, p, f, g in self._ops])
        d_ops = torch.frombuffer(bytearray(arr), dtype=torch.uint8).cuda()
        nsel = sum(1 for o in self._ops if o[0] == _OP_SELECT)
        res = torch.full((max(1, nsel),), -1, dtype=torch.int32, device="cuda")
        lib().esim_policy_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        _check(lib().esim_policy_apply(C.addressof(st), d_ops.data_ptr(), len(self._ops), res.data_ptr(), _stream()),
               "policy")
        self._ops = []
        return res.cpu().numpy()[:nsel]

    def _sync_state(self):
        if self._ops or self._dev is None:
            self._flush()
        return self._dev


class LRUPolicy(EvictionPolicy):
    """Evict the least recently accessed resident (eviction.py:65-87)."""
    name = "lru"


class LFUPolicy(EvictionPolicy):
    """Lowest run-lifetime access count; counts persist across evictions (eviction.py:90-129)."""
    name = "lfu"


class LHUPolicy(LFUPolicy):
    """LFU counting only accesses served at the highest precision (eviction.py:132-142)."""
    name = "lhu"

    def __init__(self, highest_precision: str = "fp16") -> None:
        super().__init__()
        self.highest_precision = highest_precision

    def _params(self):
        return (0, self.highest_precision, 0.9)


class FLDPolicy(EvictionPolicy):
    """Cyclically farthest layer ahead of the executing one (eviction.py:145-173)."""
    name = "fld"

    def __init__(self, num_layers: int = 1) -> None:
        super().__init__()
        self.num_layers = num_layers

    def _params(self):
        return (self.num_layers, "fp16", 0.9)


class SBPolicy(EvictionPolicy):
    """Lowest decayed accumulated gate score (eviction.py:176-215)."""
    name = "sb"

    def __init__(self, decay: float = 0.9) -> None:
        super().__init__()
        if not 0.0 < decay <= 1.0:
            raise ConfigError(f"sb decay must be in (0, 1], got {decay}")
        self.decay = decay

    def _params(self):
        return (0, "fp16", self.decay)


class LSPolicy(EvictionPolicy):
    """Least-Stale (eviction.py:218-294): stale residents in last-pass order,
    then (forced requests only) the current pass in touch order."""
    name = "ls"

    @property
    def forced_current_evictions(self) -> int:
        return int(self._sync_state()["counters"][0].item())

    @property
    def unforced_current_evictions(self) -> int:
        return 0                          # structural guarantee: unforced requests are refused

    @property
    def refusals(self) -> int:
        return int(self._sync_state()["counters"][1].item())

    def _sizes(self):
        f = self._sync_state()["flags"][:len(self._keys)].cpu().numpy()
        tracked = (f & 1) != 0
        cur = (f & 8) != 0
        return int((tracked & ~cur).sum()), int((tracked & cur).sum())

    def stale_size(self) -> int:
        return self._sizes()[0]

    def current_size(self) -> int:
        return self._sizes()[1]


def make_eviction_policy(name: str, num_layers: int, highest_precision: str, sb_decay: float = 0.9):
    """Policy object by config token (eviction.py:300-318)."""
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
