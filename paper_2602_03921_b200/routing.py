"""Router plug-in surface (mirror of expertsim/routing.py:1-161).

Routing math runs on the device (csrc/router.cu, csrc/numpy_f32.cuh): a
bit-exact restatement of numpy's float32 softmax followed by a stable top-k.
The host functions here keep the reference's signatures and call the CUDA
kernels through the C ABI; there is no host fallback.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .models import ConfigError

STANDARD = "standard"
CACHE_AWARE = "cache_aware"
ROUTING_CODE = {STANDARD: 0, CACHE_AWARE: 1}
LAMBDA_RANGE = (0.0, 10.0)


def validate_lambda(lam: float) -> float:
    lo, hi = LAMBDA_RANGE
    if lam < lo or lam > hi:
        raise ConfigError(f"lambda must be in [{lo}, {hi}], got {lam}")
    return lam


@dataclass
class RoutingDecision:
    """One token row's routing (routing.py:93-99)."""

    selected: list
    weights: list
    original_selected: list
    original_weights: list
    modified: bool


@dataclass
class DeltaAvgState:
    """Per-layer running mean of routed logits (routing.py:72-90); the device
    keeps the same sums in fp64 inside the replay kernel."""

    sums: dict = field(default_factory=dict)
    counts: dict = field(default_factory=dict)

    def mean(self, layer: int) -> float:
        n = self.counts.get(layer, 0)
        return self.sums.get(layer, 0.0) / n if n else 0.0


def softmax_rows(logits) -> np.ndarray:
    """Row-wise float32 softmax, computed by the device router."""
    from . import _device
    return _device.softmax(np.asarray(logits, dtype=np.float32))


def topk_indices(scores, k: int) -> list:
    """k largest, ties to the lower index, computed on the device."""
    from . import _device
    return _device.topk(np.asarray(scores, dtype=np.float32), k)


def route_event(logits, k: int, policy: str, lam: float, cached, delta: DeltaAvgState, layer: int) -> list:
    """Route all rows of one event on the device (routing.py:109-161)."""
    if policy not in ROUTING_CODE:
        raise ConfigError(f"unknown routing policy {policy!r}")
    from . import _device
    return _device.route_event(np.asarray(logits, dtype=np.float32), k, policy, lam, set(cached), delta, layer)
