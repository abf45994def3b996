"""Prefetcher plug-in surface (mirror of expertsim/prefetch.py:1-221).

Prediction (topk / score-percentile / oracle over the NEXT layer's router
scores, unioned over token rows) runs inside the fused router kernel
(csrc/router.cu). The watchdog's two sweeps run inside the replay kernel
(csrc/replay.cu). Prediction noise over a whole trace runs on the device
(csrc/noise.cu: numpy's default_rng PCG64 stream restated in CUDA, drawn in
the reference's order, prefetch.py:110-136, engine.py:413, 661-666).
`apply_prediction_noise` below is the plug-in itself, for callers that hold
their own numpy Generator.
"""
from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass

import numpy as np

from .models import ConfigError

NONE = "none"
TOPK = "topk"
SCORE = "score"
ORACLE = "oracle"
PREFETCH_MODES = (NONE, TOPK, SCORE, ORACLE)
PREFETCH_CODE = {m: i for i, m in enumerate(PREFETCH_MODES)}


def nearest_rank_percentile(values, p: float) -> float:
    """Nearest-rank percentile (prefetch.py:30-36)."""
    if not 0.0 <= p < 100.0:
        raise ConfigError(f"percentile must be in [0, 100), got {p}")
    v = np.sort(np.asarray(values), kind="stable")
    return float(v[max(1, math.ceil(p / 100.0 * v.shape[0])) - 1])


def predict_event(next_logits, k: int, mode: str, overfetch: float = 1.0, percentile: float = 80.0):
    """(predictions, clamped) for one event, computed on the device."""
    if mode not in (TOPK, SCORE, ORACLE):
        raise ConfigError(f"unknown prefetch mode {mode!r}")
    if mode == TOPK and overfetch <= 0:
        raise ConfigError(f"overfetch must be positive, got {overfetch}")
    from . import _device
    return _device.predict_event(np.asarray(next_logits, dtype=np.float32), k, mode, overfetch, percentile)


def apply_prediction_noise(predictions, num_experts: int, noise: float, rng: np.random.Generator):
    """Swap each prediction for a random unchosen expert with probability
    `noise`; scores ride along; noise 0 draws nothing (prefetch.py:110-136)."""
    if noise == 0.0 or not predictions:
        return predictions
    if not 0.0 <= noise <= 1.0:
        raise ConfigError(f"prediction noise must be in [0, 1], got {noise}")
    chosen = {e for e, _ in predictions}
    out = []
    for e, s in predictions:
        if rng.random() < noise:
            pool = [x for x in range(num_experts) if x not in chosen]
            if pool:
                pick = pool[rng.integers(len(pool))]
                chosen.discard(e)
                chosen.add(pick)
                e = pick
        out.append((e, s))
    return out


@dataclass
class PrefetchRequest:
    target_layer: int
    expert: int
    score: float
    submit_us: int


class PrefetchQueue:
    """FIFO of submitted requests (prefetch.py:147-160)."""

    def __init__(self) -> None:
        self._q: deque = deque()

    def submit(self, req: PrefetchRequest) -> None:
        self._q.append(req)

    def __len__(self) -> int:
        return len(self._q)

    def pop(self) -> PrefetchRequest:
        return self._q.popleft()
