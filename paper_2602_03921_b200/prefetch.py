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


def watchdog_step(queue: PrefetchQueue, cache, policy, channel, now_us: int, ctx, nbytes: int, precision: str,
                  evict_fn, on_start, on_skip, on_drop) -> int:
    """Drain the prefetch queue (prefetch.py:163-221), the plug-in form for
    callers with their own engine objects; inside a run the replay kernel
    executes the same two sweeps on its device directory. Sweep 1 settles
    what needs no transfer -- residents are marked prefetch-selected via
    policy.note_prefetch_hit (so a peer request of the same prediction can
    never evict them), in-flight experts are skipped; sweep 2 admits the
    rest, evicting unforced (policy.select_victim: a device-backed policy
    object, eviction.make_eviction_policy) until `nbytes` fit or dropping the
    request ("no_space"), then reserves and appends the transfer. This
    function only sequences decisions; cache, channel and the callbacks are
    the caller's. Returns the number of transfers started."""
    pending = []
    while len(queue):
        req = queue.pop()
        ident = (req.target_layer, req.expert)
        if cache.is_resident(ident):
            policy.note_prefetch_hit(ident, ctx)
            on_skip(req, "resident")
        elif channel.in_flight(ident) is not None:
            on_skip(req, "in_flight")
        else:
            pending.append(req)
    started = 0
    for req in pending:
        ident = (req.target_layer, req.expert)
        while cache.free_bytes < nbytes:
            victim = policy.select_victim(ctx, forced=False)
            if victim is None:
                on_drop(req, "no_space")
                break
            evict_fn(victim, "prefetch", False)
        else:
            cache.reserve(nbytes)
            channel.append(ident, nbytes, "prefetch", now_us, req.score, precision)
            on_start(req)
            started += 1
    return started
