"""The layer-step engine: config surface + device-backed simulation.

Mirror of expertsim/engine.py's public API (SimConfig engine.py:78-185,
Simulation engine.py:382-748, run_simulation engine.py:751). A run is one
logical timeline in integer microseconds; here that timeline is executed
by the replay kernel on the B200 (csrc/replay.cu) after the fused router
kernel (csrc/router.cu) has produced the trace's routing, demand and
prediction streams. The host only validates the config, resolves it to
integers (EsimConfig), applies prediction noise (numpy PCG64, the
reference's own draw order) and formats the report.
"""
from __future__ import annotations

import warnings
from dataclasses import dataclass, field

from . import _abi
from .eviction import EVICTION_CODE, EVICTION_NAMES
from .miss import FETCH, FETCH_PRIORITY, DROP as MISS_DROP, MISS_CODE, SUBST, MissConfig
from .models import PRECISION_CODE, ConfigError, HardwareSpec, ModelSpec, resolve_capacity
from .prefetch import NONE, PREFETCH_CODE, PREFETCH_MODES
from .routing import CACHE_AWARE, ROUTING_CODE, STANDARD, validate_lambda

DEMAND = "demand"
PREFETCH = "prefetch"


@dataclass(frozen=True)
class SimConfig:
    """Everything one run depends on except the trace (engine.py:78-185)."""

    model: ModelSpec
    hardware: HardwareSpec = HardwareSpec(capacity_fraction=0.05)
    working_precision: str = "fp16"
    routing: str = STANDARD
    lam: float = 0.3
    eviction: str = "lru"
    sb_decay: float = 0.9
    prefetch: str = NONE
    overfetch: float = 1.0
    percentile: float = 80.0
    prefetch_noise: float = 0.0
    miss: str = FETCH
    drop_rank_threshold: int = 2
    subst_tolerance: float = 0.05
    degrade_percentile: float = 60.0
    seed: int = 0

    def __post_init__(self) -> None:
        if self.working_precision not in self.model.precisions:
            raise ConfigError(f"working precision {self.working_precision!r} not in model "
                              f"precisions {self.model.precisions}")
        if self.routing not in (STANDARD, CACHE_AWARE):
            raise ConfigError(f"unknown routing policy {self.routing!r}")
        validate_lambda(self.lam)
        if self.eviction not in EVICTION_NAMES:
            raise ConfigError(f"unknown eviction policy {self.eviction!r}; "
                              f"expected one of {', '.join(EVICTION_NAMES)}")
        if self.prefetch not in PREFETCH_MODES:
            raise ConfigError(f"unknown prefetch mode {self.prefetch!r}; "
                              f"expected one of {', '.join(PREFETCH_MODES)}")
        if self.overfetch <= 0:
            raise ConfigError(f"overfetch must be positive, got {self.overfetch}")
        if not 0.0 <= self.percentile < 100.0:
            raise ConfigError(f"percentile must be in [0, 100), got {self.percentile}")
        if not 0.0 <= self.prefetch_noise <= 1.0:
            raise ConfigError(f"prefetch_noise must be in [0, 1], got {self.prefetch_noise}")
        self.miss_config()
        capacity = self.capacity_bytes()
        need = self.model.expert_bytes(self.working_precision)
        if self.miss in (FETCH, MISS_DROP, SUBST) and capacity < need:
            raise ConfigError(f"capacity {capacity} B cannot hold one {self.working_precision} "
                              f"expert ({need} B) required by miss policy {self.miss!r}")
        if self.model.experts_per_layer > _abi.ESIM_MAX_E or self.model.top_k > _abi.ESIM_MAX_K:
            raise ConfigError(f"device path supports E <= {_abi.ESIM_MAX_E}, k <= {_abi.ESIM_MAX_K}")
        if self.eviction == "lhu" and self.miss != FETCH_PRIORITY:
            warnings.warn("lhu eviction tracks precision levels and is intended to pair "
                          "with miss=fetch_priority", stacklevel=2)

    def miss_config(self) -> MissConfig:
        return MissConfig(self.miss, self.drop_rank_threshold, self.subst_tolerance, self.degrade_percentile)

    def capacity_bytes(self) -> int:
        return resolve_capacity(self.model, self.hardware, self.working_precision)

    def echo(self) -> dict:
        """Stable-order config echo embedded in every report (engine.py:152-185)."""
        m, hw = self.model, self.hardware
        return {
            "model": {"name": m.name, "num_layers": m.num_layers, "experts_per_layer": m.experts_per_layer,
                      "top_k": m.top_k, "expert_bytes_fp16": m.expert_bytes_fp16,
                      "precisions": list(m.precisions)},
            "hardware": {"capacity_fraction": hw.capacity_fraction, "capacity_bytes": hw.capacity_bytes,
                         "resolved_capacity_bytes": self.capacity_bytes(),
                         "bandwidth_bytes_per_sec": hw.bandwidth_bytes_per_sec,
                         "per_layer_compute_us": hw.per_layer_compute_us},
            "working_precision": self.working_precision, "routing": self.routing, "lambda": self.lam,
            "eviction": self.eviction, "sb_decay": self.sb_decay, "prefetch": self.prefetch,
            "overfetch": self.overfetch, "percentile": self.percentile,
            "prefetch_noise": self.prefetch_noise, "miss": self.miss,
            "drop_rank_threshold": self.drop_rank_threshold, "subst_tolerance": self.subst_tolerance,
            "degrade_percentile": self.degrade_percentile, "seed": self.seed,
        }

    def to_c(self, trace_id: int = 0, full_log: bool = False) -> _abi.EsimConfig:
        """Resolve to the device's integer config (EsimConfig)."""
        m = self.model
        c = _abi.EsimConfig()
        c.num_layers, c.experts, c.top_k = m.num_layers, m.experts_per_layer, m.top_k
        c.n_precisions = len(m.precisions)
        for i, p in enumerate(m.precisions):
            c.precisions[i] = PRECISION_CODE[p]
            c.expert_bytes[PRECISION_CODE[p]] = m.expert_bytes(p)
        c.capacity_bytes = self.capacity_bytes()
        c.bandwidth = self.hardware.bandwidth_bytes_per_sec
        c.compute_us = self.hardware.per_layer_compute_us
        c.working_prec = PRECISION_CODE[self.working_precision]
        c.routing = ROUTING_CODE[self.routing]
        c.lam = self.lam
        c.eviction = EVICTION_CODE[self.eviction]
        c.prefetch = PREFETCH_CODE[self.prefetch]
        c.sb_decay, c.overfetch, c.percentile = self.sb_decay, self.overfetch, self.percentile
        c.miss = MISS_CODE[self.miss]
        c.drop_rank_threshold = self.drop_rank_threshold
        c.subst_tolerance, c.degrade_percentile = self.subst_tolerance, self.degrade_percentile
        c.flags = _abi.ESIM_FLAG_FULL_LOG if full_log else 0
        c.trace_id = trace_id
        # noise is only drawn when something is predicted (engine.py:651-666)
        c.prefetch_noise = self.prefetch_noise if self.prefetch != "none" else 0.0
        c.seed = self.seed if c.prefetch_noise > 0 else 0
        return c


def check_geometry(config: SimConfig, trace) -> None:
    s, m = trace.spec, config.model
    if (s.num_layers, s.experts_per_layer, s.top_k) != (m.num_layers, m.experts_per_layer, m.top_k):
        raise ConfigError(
            f"trace geometry (L={s.num_layers}, E={s.experts_per_layer}, k={s.top_k}) does not "
            f"match the model (L={m.num_layers}, E={m.experts_per_layer}, k={m.top_k})")
    if trace.num_passes * s.num_layers * s.experts_per_layer >= 2**31:
        raise ConfigError("trace too long for the device replay: passes x layers x experts must be < 2^31")


@dataclass
class PolicyStats:
    """LS structural counters the reference exposes on `Simulation.policy`
    (eviction.py:240-243)."""

    name: str
    forced_current_evictions: int = 0
    unforced_current_evictions: int = 0
    refusals: int = 0


@dataclass
class Simulation:
    """One deterministic run of a config over a trace, executed on the GPU.

    `run()` returns the reference-format report; `log` then holds the full
    decoded event log (the parity artefact)."""

    cfg: SimConfig
    trace: object
    full_log: bool = True
    log: list = field(default_factory=list)
    counters: object = None

    def __init__(self, config: SimConfig, trace, full_log: bool = True) -> None:
        check_geometry(config, trace)
        if config.eviction == "sb" and not 0.0 < config.sb_decay <= 1.0:
            raise ConfigError(f"sb decay must be in (0, 1], got {config.sb_decay}")
        self.cfg, self.trace, self.full_log = config, trace, full_log
        self.log = []
        self.counters = None
        self.policy = PolicyStats(config.eviction)
        self.spec = config.model

    def run(self) -> dict:
        from . import _device
        res = _device.run_simulations([self.cfg], [self.trace], full_log=self.full_log)[0]
        self.log = res.log
        self.counters = res.counters
        self.policy.forced_current_evictions = int(res.counters.ls_forced)
        self.policy.unforced_current_evictions = int(res.counters.ls_unforced)
        self.policy.refusals = int(res.counters.ls_refusals)
        return res.report


def run_simulation(config: SimConfig, trace) -> dict:
    """Run one config over one trace on the device; return the report."""
    return Simulation(config, trace, full_log=False).run()
