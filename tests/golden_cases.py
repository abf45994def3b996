"""Load tests/golden fixtures (written by tests/golden/make_golden.py from the
real reference) and rebuild their traces/configs with this package."""
from __future__ import annotations

import gzip
import json
import os
import warnings
from functools import lru_cache

import numpy as np

from paper_2602_03921_b200.engine import SimConfig
from paper_2602_03921_b200.models import HardwareSpec, ModelSpec
from paper_2602_03921_b200.trace import ForwardPass, LayerEvent, Trace, generate_synthetic

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@lru_cache(maxsize=1)
def cases() -> list:
    with gzip.open(os.path.join(GOLDEN, "cases.json.gz"), "rt") as fh:
        return json.load(fh)


def case(name: str) -> dict:
    for c in cases():
        if c["name"] == name:
            return c
    raise KeyError(name)


def spec_from(d: dict) -> ModelSpec:
    return ModelSpec(**{**d, "precisions": tuple(d["precisions"])})


_TRACES: dict = {}


def trace_from(recipe: dict) -> Trace:
    key = json.dumps(recipe, sort_keys=True)
    if key in _TRACES:
        return _TRACES[key]
    spec = spec_from(recipe["spec"])
    if recipe["kind"] == "synthetic":
        tr = generate_synthetic(spec, **recipe["gen"])
    else:
        passes = []
        for pid, layers in enumerate(recipe["rows"]):
            kind = "prefill" if pid == 0 else "decode"
            evs = [LayerEvent(pid, kind, l, np.asarray(r, np.float32).reshape(-1, spec.experts_per_layer))
                   for l, r in enumerate(layers)]
            passes.append(ForwardPass(pid, kind, evs))
        tr = Trace(spec, passes)
        tr.validate()
    _TRACES[key] = tr
    return tr


def config_from(c: dict) -> SimConfig:
    spec = spec_from(c.get("model_override") or c["trace"]["spec"])
    cfg = dict(c["config"])
    hw = HardwareSpec(**cfg.pop("hardware"))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return SimConfig(model=spec, hardware=hw, **cfg)
