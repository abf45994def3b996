"""Generate golden fixtures by running the REAL reference simulator.

Run in the build container only (it imports the read-only reference from
/root/reference/pkg/src, which does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (committed, small):
  cases.json.gz   -- per case: the config, trace recipe, the reference report,
                     the sha256 digest of the canonical event log, and (for the
                     small cases) the full canonical log.
  traces.json     -- sha256 of generate_synthetic() logits for each recipe,
                     pinning this repo's generator to the reference's.
  router.json.gz  -- route/predict known-answer vectors from the reference.

The canonical record form is defined in paper_2602_03921_b200/records.py
(`canon_reference_record`), shared by the tests so both sides hash the
same tuples.
"""
from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import expertsim  # noqa: E402  (reference, read-only)
from expertsim.engine import SimConfig, Simulation  # noqa: E402
from expertsim.models import GB, HardwareSpec, ModelSpec, builtin_spec  # noqa: E402
from expertsim.trace import ForwardPass, LayerEvent, Trace, generate_synthetic  # noqa: E402
from expertsim.cli import PRESETS, build_config, DEFAULTS, _merge  # noqa: E402
from expertsim.routing import route_event, DeltaAvgState, softmax_rows  # noqa: E402
from expertsim.prefetch import predict_event  # noqa: E402

from paper_2602_03921_b200.records import canon_reference_record, digest_records  # noqa: E402

assert "/root/reference" in expertsim.__file__, expertsim.__file__


def spec_dict(spec: ModelSpec) -> dict:
    return {"name": spec.name, "num_layers": spec.num_layers,
            "experts_per_layer": spec.experts_per_layer, "top_k": spec.top_k,
            "expert_bytes_fp16": spec.expert_bytes_fp16,
            "precisions": list(spec.precisions)}


def trace_sha(trace: Trace) -> str:
    h = hashlib.sha256()
    for fp in trace.passes:
        for ev in fp.events:
            h.update(np.ascontiguousarray(ev.logits, dtype=np.float32).tobytes())
    return h.hexdigest()


HAND_ROWS = [
    [[3.0, 0, 0, 0], [0, 2.0, 0, 0]],
    [[0, 0, 4.0, 0], [0, 1.5, 0, 0]],
    [[2.5, 0, 0, 0], [0, 0, 0, 3.5]],
]


def explicit_trace(spec: ModelSpec, rows_per_pass) -> Trace:
    passes = []
    for pid, layers in enumerate(rows_per_pass):
        kind = "prefill" if pid == 0 else "decode"
        evs = [LayerEvent(pid, kind, l, np.asarray(r, np.float32).reshape(-1, spec.experts_per_layer))
               for l, r in enumerate(layers)]
        passes.append(ForwardPass(pid, kind, evs))
    t = Trace(spec, passes)
    t.validate()
    return t


def alternating_rows(num_passes=8):
    out = []
    for p in range(num_passes):
        pairs = [(0, 1), (2, 3) if p % 2 == 0 else (4, 5), (6, 7), (0, 1) if p % 2 == 0 else (2, 3)]
        layers = []
        for pair in pairs:
            v = [0.0] * 8
            v[pair[0]] = 5.0
            v[pair[1]] = 4.0
            layers.append([v])
        out.append(layers)
    return out


def make_trace(recipe: dict) -> Trace:
    spec = ModelSpec(**{**recipe["spec"], "precisions": tuple(recipe["spec"]["precisions"])})
    if recipe["kind"] == "synthetic":
        g = recipe["gen"]
        return generate_synthetic(spec, **g)
    return explicit_trace(spec, recipe["rows"])


def sim_config(spec: ModelSpec, c: dict) -> SimConfig:
    hw = HardwareSpec(**c["hardware"])
    fields = {k: v for k, v in c.items() if k not in ("hardware",)}
    return SimConfig(model=spec, hardware=hw, **fields)


def run_case(case: dict) -> dict:
    trace = make_trace(case["trace"])
    spec = trace.spec
    if "model_override" in case:
        spec = ModelSpec(**{**case["model_override"], "precisions": tuple(case["model_override"]["precisions"])})
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        cfg = sim_config(spec, case["config"])
    sim = Simulation(cfg, trace)
    report = sim.run()
    canon = [canon_reference_record(r) for r in sim.log]
    out = {"name": case["name"], "trace": case["trace"], "config": case["config"],
           "report": report, "log_sha256": digest_records(canon), "log_len": len(canon),
           "ls_counters": None}
    if "model_override" in case:
        out["model_override"] = case["model_override"]
    if cfg.eviction == "ls":
        out["ls_counters"] = [sim.policy.forced_current_evictions,
                              sim.policy.unforced_current_evictions, sim.policy.refusals]
    if case.get("full_log"):
        out["log"] = canon
    return out


def hw(capacity_bytes=None, capacity_fraction=None, bw=5 * GB, compute=2000):
    d = {"bandwidth_bytes_per_sec": bw, "per_layer_compute_us": compute}
    if capacity_bytes is not None:
        d["capacity_bytes"] = capacity_bytes
    else:
        d["capacity_fraction"] = capacity_fraction
    return d


def synth(spec, seed, prefill, decode, affinity=0.6, skew=1.0, drift=0.0, depth_bias=0.0):
    return {"kind": "synthetic", "spec": spec_dict(spec),
            "gen": {"seed": seed, "prefill_tokens": prefill, "decode_tokens": decode,
                    "affinity": affinity, "skew": skew, "drift": drift, "depth_bias": depth_bias}}


def preset_config(preset: str | None, eviction: str | None, extra: dict, spec: ModelSpec):
    """Resolve a CLI preset stack the way `expertsim sweep` does (cli.py:389-411)."""
    settings = dict(DEFAULTS)
    explicit: set = set()
    if preset:
        _merge(settings, PRESETS[preset], explicit)
    _merge(settings, extra, explicit)
    if eviction and eviction != "original":
        _merge(settings, {"eviction": eviction}, explicit)
    cfg = build_config(settings, explicit, spec)
    c = {k: getattr(cfg, k) for k in (
        "working_precision", "routing", "lam", "eviction", "sb_decay", "prefetch", "overfetch",
        "percentile", "prefetch_noise", "miss", "drop_rank_threshold", "subst_tolerance",
        "degrade_percentile", "seed")}
    h = cfg.hardware
    c["hardware"] = {"bandwidth_bytes_per_sec": h.bandwidth_bytes_per_sec,
                     "per_layer_compute_us": h.per_layer_compute_us}
    if h.capacity_bytes is not None:
        c["hardware"]["capacity_bytes"] = h.capacity_bytes
    else:
        c["hardware"]["capacity_fraction"] = h.capacity_fraction
    return c, spec_dict(cfg.model)


def build_cases() -> list[dict]:
    cases = []
    tiny = ModelSpec("tiny", 2, 4, 1, 1_000_000)
    mini = ModelSpec("mini", 4, 8, 2, 100_000)
    olmoe = builtin_spec("olmoe")
    # 1. hand walkthrough, every policy (test_engine.py:120-188)
    for ev in ("lru", "ls", "fld", "sb", "lfu", "lhu"):
        cases.append({"name": f"hand_{ev}", "full_log": True,
                      "trace": {"kind": "explicit", "spec": spec_dict(tiny), "rows": HAND_ROWS},
                      "config": {"hardware": hw(capacity_bytes=2_000_000, bw=1 * GB, compute=2000),
                                 "working_precision": "fp16", "eviction": ev, "sb_decay": 0.9,
                                 "miss": "fetch_priority" if ev == "lhu" else "fetch"}})
    # 2. alternating trace (test_acceptance.py:145-215)
    alt = ModelSpec("alt", 4, 8, 2, 1000, precisions=("fp16",))
    for ev in ("ls", "lru"):
        cases.append({"name": f"alternating_{ev}", "full_log": True,
                      "trace": {"kind": "explicit", "spec": spec_dict(alt), "rows": alternating_rows()},
                      "config": {"hardware": hw(capacity_bytes=8000, bw=1 * GB, compute=100),
                                 "eviction": ev, "seed": 0}})
    # 3. mini matrix: every policy axis on a tiny model (test_engine.py:205-225 regime)
    i = 0
    for ev in ("lru", "lfu", "lhu", "fld", "sb", "ls"):
        for pf in ({"prefetch": "none"}, {"prefetch": "topk", "overfetch": 1.5},
                   {"prefetch": "score", "percentile": 80.0}, {"prefetch": "oracle"}):
            for miss in ({"miss": "fetch"}, {"miss": "fetch_low"}, {"miss": "fetch_priority"},
                         {"miss": "drop", "drop_rank_threshold": 1}, {"miss": "subst", "subst_tolerance": 0.05}):
                for routing in ({"routing": "standard"}, {"routing": "cache_aware", "lam": 0.5}):
                    for noise in (0.0, 0.3):
                        for cap in (500_000, 150_000):
                            i += 1
                            c = {"hardware": hw(capacity_bytes=cap, bw=1 * GB, compute=100),
                                 "working_precision": "fp16", "eviction": ev, "prefetch_noise": noise,
                                 "seed": 11, **pf, **miss, **routing}
                            cases.append({"name": f"mini_{i:03d}", "full_log": (i % 16 == 1),
                                          "trace": synth(mini, 5, 4, 6), "config": c})
    # 4. mini with int8/int4/int2 ladder (test_engine.py:299-305)
    mini8 = ModelSpec("mini8", 4, 8, 2, 100_000, precisions=("int8", "int4", "int2"))
    for ev in ("lhu", "lru", "ls"):
        for miss in ("fetch", "fetch_low", "fetch_priority"):
            cases.append({"name": f"mini8_{ev}_{miss}", "full_log": False,
                          "trace": synth(mini, 5, 4, 6), "model_override": spec_dict(mini8),
                          "config": {"hardware": hw(capacity_bytes=200_000, bw=1 * GB, compute=100),
                                     "working_precision": "int8", "eviction": ev, "miss": miss,
                                     "prefetch": "topk", "overfetch": 1.0, "seed": 3}})
    # 5. OLMoE config5 vs LRU at 5% (the north-star C1 pair), both capacity forms
    for ev in ("ls", "lru"):
        for capd in ({"capacity_fraction": 0.05}, {"capacity_bytes": 614_400_000}):
            cases.append({"name": f"olmoe_c5_{ev}_{'frac' if 'capacity_fraction' in capd else 'bytes'}",
                          "trace": synth(olmoe, 1, 64, 64),
                          "config": {"hardware": {**capd, "bandwidth_bytes_per_sec": 5 * GB,
                                                  "per_layer_compute_us": 2000},
                                     "working_precision": "int4", "eviction": ev, "prefetch": "score",
                                     "percentile": 80.0, "miss": "fetch", "seed": 0}})
    # 5b. the bf16 layer-step logical config (fp16 working, 0.6 GB -> 51 slots)
    for ev in ("ls", "lru"):
        cases.append({"name": f"olmoe_layerstep_{ev}", "trace": synth(olmoe, 1, 64, 64),
                      "config": {"hardware": hw(capacity_bytes=614_400_000), "working_precision": "fp16",
                                 "eviction": ev, "prefetch": "score", "percentile": 80.0,
                                 "miss": "fetch", "seed": 0}})
    # 6. acceptance regime C1 (test_acceptance.py:55-83)
    for seed in range(1, 6):
        for ev in ("ls", "lru", "sb"):
            cases.append({"name": f"accept_c1_s{seed}_{ev}",
                          "trace": synth(olmoe, seed, 64, 64, 0.5, 0.8, 0.3, 5.0),
                          "config": {"hardware": hw(capacity_bytes=614_400_000, bw=10 * GB),
                                     "working_precision": "int4", "eviction": ev, "prefetch": "topk",
                                     "overfetch": 1.0, "miss": "fetch", "seed": seed}})
    # 7. preset stacks x {original, ls} with noise (test_acceptance.py:427-453), plus config5
    for seed in (1, 2):
        for preset in ("config1", "config2", "config3", "config4", "config5"):
            for ev in ("original", "ls"):
                c, sd = preset_config(preset, ev, {"prefetch_noise": 0.3, "seed": seed}, olmoe)
                cases.append({"name": f"preset_{preset}_{ev}_s{seed}", "trace": synth(olmoe, seed, 64, 8),
                              "model_override": sd, "config": c})
    # 8. Mixtral bandwidth-limited (C3) and Qwen subst (C4)
    mixtral, qwen, phi = builtin_spec("mixtral"), builtin_spec("qwen15moe"), builtin_spec("phi35moe")
    for cap in (0.01, 0.05, 0.25):
        for bw in (1 * GB, 5 * GB):
            for ev in ("ls", "lru"):
                cases.append({"name": f"mixtral_{ev}_{cap}_{bw // GB}g", "trace": synth(mixtral, 1, 64, 64),
                              "config": {"hardware": hw(capacity_fraction=cap, bw=bw),
                                         "working_precision": "int4", "eviction": ev, "prefetch": "score",
                                         "percentile": 80.0, "miss": "fetch", "seed": 0}})
    for cap in (0.01, 0.05, 0.25):
        for ev in ("ls", "lru", "sb"):
            cases.append({"name": f"qwen_subst_{ev}_{cap}", "trace": synth(qwen, 1, 64, 64),
                          "config": {"hardware": hw(capacity_fraction=cap),
                                     "working_precision": "int4", "eviction": ev, "prefetch": "score",
                                     "percentile": 80.0, "miss": "subst", "subst_tolerance": 0.05, "seed": 0}})
    # 9. the C5 sweep grid, in cli.py:446 product order (eviction, capacity, bandwidth), per model
    for model in (olmoe, mixtral, qwen, phi):
        for ev in ("lru", "lfu", "ls"):
            for cap in (0.01, 0.05, 0.25):
                for bw in (1 * GB, 5 * GB, 25 * GB):
                    cases.append({"name": f"sweep_{model.name}_{ev}_{cap}_{bw // GB}g",
                                  "trace": synth(model, 1, 64, 64),
                                  "config": {"hardware": hw(capacity_fraction=cap, bw=bw),
                                             "working_precision": "int4", "eviction": ev, "prefetch": "score",
                                             "percentile": 80.0, "miss": "fetch", "seed": 0}})
    return cases


def router_kats() -> dict:
    """route_event / predict_event known answers on synthetic and adversarial rows."""
    rng = np.random.default_rng(1234)
    out = []
    shapes = [(1, 64, 8), (64, 64, 8), (7, 60, 4), (3, 8, 2), (5, 16, 2), (2, 128, 8), (4, 5, 1)]
    for t, e, k in shapes:
        for trial in range(3):
            x = (rng.standard_normal((t, e)) * rng.uniform(0.1, 30.0)).astype(np.float32)
            if trial == 2:  # exact ties and repeated values
                x = np.round(x).astype(np.float32)
            sm = softmax_rows(x)
            dec = route_event(x, k, "standard", 0.3, set(), DeltaAvgState(), 0)
            preds = {}
            for mode, kw in (("topk", {"overfetch": 1.5}), ("score", {"percentile": 80.0}),
                             ("oracle", {}), ("score0", {"percentile": 0.0})):
                m = "score" if mode == "score0" else mode
                p, cl = predict_event(x, k, m, **kw)
                preds[mode] = [[int(a), float(b).hex()] for a, b in p] + [bool(cl)]
            out.append({"logits": [[float(v).hex() for v in row] for row in x], "k": k,
                        "softmax": [[float(v).hex() for v in row] for row in sm],
                        "selected": [d.selected for d in dec],
                        "weights": [[float(w).hex() for w in d.weights] for d in dec],
                        "predict": preds})
    return {"cases": out}


def main():
    cases = build_cases()
    print(f"{len(cases)} cases", flush=True)
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as pool:
        results = list(pool.map(run_case, cases, chunksize=4))
    with gzip.open(os.path.join(HERE, "cases.json.gz"), "wt") as fh:
        json.dump(results, fh, separators=(",", ":"))
    recipes = {}
    for c in cases:
        if c["trace"]["kind"] == "synthetic":
            key = json.dumps(c["trace"], sort_keys=True)
            if key not in recipes:
                recipes[key] = trace_sha(make_trace(c["trace"]))
    with open(os.path.join(HERE, "traces.json"), "w") as fh:
        json.dump([{"recipe": json.loads(k), "sha256": v} for k, v in recipes.items()], fh, indent=1)
    with gzip.open(os.path.join(HERE, "router.json.gz"), "wt") as fh:
        json.dump(router_kats(), fh, separators=(",", ":"))
    print("done")


if __name__ == "__main__":
    main()
