"""Randomised parity: seeded random model geometries, traces and configs --
every policy axis, capacities from one expert to most of the store,
bandwidths from free (0) to slow, compute 0..5000 us, prediction noise,
cache-aware routing -- replayed on the device in one batch (the sweep's
persistent common-path kernels and the general-path kernels) and through
the C-ABI sweep plan, against the C oracle: counters, per-layer rows and
event-log digests identical, full logs record-identical on a subset."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _random_cases(n, seed):
    from paper_2602_03921_b200 import HardwareSpec, ModelSpec, SimConfig, generate_synthetic
    import warnings
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        L = int(rng.integers(2, 9))
        E = int(rng.choice([4, 8, 16, 32, 60, 64]))
        k = int(rng.integers(1, min(E, 8) + 1))
        ladder = [("fp16", "int8", "int4", "int2"), ("fp16", "int8", "int4"), ("int8", "int4", "int2"), ("fp16",)]
        prec = ladder[int(rng.integers(0, len(ladder)))]
        spec = ModelSpec(f"fz{i}", L, E, k, int(rng.choice([1_000_000, 12_000_000, 3_000_000])), precisions=prec)
        tr = generate_synthetic(spec, seed=int(rng.integers(0, 1 << 30)), prefill_tokens=int(rng.integers(1, 40)),
                                decode_tokens=int(rng.integers(0, 12)), affinity=float(rng.uniform(0, 1)),
                                skew=float(rng.uniform(0.2, 2.5)), drift=float(rng.choice([0.0, 0.2])),
                                depth_bias=float(rng.choice([0.0, 3.0])))
        working = prec[int(rng.integers(0, len(prec)))]
        nb = spec.expert_bytes(working)
        cap = int(nb * rng.uniform(1.0, 0.8 * L * E))
        miss = str(rng.choice(["fetch", "fetch", "fetch", "fetch_low", "fetch_priority", "drop", "subst"]))
        pf = str(rng.choice(["none", "topk", "score", "score", "oracle"]))
        kw = dict(working_precision=working, eviction=str(rng.choice(["lru", "lfu", "lhu", "fld", "sb", "ls"])),
                  prefetch=pf, miss=miss, seed=int(rng.integers(0, 100)))
        if pf == "topk":
            kw["overfetch"] = float(rng.choice([1.0, 1.5, 2.0]))
        if pf == "score":
            kw["percentile"] = float(rng.choice([50.0, 80.0, 95.0]))
        if pf != "none" and rng.random() < 0.3:
            kw["prefetch_noise"] = float(rng.choice([0.1, 0.5]))
        if rng.random() < 0.3:
            kw.update(routing="cache_aware", lam=float(rng.uniform(0, 2)))
        if miss == "drop":
            kw["drop_rank_threshold"] = int(rng.integers(1, k + 1))
        if miss == "subst":
            kw["subst_tolerance"] = float(rng.choice([0.01, 0.05, 0.2]))
        if miss == "fetch_priority":
            kw["degrade_percentile"] = float(rng.choice([30.0, 60.0]))
        hw = HardwareSpec(capacity_bytes=cap, bandwidth_bytes_per_sec=int(rng.choice([0, 10**8, 10**9, 5 * 10**9])),
                          per_layer_compute_us=int(rng.choice([0, 100, 2000, 5000])))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            try:
                cfg = SimConfig(model=spec, hardware=hw, **kw)
            except Exception:
                continue                     # invalid combination (the reference rejects it too)
        out.append((cfg, tr))
    return out


@pytest.mark.parametrize("seed", [101, 202, 404])
def test_random_configs_device_vs_oracle(seed, oracle_lib):
    from paper_2602_03921_b200 import _device
    from paper_2602_03921_b200.records import canon_reference_record
    cases = _random_cases(400, seed)
    assert len(cases) > 300
    cfgs, trs = [c for c, _ in cases], [t for _, t in cases]
    res = _device.run_simulations(cfgs, trs)
    bad = []
    for i, (cfg, tr, r) in enumerate(zip(cfgs, trs, res)):
        o = oracle_lib.run(cfg, tr, full_log=i % 8 == 0)
        if int(o.counters.digest) != int(r.counters.digest):
            bad.append((i, "digest", cfg.eviction, cfg.miss, cfg.prefetch, cfg.routing))
        if list(o.counters.totals) != list(r.counters.totals):
            bad.append((i, "totals"))
        if not np.array_equal(np.asarray(o.per_layer)[:, :8], np.asarray(r.per_layer)[:, :8]):
            bad.append((i, "per-layer"))
    assert not bad, bad[:10]
    # a subset with full logs on the device: record for record
    sub = list(range(0, len(cfgs), 8))
    full = _device.run_simulations([cfgs[i] for i in sub], [trs[i] for i in sub], full_log=True)
    for j, i in enumerate(sub):
        o = oracle_lib.run(cfgs[i], trs[i], full_log=True)
        assert [canon_reference_record(x) for x in full[j].log] == [canon_reference_record(x) for x in o.log], i


def test_random_configs_through_the_c_abi_plan(oracle_lib):
    from paper_2602_03921_b200.sweep import run_grid_host
    cases = _random_cases(300, 303)
    cfgs, trs = [c for c, _ in cases], [t for _, t in cases]
    cs, _ = run_grid_host(cfgs, trs)
    want = [int(oracle_lib.run(c, t, full_log=False).counters.digest) for c, t in cases]
    assert [int(c.digest) for c in cs] == want
