"""GPU parity: the replay + router kernels against the reference's golden
outputs (reports byte-identical) and against the C oracle (event logs
record-identical on small cases, FNV digests identical everywhere)."""
import json

import pytest

from golden_cases import cases, config_from, trace_from
from paper_2602_03921_b200.records import canon_reference_record, digest_records

pytestmark = pytest.mark.gpu

ALL = cases()
SMALL = [c for c in ALL if c["log_len"] <= 20000]
BIG = [c for c in ALL if c["log_len"] > 20000]


def _batch(cs, full_log):
    from paper_2602_03921_b200 import _device
    cfgs = [config_from(c) for c in cs]
    trs = [trace_from(c["trace"]) for c in cs]
    b = _device.ReplayBatch(cfgs, trs, full_log=full_log)
    b.launch()
    return cfgs, trs, b.results()


@pytest.mark.parametrize("chunk", range(4))
def test_small_cases_full_log_vs_reference(chunk):
    cs = SMALL[chunk::4]
    cfgs, trs, res = _batch(cs, full_log=True)
    bad = []
    for c, r in zip(cs, res):
        canon = [canon_reference_record(x) for x in r.log]
        if json.dumps(r.report) != json.dumps(c["report"]):
            bad.append((c["name"], "report"))
        if digest_records(canon) != c["log_sha256"]:
            bad.append((c["name"], "log"))
        if "log" in c and [list(t) for t in canon] != c["log"]:
            bad.append((c["name"], "records"))
        if c["ls_counters"] is not None:
            got = [r.counters.ls_forced, r.counters.ls_unforced, r.counters.ls_refusals]
            if got != c["ls_counters"]:
                bad.append((c["name"], "ls counters", got, c["ls_counters"]))
    assert not bad, bad[:8]


def test_big_cases_reports_and_digests(oracle_lib):
    cfgs, trs, res = _batch(BIG, full_log=False)
    bad = []
    for c, cfg, tr, r in zip(BIG, cfgs, trs, res):
        if json.dumps(r.report) != json.dumps(c["report"]):
            bad.append((c["name"], "report"))
        o = oracle_lib.run(cfg, tr, full_log=False)
        if o.counters.digest != r.counters.digest:
            bad.append((c["name"], "digest vs oracle"))
    assert not bad, bad[:8]


def test_device_digest_matches_oracle_on_small(oracle_lib):
    cs = SMALL[::7]
    cfgs, trs, res = _batch(cs, full_log=False)
    for c, cfg, tr, r in zip(cs, cfgs, trs, res):
        o = oracle_lib.run(cfg, tr, full_log=False)
        assert o.counters.digest == r.counters.digest, c["name"]
        assert o.counters.n_recs == r.counters.n_recs, c["name"]


def test_softmax_and_topk_plugins_bit_exact():
    import numpy as np
    from paper_2602_03921_b200 import routing
    rng = np.random.default_rng(0)
    for E in (4, 8, 16, 60, 64, 128, 200, 248, 249, 250, 251, 252, 253, 254, 255, 256):   # 249..255: numpy splits the upper half again
        x = (rng.standard_normal((33, E)) * rng.uniform(0.1, 40)).astype(np.float32)
        x[0, :] = np.round(x[0, :])
        x32 = x.astype(np.float32)
        shifted = x32 - x32.max(axis=1, keepdims=True)
        e = np.exp(shifted, dtype=np.float32)
        ref = e / e.sum(axis=1, keepdims=True, dtype=np.float32)
        got = routing.softmax_rows(x32)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), E
        for r in range(3):
            k = min(8, E)
            want = [int(i) for i in np.argsort(-ref[r], kind="stable")[:k]]
            assert routing.topk_indices(ref[r], k) == want


def test_device_sweep_batched_router_matches_oracle(oracle_lib):
    """C5 grid over two seeds through DeviceSweep (one batched router launch +
    concurrent per-model replay launches) == the oracle, point by point."""
    from paper_2602_03921_b200.models import builtin_spec
    from paper_2602_03921_b200.sweep import C5_MODELS, DeviceSweep, c5_points
    from paper_2602_03921_b200.trace import generate_synthetic
    trs = {m: [generate_synthetic(builtin_spec(m), seed=s, prefill_tokens=64, decode_tokens=16)
               for s in (3, 4)] for m in C5_MODELS}
    cfgs, tl = c5_points(trs)
    ds = DeviceSweep(cfgs, tl)
    ds.step()
    ds.step()
    res = ds.results()
    for cfg, tr, r in zip(cfgs, tl, res):
        o = oracle_lib.run(cfg, tr, full_log=False)
        assert o.counters.digest == r.counters.digest, (cfg.model.name, cfg.eviction)
        assert json.dumps(o.report) == json.dumps(r.report)


def test_c_abi_host_path_matches_oracle(oracle_lib):
    """esim_run_host (host buffers in/out, grouped concurrent replays) == oracle."""
    from paper_2602_03921_b200.models import builtin_spec
    from paper_2602_03921_b200.sweep import C5_MODELS, c5_points, reports, run_grid_host
    from paper_2602_03921_b200.trace import generate_synthetic
    trs = {m: [generate_synthetic(builtin_spec(m), seed=5, prefill_tokens=32, decode_tokens=24)] for m in C5_MODELS}
    cfgs, tl = c5_points(trs)
    # interleave models so the C side has to regroup and restore the order
    perm = sorted(range(len(cfgs)), key=lambda i: (i % 27, i // 27))
    cfgs, tl = [cfgs[i] for i in perm], [tl[i] for i in perm]
    cs, pl = run_grid_host(cfgs, tl)
    reps = reports(cfgs, cs, pl)
    for cfg, tr, c, rep in zip(cfgs, tl, cs, reps):
        o = oracle_lib.run(cfg, tr, full_log=False)
        assert o.counters.digest == c.digest, (cfg.model.name, cfg.eviction)
        assert json.dumps(o.report) == json.dumps(rep)


def test_standalone_route_event_cache_aware_matches_reference():
    import os
    import numpy as np
    from paper_2602_03921_b200.routing import DeltaAvgState, route_event
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "router_cache_aware.json")))
    for case in gold:
        delta = DeltaAvgState()
        for ev in case["events"]:
            x = np.array([[float.fromhex(v) for v in r] for r in ev["logits"]], np.float32)
            dec = route_event(x, case["k"], "cache_aware", case["lam"], set(ev["cached"]), delta, ev["layer"])
            assert [d.selected for d in dec] == ev["selected"]
            assert [d.original_selected for d in dec] == ev["original"]
            assert [[float(w).hex() for w in d.weights] for d in dec] == ev["weights"]
            assert [d.modified for d in dec] == ev["modified"]
            assert [float(delta.sums[ev["layer"]]).hex(), delta.counts[ev["layer"]]] == ev["delta"]


def test_standalone_router_kats_match_reference():
    import gzip
    import os
    import numpy as np
    from paper_2602_03921_b200.prefetch import predict_event
    from paper_2602_03921_b200.routing import DeltaAvgState, route_event, softmax_rows
    gold = json.load(gzip.open(os.path.join(os.path.dirname(__file__), "golden", "router.json.gz"), "rt"))
    for c in gold["cases"]:
        x = np.array([[float.fromhex(v) for v in r] for r in c["logits"]], np.float32)
        sm = softmax_rows(x)
        assert [[float(v).hex() for v in r] for r in sm] == c["softmax"]
        dec = route_event(x, c["k"], "standard", 0.3, set(), DeltaAvgState(), 0)
        assert [d.selected for d in dec] == c["selected"]
        for mode, kw in (("topk", {"overfetch": 1.5}), ("score", {"percentile": 80.0}), ("oracle", {}),
                         ("score0", {"percentile": 0.0})):
            p, cl = predict_event(x, c["k"], "score" if mode == "score0" else mode, **kw)
            assert [[int(a), float(b).hex()] for a, b in p] + [bool(cl)] == c["predict"][mode], mode


@pytest.mark.parametrize("experts,top_k", [(5, 2), (33, 3), (60, 4), (64, 8), (96, 6), (200, 16), (251, 8)])
def test_router_paths_by_width_match_oracle(oracle_lib, experts, top_k):
    """Every router path (single-row warp path for E <= 32 / <= 64, multi-row
    CTA path, generic E > 64 path) under every predictor mode == the oracle."""
    from paper_2602_03921_b200 import HardwareSpec, ModelSpec, SimConfig
    from paper_2602_03921_b200 import _device
    from paper_2602_03921_b200.trace import generate_synthetic
    spec = ModelSpec(f"w{experts}", num_layers=4, experts_per_layer=experts, top_k=top_k,
                     expert_bytes_fp16=1_000_000)
    tr = generate_synthetic(spec, seed=experts, prefill_tokens=70, decode_tokens=6)
    cfgs = []
    for pf, kw in (("topk", {"overfetch": 1.5}), ("score", {"percentile": 80.0}), ("score", {"percentile": 35.0}),
                   ("oracle", {}), ("none", {})):
        cfgs.append(SimConfig(model=spec, hardware=HardwareSpec(capacity_bytes=3 * experts * 250_000),
                              working_precision="int4", eviction="ls", prefetch=pf, **kw))
    b = _device.ReplayBatch(cfgs, [tr] * len(cfgs), full_log=True)
    b.launch()
    for cfg, r in zip(cfgs, b.results()):
        o = oracle_lib.run(cfg, tr, full_log=True)
        assert [canon_reference_record(x) for x in r.log] == [canon_reference_record(x) for x in o.log], cfg.prefetch
        assert json.dumps(r.report) == json.dumps(o.report)


def test_sweep_plan_full_logs_match_reference():
    """esim_sweep_plan_* with record buffers (results at the caller's rows,
    reused across runs): full event logs == the reference goldens."""
    import ctypes as C
    import numpy as np
    from paper_2602_03921_b200 import _abi
    from paper_2602_03921_b200._device import lib, rec_capacity
    from paper_2602_03921_b200.records import REC_DTYPE, decode_records
    from paper_2602_03921_b200.metrics import report_from_counters
    cs = SMALL[::11][:40] + [c for c in SMALL if c["config"].get("prefetch_noise")][::9][:12]   # noise: on the device
    cfgs = [config_from(c) for c in cs]
    trs = [trace_from(c["trace"]) for c in cs]
    descs, keep, ccfg = [], [], []
    for cfg, tr in zip(cfgs, trs):
        d, k = _abi.trace_desc_host(tr.packed())
        descs.append(d)
        keep.append(k)
        ccfg.append(cfg.to_c(len(descs) - 1, True))
    n = len(ccfg)
    L = max(c.model.num_layers for c in cfgs)
    rec_cap = max(rec_capacity(t.packed())[0] for t in trs)
    pe_cap = max(rec_capacity(t.packed())[1] for t in trs)
    carr = (_abi.EsimConfig * n)(*ccfg)
    darr = (_abi.EsimTraceDesc * n)(*descs)
    plan = C.c_void_p()
    assert lib().esim_sweep_plan_create(C.addressof(carr), n, C.addressof(darr), n, L, rec_cap, pe_cap,
                                        C.byref(plan)) == 0, lib().esim_last_error()
    try:
        for _ in range(2):                                  # the plan is reusable
            counters = (_abi.EsimCounters * n)()
            per_layer = np.zeros((n, L, _abi.ESIM_PL_FIELDS), np.int64)
            recs = np.zeros(n * rec_cap, REC_DTYPE)
            pexp = np.zeros(n * pe_cap, np.int32)
            rc = lib().esim_sweep_plan_run(plan, C.addressof(counters), per_layer.ctypes.data, recs.ctypes.data,
                                           pexp.ctypes.data)
            assert rc == 0, lib().esim_last_error()
            for i, (c, cfg) in enumerate(zip(cs, cfgs)):
                ctr = counters[i]
                log = decode_records(recs[i * rec_cap:i * rec_cap + ctr.n_recs], pexp[i * pe_cap:(i + 1) * pe_cap])
                canon = [canon_reference_record(x) for x in log]
                assert digest_records(canon) == c["log_sha256"], c["name"]
                rep = report_from_counters(cfg.echo(), cfg.model.num_layers, cfg.hardware.per_layer_compute_us, ctr,
                                           per_layer[i][:cfg.model.num_layers])
                assert json.dumps(rep) == json.dumps(c["report"]), c["name"]
    finally:
        lib().esim_sweep_plan_destroy(plan)


def test_sweep_plan_pipelined_steps_match_run(oracle_lib):
    """submit/wait over the plan's two slabs == the synchronous run, step by step."""
    from paper_2602_03921_b200.models import builtin_spec
    from paper_2602_03921_b200.sweep import C5_MODELS, HostGrid, c5_points, pin_traces
    from paper_2602_03921_b200.trace import generate_synthetic
    trs = {m: [generate_synthetic(builtin_spec(m), seed=s, prefill_tokens=16, decode_tokens=8) for s in (2, 3)]
           for m in C5_MODELS}
    cfgs, tl = c5_points(trs)
    pin_traces(tl)
    g = HostGrid(cfgs, tl)
    try:
        want = [int(c.digest) for c in g.run()[0]]
        g.submit()
        for _ in range(3):
            g.submit()
            cs, _ = g.wait()
            assert [int(c.digest) for c in cs] == want
        cs, _ = g.wait()
        assert [int(c.digest) for c in cs] == want
        o = oracle_lib.run(cfgs[5], tl[5], full_log=False)
        assert int(o.counters.digest) == want[5]
    finally:
        g.close()


def test_pinned_traces_leave_no_stale_registration(oracle_lib):
    """pin_traces + a host-API grid, then the traces and the grid go away: later
    host<->device copies into recycled host memory must keep working (a
    cudaHostRegister that outlived its array used to break them)."""
    import gc
    import numpy as np
    import torch
    from paper_2602_03921_b200.models import builtin_spec
    from paper_2602_03921_b200.sweep import C5_MODELS, c5_points, pin_traces, run_grid_host
    from paper_2602_03921_b200.trace import generate_synthetic
    trs = {m: [generate_synthetic(builtin_spec(m), seed=5, prefill_tokens=16, decode_tokens=8)] for m in C5_MODELS}
    cfgs, tl = c5_points(trs)
    pin_traces(tl)
    cs, _ = run_grid_host(cfgs, tl)
    assert all(c.status == 0 for c in cs)
    del trs, cfgs, tl, cs
    gc.collect()
    x = torch.randn(1 << 20, device="cuda")
    for n in (1 << 10, 1 << 14, 1 << 18, 1 << 20):
        for _ in range(8):
            host = [np.empty(n, np.float32) for _ in range(4)]       # recycle freed host ranges
            y = x[:n].cpu()
            assert torch.equal(y, x[:n].cpu())
            del host


NOISED = [c for c in ALL if c["config"].get("prefetch_noise") and c["config"].get("prefetch", "none") != "none"]


def test_device_noise_stream_matches_numpy_pcg64():
    """esim_noise_launch (numpy's default_rng PCG64 restated in CUDA) == the
    reference's apply_prediction_noise driven by numpy itself, prediction by
    prediction, over whole traces and several seeds / noise levels (including
    noise 1.0: every prediction draws, and seeds >= 2^32: two entropy words)."""
    import numpy as np
    import torch
    from oracle.oracle import noised_prediction_stream
    from paper_2602_03921_b200 import _device
    from paper_2602_03921_b200.models import builtin_spec
    from paper_2602_03921_b200.trace import generate_synthetic
    for model, seed, noise, mode in (("olmoe", 0, 0.3, "score"), ("qwen15moe", 7, 1.0, "topk"),
                                     ("mixtral", 2 ** 32 + 5, 0.5, "oracle"), ("olmoe", 2 ** 63 + 11, 0.05, "score")):
        tr = generate_synthetic(builtin_spec(model), seed=3, prefill_tokens=16, decode_tokens=12)
        pk = tr.packed()
        dt = _device.DeviceTrace(pk)
        ro = _device.route_trace(dt, mode, 1.5, 80.0)
        E, ne = pk.experts, pk.n_events
        n_pred = ro.t["n_pred"].cpu().numpy()[:ne].copy()
        pe = ro.t["pred_expert"].cpu().numpy()[:ne * E].reshape(ne, E).copy()
        ps = ro.t["pred_score"].cpu().numpy()[:ne * E].reshape(ne, E).copy()
        cl = ro.t["pred_clamped"].cpu().numpy()[:ne].copy()
        off = np.zeros(ne + 1, np.int32)
        np.cumsum(n_pred, out=off[1:])
        flat_e = np.concatenate([pe[i, :n_pred[i]] for i in range(ne)])
        flat_s = np.concatenate([ps[i, :n_pred[i]] for i in range(ne)])
        noff, want_e, want_s, _ = noised_prediction_stream(off, flat_e, flat_s, cl, pk.num_layers, pk.n_passes, E,
                                                           noise, seed)
        _device.apply_noise(dt, ro, mode, noise, seed)
        torch.cuda.synchronize()
        got = ro.t["pred_expert"].cpu().numpy()[:ne * E].reshape(ne, E)
        tgt = np.arange(ne) % pk.num_layers != 0
        assert np.array_equal(ro.t["n_pred"].cpu().numpy()[:ne][tgt], np.diff(noff)[tgt])
        for ev in range(ne):
            if ev % pk.num_layers == 0:
                continue                      # layer-0 targets are never predicted (engine.py:651)
            assert got[ev, :n_pred[ev]].tolist() == want_e[noff[ev]:noff[ev + 1]].tolist(), (model, ev)
        assert (got != pe).any(), "noise changed nothing"


def test_noised_golden_cases_through_every_device_entry_point():
    """The reference's prediction-noise goldens (noise 0.3, several seeds):
    byte-identical reports through the C-ABI host path (esim_run_host /
    sweep plan), DeviceSweep (batched router + device noise), and
    Simulation -- no host-prepared predictions anywhere."""
    from paper_2602_03921_b200 import Simulation
    from paper_2602_03921_b200.sweep import DeviceSweep, reports, run_grid_host
    assert len(NOISED) >= 20
    cfgs = [config_from(c) for c in NOISED]
    trs = [trace_from(c["trace"]) for c in NOISED]
    cs, pl = run_grid_host(cfgs, trs)
    for c, rep in zip(NOISED, reports(cfgs, cs, pl)):
        assert json.dumps(rep) == json.dumps(c["report"]), ("host", c["name"])
    ds = DeviceSweep(cfgs, trs)
    ds.step()
    for c, r in zip(NOISED, ds.results()):
        assert json.dumps(r.report) == json.dumps(c["report"]), ("sweep", c["name"])
    for c, cfg, tr in list(zip(NOISED, cfgs, trs))[::25]:
        assert json.dumps(Simulation(cfg, tr).run()) == json.dumps(c["report"]), ("sim", c["name"])


def test_sweep_plan_rejects_a_shared_trace_id_with_different_noise():
    import ctypes as C
    from paper_2602_03921_b200 import _abi
    from paper_2602_03921_b200._device import lib
    c = NOISED[0]
    cfg = config_from(c)
    tr = trace_from(c["trace"])
    d, keep = _abi.trace_desc_host(tr.packed())
    a, b = cfg.to_c(0, False), cfg.to_c(0, False)
    b.seed = a.seed + 1
    carr = (_abi.EsimConfig * 2)(a, b)
    darr = (_abi.EsimTraceDesc * 1)(d)
    plan = C.c_void_p()
    rc = lib().esim_sweep_plan_create(C.addressof(carr), 2, C.addressof(darr), 1, cfg.model.num_layers, 0, 0,
                                      C.byref(plan))
    assert rc == -1 and b"noise" in lib().esim_last_error()
