"""Host-side API parity with the reference's own unit tests (restated):
config arithmetic (test_models.py), trace generation/IO (test_trace.py),
report assembly/emission (test_metrics.py), prediction noise and
percentiles (test_prefetch.py), SimConfig validation (test_engine.py)."""
import copy
import os
import csv
import json
import warnings

import numpy as np
import pytest

from paper_2602_03921_b200 import (BUILTIN_SPECS, ConfigError, ExpertKey, HardwareSpec, ModelSpec, SimConfig,
                                   TraceFormatError, builtin_spec, emit, flatten_report, generate_synthetic,
                                   load_spec_file, read_trace, resolve_capacity, transfer_us, write_trace,
                                   write_trace_binary)
from paper_2602_03921_b200.metrics import (ResidencyHistory, check_identities, classify_miss,
                                           prefetch_precision_recall)
from paper_2602_03921_b200.models import GB, MB, PRECISION_SIZE_FACTOR, sort_precisions
from paper_2602_03921_b200.prefetch import apply_prediction_noise, nearest_rank_percentile
from paper_2602_03921_b200.records import PredictionRec

from golden_cases import cases

# ---- models.py -------------------------------------------------------------


def test_precision_ladder_and_expert_bytes():
    assert PRECISION_SIZE_FACTOR == {"fp16": 1.0, "int8": 0.5, "int4": 0.25, "int2": 0.125}
    o = builtin_spec("olmoe")
    assert [o.expert_bytes(p) for p in ("fp16", "int8", "int4", "int2")] == [12 * MB, 6 * MB, 3 * MB, 1_500_000]
    assert ModelSpec("t", 1, 2, 1, 5).expert_bytes("int2") == 0
    assert o.store_bytes("int4") == 16 * 64 * 3 * MB
    assert sorted(BUILTIN_SPECS) == ["mixtral", "olmoe", "phi35moe", "qwen15moe"]
    assert sort_precisions(["int4", "fp16", "int8"]) == ("fp16", "int8", "int4")
    with pytest.raises(ConfigError, match="unknown precision"):
        sort_precisions(("fp32",))
    with pytest.raises(ConfigError, match="olmoe"):
        builtin_spec("gpt17")
    assert ExpertKey(3, 17, "int4").ident == (3, 17)


def test_model_and_hardware_validation():
    for bad in (lambda: ModelSpec("t", 0, 4, 1, MB), lambda: ModelSpec("t", 2, 4, 5, MB),
                lambda: ModelSpec("t", 2, 4, 1, 0), lambda: ModelSpec("t", 2, 4, 1, MB, precisions=()),
                lambda: HardwareSpec(), lambda: HardwareSpec(capacity_fraction=0.05, capacity_bytes=MB),
                lambda: HardwareSpec(capacity_fraction=0.0), lambda: HardwareSpec(capacity_bytes=0),
                lambda: HardwareSpec(capacity_fraction=0.05, bandwidth_bytes_per_sec=-1)):
        with pytest.raises(ConfigError):
            bad()
    with pytest.raises(ConfigError, match="not available"):
        ModelSpec("t", 2, 4, 1, MB, precisions=("int4",)).expert_bytes("fp16")


def test_capacity_and_transfer_arithmetic():
    o = builtin_spec("olmoe")
    assert resolve_capacity(o, HardwareSpec(capacity_fraction=0.05), "int4") == 153_600_000
    assert resolve_capacity(o, HardwareSpec(capacity_fraction=0.05), "fp16") // o.expert_bytes("fp16") == 51
    with pytest.raises(ConfigError, match="cannot hold"):
        resolve_capacity(o, HardwareSpec(capacity_bytes=1_499_999), "fp16")
    assert transfer_us(12_000_000, 5 * GB) == 2400
    assert transfer_us(1, 3) == 333334
    assert transfer_us(0, 5 * GB) == 0 and transfer_us(10, 0) == 0
    with pytest.raises(ValueError):
        transfer_us(-1, 1)


def test_spec_file_round_trip_and_errors(tmp_path):
    p = tmp_path / "m.spec"
    p.write_text("# comment\nname = m\nnum_layers = 3\nexperts_per_layer = 8\ntop_k = 2\n"
                 "expert_bytes_fp16 = 1000\nprecisions = int8, int4\n")
    spec = load_spec_file(p)
    assert (spec.num_layers, spec.precisions) == (3, ("int8", "int4"))
    p.write_text("name = m\nnum_layrs = 3\n")
    with pytest.raises(ConfigError, match="num_layrs"):
        load_spec_file(p)


# ---- SimConfig -------------------------------------------------------------


def test_simconfig_validation_messages():
    mini = ModelSpec("mini", 4, 8, 2, 100_000)
    hw = HardwareSpec(capacity_bytes=500_000)
    with pytest.raises(ConfigError, match="working precision"):
        SimConfig(model=ModelSpec("m", 2, 4, 1, 1000, precisions=("fp16",)), working_precision="int4")
    with pytest.raises(ConfigError, match="eviction"):
        SimConfig(model=mini, hardware=hw, eviction="belady")
    with pytest.raises(ConfigError, match="overfetch"):
        SimConfig(model=mini, hardware=hw, overfetch=0.0)
    with pytest.raises(ConfigError, match="prefetch_noise"):
        SimConfig(model=mini, hardware=hw, prefetch_noise=1.5)
    with pytest.raises(ConfigError, match="cannot hold"):
        SimConfig(model=mini, hardware=HardwareSpec(capacity_bytes=10_000))
    with pytest.warns(UserWarning, match="lhu"):
        SimConfig(model=mini, hardware=hw, eviction="lhu", miss="fetch")
    echo = SimConfig(model=mini, hardware=hw, lam=0.5).echo()
    assert json.loads(json.dumps(echo)) == echo and echo["hardware"]["resolved_capacity_bytes"] == 500_000


# ---- trace.py --------------------------------------------------------------


def test_generator_determinism_and_shape():
    spec = ModelSpec("mini", 4, 8, 2, 100_000)
    a = generate_synthetic(spec, seed=5, prefill_tokens=4, decode_tokens=6)
    b = generate_synthetic(spec, seed=5, prefill_tokens=4, decode_tokens=6)
    assert a.num_passes == 7 and a.decode_passes == 6
    assert all(np.array_equal(x.logits, y.logits) for fa, fb in zip(a.passes, b.passes)
               for x, y in zip(fa.events, fb.events))
    assert a.passes[0].events[0].logits.shape == (4, 8) and a.passes[1].events[3].logits.dtype == np.float32
    with pytest.raises(ConfigError):
        generate_synthetic(spec, seed=0, prefill_tokens=0, decode_tokens=1)


@pytest.mark.parametrize("binary", [False, True])
def test_trace_round_trip_bit_exact(tmp_path, binary):
    spec = ModelSpec("mini", 3, 6, 2, 100_000)
    tr = generate_synthetic(spec, seed=9, prefill_tokens=5, decode_tokens=4, drift=0.3, depth_bias=2.0)
    path = tmp_path / "t.trace"
    (write_trace_binary if binary else write_trace)(tr, path)
    back = read_trace(path)
    assert back.spec == tr.spec and back.meta == tr.meta
    assert np.array_equal(back.packed().logits.view(np.uint32), tr.packed().logits.view(np.uint32))


def test_trace_validation_errors(tmp_path):
    path = tmp_path / "bad.trace"
    path.write_text('{"record": "spec", "name": "m", "num_layers": 1, "experts_per_layer": 2, "top_k": 1, '
                    '"expert_bytes_fp16": 10, "precisions": ["fp16"]}\n{"record": "event", "pass_id": 0, '
                    '"kind": "warmup", "layer": 0, "logits": [[0.0, 1.0]]}\n')
    with pytest.raises(TraceFormatError, match="unknown kind"):
        read_trace(path)
    path.write_text("not json\n")
    with pytest.raises(TraceFormatError, match=":1"):
        read_trace(path)


# ---- metrics.py ------------------------------------------------------------


def test_classify_and_precision_recall():
    hist = ResidencyHistory()
    assert classify_miss((0, 1), 0, hist) == "compulsory"
    hist.note_admit((0, 1))
    hist.note_evict((0, 1), 2)
    assert classify_miss((0, 1), 2, hist) == "collision"
    assert classify_miss((0, 1), 3, hist) == "capacity"
    preds = [PredictionRec(0, 0, 1, (1, 2, 3, 4), False), PredictionRec(0, 1, 2, (5,), False)]
    out = prefetch_precision_recall(preds, {(0, 1): {1}, (0, 2): {5}})
    assert out["precision_micro"] == pytest.approx(0.4)
    assert out["precision_macro"] == pytest.approx(0.625)
    assert prefetch_precision_recall([], {})["zero_denominator"]


def _golden_report(name="mini_001"):
    return copy.deepcopy(next(c for c in cases() if c["name"] == name)["report"])


def test_check_identities_and_emit(tmp_path):
    rep = _golden_report()
    check_identities(rep)
    broken = copy.deepcopy(rep)
    broken["totals"]["hits"] += 1
    with pytest.raises(ValueError, match="identity"):
        check_identities(broken)
    written = emit(rep, "json", tmp_path / "run.json")
    assert json.loads(written[0].read_text()) == rep
    emit(rep, "csv", tmp_path / "s.csv")
    emit(_golden_report("mini_002"), "csv", tmp_path / "s.csv")
    with open(tmp_path / "s.csv", newline="") as fh:
        rows = list(csv.DictReader(fh))
    assert len(rows) == 2 and "rates.hit_rate" in rows[0]
    assert "per_layer" not in flatten_report(rep)
    with pytest.raises(ValueError, match="json or csv"):
        emit(rep, "yaml", tmp_path / "x")


# ---- prefetch.py -------------------------------------------------------------


def test_percentile_and_noise_semantics():
    scores = np.array([0.4, 0.3, 0.15, 0.1, 0.05])
    assert nearest_rank_percentile(scores, 80.0) == pytest.approx(0.3)
    assert nearest_rank_percentile(scores, 0.0) == pytest.approx(0.05)
    with pytest.raises(ConfigError):
        nearest_rank_percentile(scores, 100.0)
    rng = np.random.default_rng(0)
    preds = [(0, 0.5), (1, 0.2)]
    assert apply_prediction_noise(preds, 8, 0.0, rng) == preds
    assert rng.bit_generator.state == np.random.default_rng(0).bit_generator.state
    out = apply_prediction_noise(preds, 8, 1.0, np.random.default_rng(1))
    assert len({e for e, _ in out}) == 2 and {e for e, _ in out} != {0, 1}
    assert [s for _, s in out] == [0.5, 0.2]
    assert apply_prediction_noise([(0, 0.6), (1, 0.4)], 2, 1.0, np.random.default_rng(2)) == [(0, 0.6), (1, 0.4)]


def test_native_csv_report_matches_python_emit(tmp_path):
    """esim_report_csv (native result columns) + config columns == metrics.emit
    csv of every report, byte for byte (C5 grid, oracle results; host code only)."""
    from oracle import oracle
    from paper_2602_03921_b200.metrics import emit
    from paper_2602_03921_b200.models import builtin_spec
    from paper_2602_03921_b200.sweep import C5_MODELS, c5_points, csv_text, reports
    from paper_2602_03921_b200.trace import generate_synthetic
    trs = {m: [generate_synthetic(builtin_spec(m), seed=4, prefill_tokens=12, decode_tokens=6)] for m in C5_MODELS}
    cfgs, tl = c5_points(trs)
    ids, traces, cc = {}, [], []
    for c, t in zip(cfgs, tl):
        if id(t) not in ids:
            ids[id(t)] = len(traces)
            traces.append(t)
        cc.append(c.to_c(ids[id(t)], False))
    cs, pl = oracle.run_batch(cc, traces, 4)
    path = tmp_path / "sweep.csv"
    for rep in reports(cfgs, cs, pl):
        emit(rep, "csv", path)
    want = path.read_bytes().decode()
    assert csv_text(cfgs, cs, pl) == want


def test_native_csv_report_matches_reference_goldens(tmp_path, oracle_lib):
    """csv_text from oracle counters == metrics.emit csv of the REAL reference's
    reports (golden fixtures), over every policy / miss / routing variant."""
    import sys as _sys
    _sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from golden_cases import cases, config_from, trace_from
    from paper_2602_03921_b200.metrics import emit
    from paper_2602_03921_b200.sweep import csv_text
    cs_ = [c for c in cases() if c["log_len"] <= 20000][::13][:60]
    cfgs, counters, pls = [], [], []
    L = max(config_from(c).model.num_layers for c in cs_)
    import numpy as np
    per_layer = np.zeros((len(cs_), L, 10), np.int64)
    path = tmp_path / "golden.csv"
    for i, c in enumerate(cs_):
        cfg = config_from(c)
        o = oracle_lib.run(cfg, trace_from(c["trace"]), full_log=False)
        cfgs.append(cfg)
        counters.append(o.counters)
        per_layer[i, :cfg.model.num_layers] = o.per_layer[:cfg.model.num_layers]
        emit(c["report"], "csv", path)
    assert csv_text(cfgs, counters, per_layer) == path.read_bytes().decode()


def test_native_csv_report_rejects_broken_identities():
    """esim_report_csv refuses counters whose accounting identities do not hold
    (metrics.check_identities, metrics.py:319-336)."""
    from paper_2602_03921_b200 import SimConfig, HardwareSpec, builtin_spec, _abi
    from paper_2602_03921_b200.sweep import csv_text
    spec = builtin_spec("mixtral")
    cfg = SimConfig(model=spec, hardware=HardwareSpec(capacity_fraction=0.05), working_precision="int4")
    c = _abi.EsimCounters()
    c.totals[0] = 5          # demanded 5, nothing resolved
    with pytest.raises(ValueError):
        csv_text([cfg], [c], np.zeros((1, spec.num_layers, _abi.ESIM_PL_FIELDS), np.int64))


def test_tile_major_pack_and_quantised_decode_on_cpu():
    """Host halves of the physical expert formats (CPU): pack_expert inverts
    expert_matrices (the tile-major layout the TMA boxes read), and
    dequant_expert decodes int8 / int4 / int2 codes (int8 one per byte,
    int4 / int2 word-interleaved, two's complement) + fp32 row scales exactly
    like the device dequantisers; pack_codes is their inverse."""
    import numpy as np
    import torch
    from paper_2602_03921_b200.ffn import expert_matrices, pack_expert
    from paper_2602_03921_b200.layer_step import dequant_expert
    H, I = 256, 128
    g = torch.Generator().manual_seed(0)
    w1, wd = torch.randn(2 * I, H, generator=g), torch.randn(H, I, generator=g)
    a, b = expert_matrices(pack_expert(w1, wd, H, I), H, I)
    assert torch.equal(a, w1) and torch.equal(b, wd)
    rows = pack_expert(torch.arange(2 * I)[:, None].expand(2 * I, H),
                       (2 * I + torch.arange(H))[:, None].expand(H, I), H, I).numpy()
    rng = np.random.default_rng(1)
    nq, ns = 3 * H * I, 2 * I + H
    for bits in (8, 4, 2):
        lo, hi = -(1 << (bits - 1)), (1 << (bits - 1)) - 1
        q = rng.integers(lo, hi + 1, nq)
        sc = rng.uniform(0.01, 0.02, ns).astype(np.float32)
        if bits == 8:
            codes = q.astype(np.int8).view(np.uint8)
        else:       # independent encoding of the word-interleaved layout: element 2j -> slot j, 2j+1 -> PER/2 + j
            per = 32 // bits
            u = (q & ((1 << bits) - 1)).astype(np.uint64).reshape(-1, per)
            words = np.zeros(nq // per, np.uint64)
            for i in range(per):
                slot = i // 2 if i % 2 == 0 else per // 2 + i // 2
                words |= u[:, i] << np.uint64(bits * slot)
            codes = words.astype("<u4").view(np.uint8)
        raw = torch.from_numpy(np.concatenate([codes, sc.view(np.uint8)]))
        d1, d2 = dequant_expert(raw, bits, H, I)
        want = torch.from_numpy((q.astype(np.float32) * sc[rows]).astype(np.float32)).to(torch.bfloat16).float()
        w1w, wdw = expert_matrices(want, H, I)
        assert torch.equal(d1, w1w) and torch.equal(d2, wdw), bits
        from paper_2602_03921_b200.layer_step import pack_codes
        assert torch.equal(pack_codes(torch.from_numpy(q), bits), torch.from_numpy(codes)), bits
