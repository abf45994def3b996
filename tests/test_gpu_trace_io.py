"""Trace files straight into HBM: binary and
JSON-lines traces loaded by load_trace_device (file -> page-locked host ->
HBM, no per-event Python objects, finite check on the device), then a C5
sweep replayed from them on the device -- every point's log digest equal to
the C oracle's on the generated traces."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_sweep_from_trace_files_matches_oracle(tmp_path):
    from oracle import oracle
    from paper_2602_03921_b200._device import load_trace_device
    from paper_2602_03921_b200.models import builtin_spec
    from paper_2602_03921_b200.sweep import C5_MODELS, DeviceSweep, c5_points
    from paper_2602_03921_b200.trace import generate_synthetic, write_trace, write_trace_binary
    gen, loaded = {}, {}
    for i, m in enumerate(C5_MODELS):
        tr = generate_synthetic(builtin_spec(m), seed=11 + i, prefill_tokens=24, decode_tokens=12)
        p = tmp_path / f"{m}.trace"
        (write_trace_binary if i % 2 else write_trace)(tr, p)
        lt = load_trace_device(p)
        assert lt._device is not None and lt.passes._src is not None       # no LayerEvent objects were built
        assert np.array_equal(lt.packed().logits.view(np.uint32), tr.packed().logits.view(np.uint32))
        gen[m], loaded[m] = [tr], [lt]
    cfgs, tl = c5_points(loaded)
    ds = DeviceSweep(cfgs, tl)
    for dt in ds.batch.dtraces.values():
        assert any(dt is t._device for t in tl)                              # the loaded HBM copy is used
    ds.step()
    got = [int(r.counters.digest) for r in ds.results()]
    gcfgs, gtl = c5_points(gen)
    want = [int(oracle.run(c, t, full_log=False).counters.digest) for c, t in zip(gcfgs, gtl)]
    assert got == want


def test_device_finite_check_names_the_event(tmp_path):
    from paper_2602_03921_b200._device import load_trace_device
    from paper_2602_03921_b200.models import builtin_spec
    from paper_2602_03921_b200.trace import TraceFormatError, generate_synthetic, write_trace_binary
    tr = generate_synthetic(builtin_spec("qwen15moe"), seed=2, prefill_tokens=16, decode_tokens=6)
    pk = tr.packed()
    L = pk.num_layers
    for (p_, layer, col, val) in ((0, 0, 0, np.inf), (3, 11, 59, np.nan), (6, L - 1, 7, -np.inf)):
        lg = pk.logits.copy()
        ev = p_ * L + layer
        lg[pk.row_offset[ev], col] = val
        t2 = generate_synthetic(builtin_spec("qwen15moe"), seed=2, prefill_tokens=16, decode_tokens=6)
        t2.packed().logits[...] = lg
        f = tmp_path / f"bad_{p_}.bin"
        write_trace_binary(t2, f)
        with pytest.raises(TraceFormatError, match=rf"^pass {p_} layer {layer}: non-finite logit value$"):
            load_trace_device(f)
