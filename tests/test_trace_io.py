"""Trace ingestion (reference trace.py:191-279):
the native JSON-lines parser against the reference-exact reader (logits bit
for bit, every error message), its decimal -> float32 conversion against
json + numpy on adversarial inputs, the binary format, and lazily built
pass/event views. Host code only (the library loads without a GPU)."""
import json

import numpy as np
import pytest

from paper_2602_03921_b200.models import builtin_spec
from paper_2602_03921_b200.trace import (TraceFormatError, _read_jsonl_python, generate_synthetic, read_trace,
                                         write_trace, write_trace_binary)


def _bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("model,seed,pre,dec", [("olmoe", 1, 64, 64), ("mixtral", 2, 16, 8),
                                                 ("qwen15moe", 3, 300, 5), ("phi35moe", 4, 1, 0)])
def test_native_jsonl_reader_matches_reference_reader(tmp_path, model, seed, pre, dec):
    tr = generate_synthetic(builtin_spec(model), seed=seed, prefill_tokens=pre, decode_tokens=dec)
    p = tmp_path / "t.trace"
    write_trace(tr, p)
    got = read_trace(p)
    want = _read_jsonl_python(p, p.read_bytes())
    assert got.spec == want.spec and got.meta == want.meta
    assert np.array_equal(_bits(got.packed().logits), _bits(want.packed().logits))
    assert np.array_equal(got.packed().pass_tokens, want.packed().pass_tokens)
    assert np.array_equal(got.packed().pass_kind, want.packed().pass_kind)
    assert np.array_equal(got.packed().row_offset, want.packed().row_offset)
    assert np.array_equal(_bits(got.packed().logits), _bits(tr.packed().logits))      # write/read round trip
    # lazily built views behave like the reference's lists
    assert len(got.passes) == len(want.passes) == 1 + dec
    assert got.num_passes == 1 + dec and got.decode_passes == dec
    fp = got.passes[-1]
    assert fp.pass_id == dec and len(fp.events) == tr.spec.num_layers
    assert np.array_equal(fp.events[-1].logits, want.passes[-1].events[-1].logits)


def test_binary_reader_and_round_trip(tmp_path):
    tr = generate_synthetic(builtin_spec("olmoe"), seed=5, prefill_tokens=32, decode_tokens=4)
    p = tmp_path / "t.bin"
    write_trace_binary(tr, p)
    got = read_trace(p)
    assert np.array_equal(_bits(got.packed().logits), _bits(tr.packed().logits))
    assert got.meta == tr.meta and got.num_passes == 5
    raw = bytearray(p.read_bytes())
    (p.parent / "short.bin").write_bytes(bytes(raw[:-4]))
    with pytest.raises(TraceFormatError, match="logit bytes"):
        read_trace(p.parent / "short.bin")
    # a NaN in pass 2, layer 7 (row 32 + 16 + 7 of the packed matrix)
    a = np.frombuffer(bytes(raw), np.uint8)
    off = len(raw) - tr.packed().logits.nbytes
    lg = tr.packed().logits.copy()
    lg[32 * 16 + 16 + 7, 3] = np.nan
    (p.parent / "nan.bin").write_bytes(bytes(a[:off]) + lg.tobytes())
    with pytest.raises(TraceFormatError, match=r"^pass 2 layer 7: non-finite logit value$"):
        read_trace(p.parent / "nan.bin")


def _events(spec, rows_per_pass, kinds):
    rng = np.random.default_rng(0)
    out = []
    for p, (t, k) in enumerate(zip(rows_per_pass, kinds)):
        for layer in range(spec.num_layers):
            out.append({"record": "event", "pass_id": p, "kind": k, "layer": layer,
                        "logits": rng.standard_normal((t, spec.experts_per_layer)).astype(np.float32).tolist()})
    return out


def _write(path, head, events, mutate=None):
    lines = [json.dumps(head)] + [json.dumps(e) for e in events]
    if mutate:
        lines = mutate(lines)
    path.write_text("\n".join(lines) + "\n")


SPEC = builtin_spec("mixtral")
HEAD = {"record": "spec", "name": "mixtral", "num_layers": SPEC.num_layers,
        "experts_per_layer": SPEC.experts_per_layer, "top_k": SPEC.top_k,
        "expert_bytes_fp16": SPEC.expert_bytes_fp16, "precisions": list(SPEC.precisions)}


def _mut_event(i, fn):
    def m(lines):
        e = json.loads(lines[i])
        fn(e)
        lines[i] = json.dumps(e)
        return lines
    return m


BAD = {
    "bad_json": lambda lines: lines[:5] + ['{"record": "event", "pass_id": 0,'] + lines[6:],
    "unexpected_record": _mut_event(3, lambda e: e.update(record="note")),
    "wrong_layer": _mut_event(3, lambda e: e.update(layer=5)),
    "pass_gap": _mut_event(40, lambda e: e.update(pass_id=7)),
    "kind_mismatch": _mut_event(4, lambda e: e.update(kind="decode")),
    "unknown_kind": _mut_event(4, lambda e: e.update(kind="warmup")),
    "row_mismatch": _mut_event(6, lambda e: e.update(logits=e["logits"][:2])),
    "width_mismatch": _mut_event(6, lambda e: e.update(logits=[r[:7] for r in e["logits"]])),
    "nan": None,                       # built in the test: a NaN literal inside a decode row
    "infinity_literal": _mut_event(9, lambda e: e["logits"][0].__setitem__(0, float("inf"))),
    "missing_key": _mut_event(2, lambda e: e.pop("layer")),
    "string_logit": _mut_event(2, lambda e: e["logits"][0].__setitem__(1, "x")),
    "empty_logits": _mut_event(1, lambda e: e.update(logits=[])),
    "truncated": lambda lines: lines[:-3],
    "not_object": lambda lines: lines[:3] + ["[1, 2]"] + lines[4:],
    "no_events": lambda lines: lines[:1],
    "spec_not_first": lambda lines: lines[1:2] + lines[:1] + lines[2:],
    "blank_lines": lambda lines: lines[:3] + ["", "   "] + lines[3:],
    "crlf": lambda lines: [x + "\r" for x in lines],
    "float_layer": _mut_event(2, lambda e: e.update(layer=2.0)),
    "extra_key": _mut_event(2, lambda e: e.update(note=1)),
    "int_logits": _mut_event(2, lambda e: e.update(logits=[[int(v * 100) for v in r] for r in e["logits"]])),
}


@pytest.mark.parametrize("case", sorted(BAD))
def test_malformed_and_unusual_files_match_reference_reader(tmp_path, case):
    """Whatever the file, read_trace behaves exactly like the reference-exact
    reader: the same TraceFormatError text, or the same logits."""
    p = tmp_path / f"{case}.trace"
    if case == "nan":
        ev = _events(SPEC, [4, 1], ["prefill", "decode"])
        lines = [json.dumps(HEAD)] + [json.dumps(e) for e in ev]
        lines[9] = lines[9].replace("[[", "[[NaN, ", 1)
        e = json.loads(lines[9])
        e["logits"][0] = e["logits"][0][:SPEC.experts_per_layer]
        lines[9] = json.dumps(e)
        p.write_text("\n".join(lines) + "\n")
    else:
        _write(p, HEAD, _events(SPEC, [4, 1, 1], ["prefill", "decode", "decode"]), BAD[case])
    raw = p.read_bytes()
    try:
        want = _read_jsonl_python(p, raw)
        want_err = None
    except (TraceFormatError, ValueError) as exc:
        want, want_err = None, (type(exc), str(exc))
    try:
        got = read_trace(p)
        got_err = None
    except (TraceFormatError, ValueError) as exc:
        got, got_err = None, (type(exc), str(exc))
    assert got_err == want_err
    if want is not None:
        assert np.array_equal(_bits(got.packed().logits), _bits(want.packed().logits))
        assert np.array_equal(got.packed().pass_tokens, want.packed().pass_tokens)


def _parse_numbers(strs, experts=64):
    """Native parse of one event per 64 numbers; returns (native, json+numpy)."""
    import ctypes as C
    from paper_2602_03921_b200._device import lib
    L = lib()
    rows = [strs[i:i + experts] for i in range(0, len(strs) - len(strs) % experts, experts)]
    lines = ['{"record": "spec"}'] + [
        '{"record": "event", "pass_id": 0, "kind": "prefill", "layer": %d, "logits": [[%s]]}' % (i, ", ".join(r))
        for i, r in enumerate(rows)]
    raw = ("\n".join(lines) + "\n").encode()
    h, nr, npass, bad = C.c_void_p(), C.c_int64(), C.c_int32(), C.c_int64()
    rc = L.esim_trace_jsonl_parse(raw, len(raw), len(rows), experts, 0, C.byref(h), C.byref(nr), C.byref(npass),
                                  C.byref(bad))
    assert rc == 0, (rc, bad.value)
    out = np.zeros(nr.value * experts, np.float32)
    L.esim_trace_jsonl_take(h, out.ctypes.data, None, None)
    want = np.asarray([json.loads(x) for r in rows for x in r], dtype=np.float32)
    return out, want


def test_native_decimal_conversion_is_json_plus_numpy_exact():
    """decimal -> double (correctly rounded) -> float32, as json.loads +
    np.asarray(float32): writer reprs, random 1-25 digit decimals, decimals at
    and next to float32 and float64 rounding midpoints, integers, zeros."""
    from decimal import Decimal, getcontext
    getcontext().prec = 60
    rng = np.random.default_rng(7)
    n = 64 * 1500
    f = (rng.standard_normal(n) * 10 ** rng.uniform(-6, 6, n)).astype(np.float32)
    cases = [repr(float(x)) for x in f]

    def rdec():
        nd = int(rng.integers(1, 26))
        digs = "".join(str(int(d)) for d in rng.integers(0, 10, nd))
        return ("-" if rng.random() < .5 else "") + digs[0] + ("." + digs[1:] if nd > 1 else "") + \
            f"e{int(rng.integers(-48, 37))}"
    cases += [rdec() for _ in range(n)]
    a = rng.standard_normal(n // 4).astype(np.float32)
    mid = (a.astype(np.float64) + np.nextafter(a, np.float32(np.inf)).astype(np.float64)) / 2
    for i, m in enumerate(mid):
        x = (m, np.nextafter(m, np.inf), np.nextafter(m, -np.inf))[i % 3]
        cases.append(repr(float(x)) if i % 2 else "%.25g" % x)
    d = rng.standard_normal(4000)
    cases += [str((Decimal(float(x)) + Decimal(float(y))) / 2) for x, y in zip(d, np.nextafter(d, np.inf))]
    cases += [str(int(x)) for x in rng.integers(-10**15, 10**15, 640)]
    cases += ["0", "-0", "0.0", "-0.0", "1e-40", "3e-45", "1e-46", "3.4028235e38", "1E5", "2.5e+3", "00.5"[1:]] * 8
    got, want = _parse_numbers(cases)
    assert np.array_equal(_bits(got), _bits(want))
