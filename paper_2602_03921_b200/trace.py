"""Routing traces: the input of the layer step.

API mirror of expertsim/trace.py (trace.py:1-279). The synthetic generator
draws the identical numpy PCG64 stream in the identical order as the
reference (trace.py:147-188) -- pinned by tests/golden/traces.json -- but
draws each pass's noise in one call and keeps the whole trace as one packed
float32 matrix, which is the layout the device consumes:

    row_offset[ev] .. row_offset[ev+1]   token rows of event ev = pass*L + layer
    logits[row][expert]                  float32, row-major

`Trace.packed()` returns that layout; `LayerEvent.logits` are views into it.
Besides the reference's JSON-lines format this module reads and writes a
binary format (magic b"ESIMTRC1": header JSON + raw float32), which loads
without parsing text.
"""
from __future__ import annotations

import json
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .models import ConfigError, ModelSpec

PREFILL = "prefill"
DECODE = "decode"
_BIN_MAGIC = b"ESIMTRC1"


class TraceFormatError(ValueError):
    """A trace file is malformed or inconsistent (trace.py:25-26)."""


@dataclass
class LayerEvent:
    pass_id: int
    kind: str
    layer: int
    logits: np.ndarray  # float32 (tokens, experts)

    @property
    def tokens(self) -> int:
        return self.logits.shape[0]


@dataclass
class ForwardPass:
    pass_id: int
    kind: str
    events: list


@dataclass
class PackedTrace:
    """Contiguous arrays handed to the C ABI (EsimTraceDesc)."""

    num_layers: int
    experts: int
    top_k: int
    pass_tokens: np.ndarray   # int32 [P]
    pass_kind: np.ndarray     # int32 [P] 0 prefill / 1 decode
    row_offset: np.ndarray    # int64 [P*L + 1]
    logits: np.ndarray        # float32 [rows, E]

    @property
    def n_passes(self) -> int:
        return int(self.pass_tokens.shape[0])

    @property
    def n_events(self) -> int:
        return self.n_passes * self.num_layers


@dataclass
class Trace:
    spec: ModelSpec
    passes: list
    meta: dict = field(default_factory=dict)
    _packed: PackedTrace | None = field(default=None, repr=False, compare=False)

    @property
    def num_passes(self) -> int:
        return len(self.passes)

    @property
    def decode_passes(self) -> int:
        return sum(fp.kind == DECODE for fp in self.passes)

    def validate(self) -> None:
        """Structural checks; messages name the pass/layer (trace.py:62-95)."""
        L, E = self.spec.num_layers, self.spec.experts_per_layer
        if isinstance(self.passes, _LazyPasses) and self.passes._src is not None:
            # packed layout: structure holds by construction; check the values
            # in one vectorised pass and name the first bad event like the loop
            pk = self._packed
            if pk is not None and (pk.pass_tokens <= 0).any():
                p = int(np.argmax(pk.pass_tokens <= 0))
                raise TraceFormatError(f"pass {p} layer 0: empty logits matrix")
            if pk is not None and pk.logits.size and not np.isfinite(pk.logits).all():
                raise TraceFormatError(_nonfinite_where(pk, int(np.argmax((~np.isfinite(pk.logits)).any(axis=1)))))
            return
        for want, fp in enumerate(self.passes):
            if fp.pass_id != want:
                raise TraceFormatError(f"pass {fp.pass_id}: expected pass_id {want}")
            if len(fp.events) != L:
                raise TraceFormatError(
                    f"pass {fp.pass_id}: has {len(fp.events)} layer events, expected {L}")
            rows0 = fp.events[0].tokens if fp.events else 0
            for layer, ev in enumerate(fp.events):
                where = f"pass {fp.pass_id} layer {ev.layer}"
                if ev.layer != layer:
                    raise TraceFormatError(f"pass {fp.pass_id}: expected layer {layer}, got {ev.layer}")
                if ev.kind != fp.kind:
                    raise TraceFormatError(f"{where}: kind {ev.kind!r} != pass kind {fp.kind!r}")
                if ev.logits.ndim != 2 or ev.logits.shape[1] != E:
                    raise TraceFormatError(
                        f"{where}: logits shape {ev.logits.shape} does not match {E} experts")
                if ev.tokens != rows0:
                    raise TraceFormatError(f"{where}: {ev.tokens} token rows, pass started with {rows0}")
                if ev.tokens == 0:
                    raise TraceFormatError(f"{where}: empty logits matrix")
                if not np.isfinite(ev.logits).all():
                    raise TraceFormatError(f"{where}: non-finite logit value")

    def packed(self) -> PackedTrace:
        if self._packed is None:
            L = self.spec.num_layers
            toks = np.array([fp.events[0].tokens for fp in self.passes], np.int32)
            kinds = np.array([0 if fp.kind == PREFILL else 1 for fp in self.passes], np.int32)
            per_event = np.repeat(toks.astype(np.int64), L)
            off = np.zeros(per_event.shape[0] + 1, np.int64)
            np.cumsum(per_event, out=off[1:])
            mats = [np.ascontiguousarray(ev.logits, np.float32) for fp in self.passes for ev in fp.events]
            logits = np.concatenate(mats, axis=0) if mats else np.zeros((0, self.spec.experts_per_layer), np.float32)
            self._packed = PackedTrace(L, self.spec.experts_per_layer, self.spec.top_k, toks, kinds, off,
                                       np.ascontiguousarray(logits))
        return self._packed


class _LazyPasses(list):
    """Trace.passes of a packed trace: the ForwardPass / LayerEvent view
    objects are built on first use (the device path never needs them; a
    C5 sweep trace would otherwise carry 65 x L Python objects)."""

    def __init__(self, spec: ModelSpec, toks, kinds, logits: np.ndarray):
        super().__init__()
        self._src = (spec, list(toks), list(kinds), logits)

    def _build(self):
        if self._src is None:
            return
        spec, toks, kinds, logits = self._src
        self._src = None
        L, row = spec.num_layers, 0
        for p, (t, k) in enumerate(zip(toks, kinds)):
            kind = PREFILL if k == 0 else DECODE
            events = []
            for layer in range(L):
                events.append(LayerEvent(p, kind, layer, logits[row:row + t]))
                row += t
            list.append(self, ForwardPass(p, kind, events))

    def __len__(self):
        return len(self._src[1]) if self._src is not None else list.__len__(self)


def _lazy_method(name):
    def m(self, *a, **k):
        self._build()
        return getattr(list, name)(self, *a, **k)
    m.__name__ = name
    return m


for _n in ("__getitem__", "__iter__", "__reversed__", "__contains__", "__eq__", "__repr__", "index", "count",
           "append", "extend", "insert", "pop", "remove", "__setitem__", "__delitem__", "copy", "__add__",
           "__iadd__", "__mul__", "sort", "reverse", "clear"):
    setattr(_LazyPasses, _n, _lazy_method(_n))


def _from_packed(spec: ModelSpec, toks, kinds, logits: np.ndarray, meta: dict) -> Trace:
    L = spec.num_layers
    tr = Trace(spec, _LazyPasses(spec, toks, kinds, logits), meta)
    per_event = np.repeat(np.asarray(toks, np.int64), L)
    off = np.zeros(per_event.shape[0] + 1, np.int64)
    np.cumsum(per_event, out=off[1:])
    tr._packed = PackedTrace(L, spec.experts_per_layer, spec.top_k, np.asarray(toks, np.int32),
                             np.asarray(kinds, np.int32), off, logits)
    return tr


def _nonfinite_where(pk: PackedTrace, row: int) -> str:
    """trace.py:94-95's message for the event holding packed row `row`."""
    ev = int(np.searchsorted(pk.row_offset, row, side="right")) - 1
    return f"pass {ev // pk.num_layers} layer {ev % pk.num_layers}: non-finite logit value"


def generate_synthetic(spec: ModelSpec, seed: int, prefill_tokens: int, decode_tokens: int,
                       affinity: float = 0.6, skew: float = 1.0, drift: float = 0.0,
                       depth_bias: float = 0.0) -> Trace:
    """Synthetic routing trace, draw-for-draw identical to trace.py:98-188.

    base ~ N(0,1)*skew per layer; token deviation AR(1):
    dev = affinity*dev + (1-affinity)*eps; optional per-pass drift of the
    base; geometric depth temperature (1+depth_bias)**(1 - 2l/(L-1)).
    """
    for bad, msg in ((prefill_tokens < 1, "prefill_tokens must be >= 1"),
                     (decode_tokens < 0, "decode_tokens must be >= 0"),
                     (not 0.0 <= affinity <= 1.0, "affinity must be in [0, 1]"),
                     (skew < 0.0, "skew must be >= 0"), (drift < 0.0, "drift must be >= 0"),
                     (depth_bias < 0.0, "depth_bias must be >= 0")):
        if bad:
            raise ConfigError(msg)
    L, E = spec.num_layers, spec.experts_per_layer
    gen = np.random.default_rng(seed)
    base = gen.standard_normal((L, E)) * skew
    dev = np.zeros((L, E))
    expo = 1.0 - 2.0 * np.arange(L) / (L - 1) if L > 1 else np.zeros(1)
    scale = ((1.0 + depth_bias) ** expo)[:, None]
    token_counts = [prefill_tokens] + [1] * decode_tokens
    total_rows = sum(token_counts) * L
    logits = np.empty((total_rows, E), np.float32)
    row = 0
    a, b = affinity, 1.0 - affinity
    for p, t in enumerate(token_counts):
        if p > 0 and drift > 0.0:
            base = base + drift * gen.standard_normal((L, E))
        eps = gen.standard_normal((t, L, E))        # == t successive (L, E) draws
        block = np.empty((L, t, E))
        for j in range(t):
            dev = a * dev + b * eps[j]
            block[:, j, :] = (base + dev) * scale
        logits[row:row + L * t] = block.reshape(L * t, E).astype(np.float32)
        row += L * t
    kinds = [0] + [1] * decode_tokens
    meta = {"generator": {"seed": seed, "prefill_tokens": prefill_tokens, "decode_tokens": decode_tokens,
                          "affinity": affinity, "skew": skew, "drift": drift, "depth_bias": depth_bias}}
    tr = _from_packed(spec, token_counts, kinds, logits, meta)
    tr.validate()
    return tr


def _spec_header(spec: ModelSpec) -> dict:
    return {"record": "spec", "name": spec.name, "num_layers": spec.num_layers,
            "experts_per_layer": spec.experts_per_layer, "top_k": spec.top_k,
            "expert_bytes_fp16": spec.expert_bytes_fp16, "precisions": list(spec.precisions)}


def write_trace(trace: Trace, path) -> None:
    """Reference JSON-lines format (trace.py:191-216)."""
    head = _spec_header(trace.spec)
    if trace.meta:
        head["meta"] = trace.meta
    lines = [json.dumps(head)]
    for fp in trace.passes:
        for ev in fp.events:
            lines.append(json.dumps({"record": "event", "pass_id": ev.pass_id, "kind": ev.kind,
                                     "layer": ev.layer, "logits": ev.logits.tolist()}))
    Path(path).write_text("\n".join(lines) + "\n")


def write_trace_binary(trace: Trace, path) -> None:
    """Binary format: magic, u64 header length, header JSON, raw float32 logits."""
    pk = trace.packed()
    head = _spec_header(trace.spec)
    head.update(meta=trace.meta, pass_tokens=pk.pass_tokens.tolist(), pass_kind=pk.pass_kind.tolist())
    hb = json.dumps(head).encode()
    with open(path, "wb") as fh:
        fh.write(_BIN_MAGIC + struct.pack("<Q", len(hb)) + hb)
        fh.write(np.ascontiguousarray(pk.logits, "<f4").tobytes())


def _spec_from_header(path, header: dict) -> ModelSpec:
    try:
        return ModelSpec(name=str(header["name"]), num_layers=int(header["num_layers"]),
                         experts_per_layer=int(header["experts_per_layer"]), top_k=int(header["top_k"]),
                         expert_bytes_fp16=int(header["expert_bytes_fp16"]),
                         precisions=tuple(header["precisions"]))
    except KeyError as exc:
        raise TraceFormatError(f"{path}:1: spec record missing {exc}") from None
    except ConfigError as exc:
        raise TraceFormatError(f"{path}:1: bad spec record: {exc}") from None


def _alloc_rows(rows: int, experts: int, alloc):
    """float32 [rows, experts] from `alloc(nbytes) -> writable uint8 buffer`
    (e.g. page-locked memory) or plain numpy."""
    if alloc is None:
        return np.empty((rows, experts), np.float32)
    buf = alloc(rows * experts * 4)
    return np.frombuffer(buf, np.float32, count=rows * experts).reshape(rows, experts)


def read_trace(path, alloc=None, check_values: bool = True) -> Trace:
    """Read either format; errors name file and line / pass and layer (trace.py:219-279).

    JSON lines: the spec line is parsed here, the event lines by the native
    parallel parser (esim_trace_jsonl_parse) straight into the packed float32
    matrix -- bit-identical to json.loads + np.asarray(float32); a file the
    fast parser refuses is re-read by the reference-exact reader below, which
    raises the reference's TraceFormatError. Binary: the logits are read from
    the file straight into the packed matrix. `alloc` places that matrix
    (e.g. pinned host memory for the H2D path, see load_trace_device);
    check_values=False leaves the binary format's finite-value check to the
    caller (the device path checks in HBM)."""
    path = Path(path)
    with open(path, "rb") as fh:
        magic = fh.read(len(_BIN_MAGIC))
        if magic == _BIN_MAGIC:
            (hl,) = struct.unpack("<Q", fh.read(8))
            head = json.loads(fh.read(hl))
            spec = _spec_from_header(path, head)
            toks = np.asarray(head["pass_tokens"], np.int32)
            rows = int(toks.astype(np.int64).sum()) * spec.num_layers
            logits = _alloc_rows(rows, spec.experts_per_layer, alloc)
            got = fh.readinto(memoryview(logits.reshape(-1).view(np.uint8)))   # file -> destination, no copy
            if got != logits.nbytes or fh.read(1):
                raise TraceFormatError(f"{path}: binary trace holds {got} logit bytes, header implies "
                                       f"{logits.nbytes}")
            tr = _from_packed(spec, toks, head["pass_kind"], logits, head.get("meta", {}))
            if check_values:
                tr.validate()
            elif (toks <= 0).any():
                tr.validate()
            return tr
        raw = magic + fh.read()
    fast = _read_jsonl_native(path, raw, alloc)
    if fast is not None:
        return fast
    return _read_jsonl_python(path, raw)


def _read_jsonl_python(path, raw: bytes) -> Trace:
    """The reference-exact JSON-lines reader (trace.py:219-279): every error
    message, and the files the native parser hands back."""
    path = Path(path)
    lines = raw.decode().splitlines()
    if not lines:
        raise TraceFormatError(f"{path}: empty trace file")

    def record(lineno: int, text: str) -> dict:
        try:
            obj = json.loads(text)
        except json.JSONDecodeError as exc:
            raise TraceFormatError(f"{path}:{lineno}: invalid JSON: {exc}") from None
        if not isinstance(obj, dict) or "record" not in obj:
            raise TraceFormatError(f"{path}:{lineno}: expected a record object")
        return obj

    head = record(1, lines[0])
    if head.get("record") != "spec":
        raise TraceFormatError(f"{path}:1: first record must be the model spec")
    spec = _spec_from_header(path, head)
    passes: list = []
    for lineno, text in enumerate(lines[1:], start=2):
        if not text.strip():
            continue
        obj = record(lineno, text)
        if obj.get("record") != "event":
            raise TraceFormatError(f"{path}:{lineno}: unexpected record {obj.get('record')!r}")
        try:
            pid, kind, layer = int(obj["pass_id"]), str(obj["kind"]), int(obj["layer"])
            mat = np.asarray(obj["logits"], dtype=np.float32)
        except (KeyError, TypeError, ValueError) as exc:
            raise TraceFormatError(f"{path}:{lineno}: bad event record: {exc}") from None
        if kind not in (PREFILL, DECODE):
            raise TraceFormatError(f"pass {pid} layer {layer}: unknown kind {kind!r}")
        if not passes or passes[-1].pass_id != pid:
            passes.append(ForwardPass(pid, kind, []))
        passes[-1].events.append(LayerEvent(pid, kind, layer, mat))
    tr = Trace(spec, passes, head.get("meta", {}))
    tr.validate()
    return tr


def _read_jsonl_native(path, raw: bytes, alloc):
    """The native fast path of read_trace for JSON lines (None: use the
    reference-exact reader, which also produces every error message)."""
    import ctypes as C
    # the native parser splits lines on \n only; str.splitlines() also splits
    # on these, so such files take the reference-exact reader
    if any(raw.find(b) >= 0 for b in (b"\x0b", b"\x0c", b"\x1c", b"\x1d", b"\x1e", b"\xc2\x85",
                                      b"\xe2\x80\xa8", b"\xe2\x80\xa9")) or \
            raw.count(b"\r") != raw.count(b"\r\n"):
        return None
    nl = raw.find(b"\n")
    first = raw[:nl if nl >= 0 else len(raw)]
    try:
        head = json.loads(first)
    except (json.JSONDecodeError, UnicodeDecodeError):
        return None
    if not isinstance(head, dict) or head.get("record") != "spec":
        return None
    try:
        spec = _spec_from_header(path, head)
    except TraceFormatError:
        return None
    from ._device import lib
    L = lib()
    h, rows, npass, bad = C.c_void_p(), C.c_int64(), C.c_int32(), C.c_int64()
    rc = L.esim_trace_jsonl_parse(raw, len(raw), spec.num_layers, spec.experts_per_layer, 0, C.byref(h),
                                  C.byref(rows), C.byref(npass), C.byref(bad))
    if rc != 0:
        return None
    logits = _alloc_rows(rows.value, spec.experts_per_layer, alloc)
    toks = np.zeros(npass.value, np.int32)
    kinds = np.zeros(npass.value, np.int32)
    L.esim_trace_jsonl_take(h, logits.ctypes.data, toks.ctypes.data, kinds.ctypes.data)
    return _from_packed(spec, toks, kinds, logits, head.get("meta", {}))
