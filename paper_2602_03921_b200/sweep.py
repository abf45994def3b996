"""Policy-sweep replay: many grid points over shared traces, on 1..N GPUs.

The reference runs a sweep as a process pool of independent simulations
(cli.py:424-495, grid order = itertools.product of the axes with the last
axis fastest, cli.py:446). Here every grid point is one warp of the replay
kernel, all points of a model share one router pass over their trace, and
N GPUs each replay a contiguous, cost-balanced block of the grid; the
fixed-size result records are gathered to rank 0 with one NCCL all-gather.

Two entry points:
  run_grid_host(cfgs, traces)    the C-ABI end-to-end call (esim_run_host):
                                 host trace buffers in, host reports out
  DeviceSweep                    device-resident staging for repeated runs
                                 (the bench's timed loop)
"""
from __future__ import annotations

import csv
import ctypes as C
from dataclasses import replace
from itertools import product

import numpy as np

from . import _abi
from .engine import SimConfig, check_geometry
from .metrics import flatten_report, report_from_counters
from .models import GB, ConfigError, HardwareSpec, builtin_spec

# BASELINE.json configs[4] / SURVEY.md section 8(d) C5
C5_MODELS = ("olmoe", "mixtral", "qwen15moe", "phi35moe")
C5_EVICTIONS = ("lru", "lfu", "ls")
C5_CAPACITIES = (0.01, 0.05, 0.25)
C5_BANDWIDTHS = (1 * GB, 5 * GB, 25 * GB)


def grid(model: str, evictions=C5_EVICTIONS, capacities=C5_CAPACITIES, bandwidths=C5_BANDWIDTHS,
         **fixed) -> list:
    """SimConfigs in cli.py:446 product order (eviction, capacity, bandwidth; last fastest)."""
    spec = builtin_spec(model)
    base = dict(working_precision="int4", prefetch="score", percentile=80.0, miss="fetch", seed=0)
    base.update(fixed)
    out = []
    for ev, cap, bw in product(evictions, capacities, bandwidths):
        hw = HardwareSpec(capacity_fraction=cap, bandwidth_bytes_per_sec=bw)
        out.append(SimConfig(model=spec, hardware=hw, eviction=ev, **base))
    return out


def c5_points(traces_by_model: dict) -> tuple[list, list]:
    """The 108-point C5 grid (x len(traces) per model): parallel lists of configs and traces."""
    cfgs, trs = [], []
    for m in C5_MODELS:
        for tr in traces_by_model.get(m, ()):
            g = grid(m)
            cfgs += g
            trs += [tr] * len(g)
    return cfgs, trs


def shard_bounds(costs: list, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of points for `rank`, balanced by cumulative cost."""
    total = float(sum(costs))
    cum = np.concatenate([[0.0], np.cumsum(costs)])
    lo = int(np.searchsorted(cum, total * rank / world, side="left"))
    hi = int(np.searchsorted(cum, total * (rank + 1) / world, side="left"))
    if rank == world - 1:
        hi = len(costs)
    return lo, hi


# ---------------------------------------------------------------------------
def _lib():
    from ._device import lib
    return lib()


def _torch():
    from ._device import _torch as t
    return t()


def pin_traces(traces) -> None:
    """Move each trace's packed logits into page-locked memory (idempotent) so
    run_grid_host's host->device copies are DMA from pinned memory (the small
    per-trace arrays travel through the plan's own pinned image).

    The pinned buffer is a cudaHostAlloc allocation owned by the array, not a
    cudaHostRegister of the caller's heap memory: a registration outliving the
    array it was made for leaves a stale page-locked range behind, and a later
    copy into memory that reuses part of it fails (cudaErrorInvalidValue)."""
    torch = _torch()
    for tr in traces:
        pk = tr.packed()
        a = pk.logits
        if a.nbytes == 0 or getattr(pk, "_pinned", False):
            continue
        buf = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
        v = buf.numpy().view(a.dtype).reshape(a.shape)
        v[...] = a
        pk.logits = v
        pk._pinned = True


_CCFG_CACHE: dict = {}


def _noise_key(cfg):
    """The prediction-noise stream a point draws (None: no draws, engine.py:651-666)."""
    return (cfg.prefetch_noise, cfg.seed) if cfg.prefetch != "none" and cfg.prefetch_noise > 0 else None


def _c_config(cfg, trace_id: int):
    key = (cfg, trace_id)
    c = _CCFG_CACHE.get(key)
    if c is None:
        c = _CCFG_CACHE[key] = bytes(cfg.to_c(trace_id, False))
    return c


class HostGrid:
    """A sweep grid as a C-ABI plan (esim_sweep_plan_*): configs, trace
    descriptors (pointers into the callers' host trace arrays), groups and the
    device slab are resolved once; every `run()` is one esim_sweep_plan_run --
    trace H2D, router, replays, results D2H straight into this object's
    page-locked output arrays, in config order.

    Points get one trace_id per (trace, predictor, noise stream): the plan
    routes each trace_id once and applies its prediction noise on the device
    (esim_noise_launch)."""

    def __init__(self, cfgs, traces, pl_stride: int | None = None):
        from ._device import ensure_host_semantics
        ensure_host_semantics()
        ids, descs, self._keep = {}, [], []
        ccfg = []
        for cfg, tr in zip(cfgs, traces):
            check_geometry(cfg, tr)
            key = (id(tr), cfg.prefetch, cfg.overfetch, cfg.percentile, _noise_key(cfg))
            if key not in ids:
                ids[key] = len(descs)
                d, k = _abi.trace_desc_host(tr.packed())
                descs.append(d)
                self._keep.append(k)
            ccfg.append(_c_config(cfg, ids[key]))
        self.n = n = len(ccfg)
        self.L = pl_stride or max(c.model.num_layers for c in cfgs)
        carr = (_abi.EsimConfig * n).from_buffer_copy(b"".join(ccfg))
        darr = (_abi.EsimTraceDesc * len(descs))(*descs)
        self.counters, self.per_layer = self._pinned_outputs()
        h = C.c_void_p()
        rc = _lib().esim_sweep_plan_create(C.addressof(carr), n, C.addressof(darr), len(descs), self.L, 0, 0,
                                           C.byref(h))
        if rc != 0:
            self._raise(rc)
        self._plan = h

    def _pinned_outputs(self):
        """Counters + per-layer result buffers in page-locked (cudaHostAlloc)
        memory, so the plan's D2H copies land directly in them."""
        torch = _torch()
        cb = torch.zeros(self.n * C.sizeof(_abi.EsimCounters), dtype=torch.uint8, pin_memory=True)
        cs = (_abi.EsimCounters * self.n).from_address(cb.data_ptr())
        cs._owner = cb                                   # keep the pinned storage alive with the view
        pl = torch.zeros((self.n, self.L, _abi.ESIM_PL_FIELDS), dtype=torch.int64, pin_memory=True).numpy()
        return cs, pl

    @staticmethod
    def _raise(rc):
        msg = _lib().esim_last_error().decode()
        if rc == -1:
            raise ConfigError(msg)
        raise RuntimeError(f"esim_run_host failed ({rc}): {msg}")

    def run(self, check: bool = True):
        """Returns (counters, per_layer [n][pl_stride][ESIM_PL_FIELDS]): this grid's
        own output buffers (no copy), overwritten by the next run().
        check=False: a point that failed (EsimCounters.status != 0, e.g. an
        expert larger than the cache) does not raise; the other points'
        results are valid and the caller inspects each status."""
        rc = _lib().esim_sweep_plan_run(self._plan, C.addressof(self.counters), self.per_layer.ctypes.data,
                                        None, None)
        if rc != 0 and (check or not any(c.status for c in self.counters)):
            self._raise(rc)
        return self.counters, self.per_layer

    # ---- pipelined steps (double-buffered plan: esim_sweep_plan_submit / wait) ----
    def _out(self, slot: int):
        if not hasattr(self, "_outs"):
            self._outs = [(self.counters, self.per_layer)]
            self._next, self._inflight = 0, []
        while len(self._outs) <= slot:
            self._outs.append(self._pinned_outputs())
        return self._outs[slot]

    def submit(self) -> None:
        """Enqueue one step (inputs H2D, router, replays, results D2H) and return;
        up to two steps in flight, the next one's copies and router overlapping
        the current one's replays."""
        cs, pl = self._out(getattr(self, "_next", 0))
        rc = _lib().esim_sweep_plan_submit(self._plan, C.addressof(cs), pl.ctypes.data)
        if rc != 0:
            self._raise(rc)
        self._inflight.append(self._next)
        self._next ^= 1

    def wait(self):
        """Results of the oldest submitted step: (counters, per_layer), valid
        until that buffer's next submit."""
        slot = self._inflight.pop(0)
        rc = _lib().esim_sweep_plan_wait(self._plan)
        if rc != 0:
            self._raise(rc)
        return self._outs[slot]

    def close(self) -> None:
        if getattr(self, "_plan", None):
            _lib().esim_sweep_plan_destroy(self._plan)
            self._plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_grid_host(cfgs, traces, pl_stride: int | None = None):
    """One end-to-end C-ABI call (esim_run_host): host buffers in and out.

    Returns (counters list, per_layer array [n][pl_stride][ESIM_PL_FIELDS])."""
    g = HostGrid(cfgs, traces, pl_stride)
    try:
        cs, pl = g.run()
        return list(cs), pl
    finally:
        g.close()


def reports(cfgs, counters, per_layer) -> list:
    return [report_from_counters(c.echo(), c.model.num_layers, c.hardware.per_layer_compute_us, k,
                                 per_layer[i][:c.model.num_layers])
            for i, (c, k) in enumerate(zip(cfgs, counters))]


def csv_rows(cfgs, counters, per_layer) -> list:
    return [flatten_report(r) for r in reports(cfgs, counters, per_layer)]


_CFG_PREFIX: dict = {}


def _config_prefix(cfg) -> str:
    """The config columns of cfg's CSV row (fixed per point), as csv writes them
    (cached per config object: SimConfig hashing costs more than the lookup)."""
    hit = _CFG_PREFIX.get(id(cfg))
    if hit is not None and hit[0] is cfg:
        return hit[1]
    import io
    echo = cfg.echo()
    vals = []
    for key in sorted(echo):
        v = echo[key]
        vals.extend(v[sub] for sub in sorted(v)) if isinstance(v, dict) else vals.append(v)
    buf = io.StringIO()
    csv.writer(buf).writerow(vals)
    p = buf.getvalue()[:-2] + ","
    _CFG_PREFIX[id(cfg)] = (cfg, p)
    return p


def csv_text(cfgs, counters, per_layer, header: bool = True) -> str:
    """The reference sweep's CSV (emit(report, "csv") per point, cli.py:486-491)
    for these points: the fixed config columns are formatted once per config
    (cached), the result columns natively (esim_report_csv), ~2 us per point
    instead of ~200 us of Python report assembly. Byte-identical to emitting
    each report with metrics.emit."""
    n = len(cfgs)
    if not isinstance(counters, C.Array):
        counters = (_abi.EsimCounters * n)(*counters)
    per_layer = np.ascontiguousarray(per_layer, np.int64)
    nl = np.array([c.model.num_layers for c in cfgs], np.int32)
    cu = np.array([c.hardware.per_layer_compute_us for c in cfgs], np.int64)
    pre = [_config_prefix(c).encode() for c in cfgs]
    poffs = np.zeros(n + 1, np.int64)
    np.cumsum([len(p) for p in pre], out=poffs[1:])
    blob = b"".join(pre)
    cap = int(poffs[-1]) + 512 * n + 64
    out = C.create_string_buffer(cap)
    offs = np.zeros(n + 1, np.int64)
    rc = _lib().esim_report_csv(C.addressof(counters), per_layer.ctypes.data, per_layer.shape[1], nl.ctypes.data,
                                cu.ctypes.data, n, blob, poffs.ctypes.data, out, cap, offs.ctypes.data)
    if rc == -1:
        raise ValueError(_lib().esim_last_error().decode())
    if rc:
        raise RuntimeError(f"esim_report_csv failed ({rc})")
    body = C.string_at(out, int(offs[-1])).decode()
    return (",".join(flatten_report_columns(cfgs[0])) + "\r\n" + body) if header else body


def flatten_report_columns(cfg) -> list:
    """Column names of metrics.flatten_report for a config (metrics.py:348-362)."""
    from .metrics import TOTAL_FIELDS
    echo = cfg.echo()
    cols = []
    for key in sorted(echo):
        v = echo[key]
        cols.extend(f"{key}.{sub}" for sub in sorted(v)) if isinstance(v, dict) else cols.append(key)
    cols += [f"totals.{k}" for k in TOTAL_FIELDS]
    cols += [f"rates.{k}" for k in ("hit_rate", "miss_rate", "collision_rate_demanded", "collision_rate_misses",
                                    "drop_rate", "substitution_rate")]
    cols += [f"timing.{k}" for k in ("ttft_us", "total_us", "decode_us", "sync_overhead_us", "passes",
                                     "decode_passes", "per_layer_compute_us", "decode_tokens_per_sec")]
    cols += [f"fidelity.{k}" for k in ("routing_fidelity", "weight_mass_preserved", "modified_rows", "total_rows")]
    cols += [f"prefetch.{k}" for k in ("precision_micro", "recall_micro", "precision_macro", "recall_macro",
                                       "predicted_layers", "predicted_total", "predicted_hit_total",
                                       "empty_predictions", "zero_denominator")]
    return cols


# ---------------------------------------------------------------------------
class DeviceSweep:
    """Grid points staged in HBM; `step()` = router over every trace +
    replay of every point (one warp each), all on one stream."""

    def __init__(self, cfgs, traces, digest: bool = True):
        from ._device import ReplayBatch
        self.cfgs, self.traces = list(cfgs), list(traces)
        self.batch = ReplayBatch(self.cfgs, self.traces, full_log=False, digest=digest)

    def _router_tables(self):
        import torch
        from ._device import PREFETCH_CODE, lib
        params, prefix = [], [0]
        for _, dt, ro, (mode, over, pct), noised in self.batch.sets:
            out4 = (C.c_int32 * 4)()
            lib().esim_predictor_params(dt.pk.top_k, dt.pk.experts, PREFETCH_CODE[mode], float(over), float(pct), out4)
            params += list(out4)
            prefix.append(prefix[-1] + dt.pk.n_events)
        self._rparams = torch.tensor(params, dtype=torch.int32, device="cuda")
        self._rprefix = torch.tensor(prefix, dtype=torch.int64, device="cuda")
        self._total_events = prefix[-1]
        self._max_e = max(dt.pk.experts for _, dt, *_ in self.batch.sets)

    def route(self, stream=None) -> None:
        """Fused router over every trace of the sweep in one launch."""
        from ._device import _check, _stream, apply_noise, lib
        if not hasattr(self, "_rparams"):
            self._router_tables()
        rc = lib().esim_router_launch_batch(self.batch.d_traces.data_ptr(), self.batch.d_routers.data_ptr(),
                                            self._rparams.data_ptr(), self._rprefix.data_ptr(),
                                            len(self.batch.sets), self._total_events, self._max_e,
                                            stream or _stream())
        _check(rc, "router batch")
        for _, dt, ro, (mode, _o, _p), noised in self.batch.sets:      # prefetch.py:110-136 on the device
            if noised:
                apply_noise(dt, ro, mode, noised[0], noised[1], stream)

    def replay(self, stream=None) -> None:
        self.batch.launch(stream)

    def tune_order(self) -> None:
        """Longest-measured replays first in every launch group (see ReplayBatch.tune_order)."""
        self.batch.tune_order()

    def step(self, stream=None) -> None:
        self.route(stream)
        self.replay(stream)

    @property
    def n_router_launches(self) -> int:
        return 3        # classify_kernel, router_persistent_kernel, route_totals_kernel

    @property
    def n_replay_launches(self) -> int:
        return len(self.batch.groups)

    def counters_tensor(self):
        return self.batch.counters

    def results(self) -> list:
        return self.batch.results()


# ---------------------------------------------------------------------------
# multi-GPU sharding: contiguous cost-balanced blocks
# of the grid per rank, fixed-size counter records all-gathered to every rank
# ---------------------------------------------------------------------------
RECORD_BYTES = C.sizeof(_abi.EsimCounters)


def point_costs(cfgs, traces) -> list:
    """Relative replay cost per point: demanded token-expert selections of its trace."""
    cache: dict = {}
    out = []
    for cfg, tr in zip(cfgs, traces):
        if id(tr) not in cache:
            pk = tr.packed()
            cache[id(tr)] = int(pk.row_offset[-1]) * pk.top_k
        out.append(cache[id(tr)])
    return out


def gather_counter_records(local: bytes, bounds: list, group=None, device=None) -> bytes:
    """All-gather each rank's packed EsimCounters records (rank r holds points
    bounds[r][0]:bounds[r][1]) and return all records in global point order.
    One all_gather_into_tensor of equal-size (padded) buffers: NCCL on GPU
    ranks, gloo on CPU."""
    return gather_records(local, bounds, RECORD_BYTES, group, device)


def gather_records(local: bytes, bounds: list, rec_bytes: int, group=None, device=None) -> bytes:
    """gather_counter_records for any fixed-size per-point record."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lens = [(hi - lo) * rec_bytes for lo, hi in bounds]
    assert len(local) == lens[rank], (len(local), lens[rank])
    width = max(max(lens), 1)
    dev = device if device is not None else torch.device("cpu")
    buf = torch.zeros(width, dtype=torch.uint8, device=dev)
    if local:
        buf[:len(local)] = torch.frombuffer(bytearray(local), dtype=torch.uint8).to(dev)
    out = torch.empty(world * width, dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(out, buf, group=group)
    host = out.cpu().numpy().tobytes()
    return b"".join(host[r * width:r * width + lens[r]] for r in range(world))


class ShardedSweep:
    """One sweep grid split across the ranks of a process group (SURVEY.md
    section 8(e); the replacement for the reference's process pool,
    cli.py:462-482): every rank replays a contiguous, cost-balanced block
    [lo:hi) of the grid (the cli.py:446 product order) on its own GPU through
    the C-ABI plan, then the fixed-size result records (EsimCounters + the
    per-layer rows) are all-gathered in point order -- one collective per
    record kind, no data-path collective -- and rank 0 formats the reference
    sweep CSV (cli.py:486-491). NCCL between GPU ranks, gloo when ranks share
    a device or run on CPU hosts."""

    def __init__(self, cfgs, traces, group=None, pl_stride: int | None = None, check: bool = True):
        import torch
        import torch.distributed as dist
        self.cfgs, self.traces, self.group, self.check = list(cfgs), list(traces), group, check
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.L = pl_stride or max(c.model.num_layers for c in self.cfgs)
        self.bounds = [shard_bounds(point_costs(self.cfgs, self.traces), r, self.world) for r in range(self.world)]
        lo, hi = self.bounds[self.rank]
        self.lo, self.hi = lo, hi
        self.grid = HostGrid(self.cfgs[lo:hi], self.traces[lo:hi], self.L) if hi > lo else None
        nccl = self.world > 1 and dist.get_backend(group) == "nccl"
        self.device = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")

    def run(self):
        """Replay this rank's block and gather everyone's results.
        Returns (counters [n], per_layer [n][L][ESIM_PL_FIELDS]) for the whole
        grid, in point order, on every rank."""
        n = len(self.cfgs)
        pl_rec = self.L * _abi.ESIM_PL_FIELDS * 8
        if self.grid is not None:
            cs, pl = self.grid.run(check=self.check)       # check=False: failed points carry their status
            loc_c, loc_p = bytes(cs), np.ascontiguousarray(pl).tobytes()
        else:
            loc_c, loc_p = b"", b""
        if self.world > 1:
            all_c = gather_records(loc_c, self.bounds, RECORD_BYTES, self.group, self.device)
            all_p = gather_records(loc_p, self.bounds, pl_rec, self.group, self.device)
        else:
            all_c, all_p = loc_c, loc_p
        counters = (_abi.EsimCounters * n).from_buffer_copy(all_c)
        per_layer = np.frombuffer(all_p, np.int64).reshape(n, self.L, _abi.ESIM_PL_FIELDS).copy()
        return counters, per_layer

    def csv(self, header: bool = True):
        """The whole grid's reference-format CSV on rank 0 (None elsewhere)."""
        cs, pl = self.run()
        return csv_text(self.cfgs, cs, pl, header) if self.rank == 0 else None

    def close(self) -> None:
        if self.grid is not None:
            self.grid.close()
            self.grid = None


def run_sharded(cfgs, traces, group=None) -> str | None:
    """shard_bounds -> device replay of [lo:hi) -> all-gather -> rank-0 CSV."""
    s = ShardedSweep(cfgs, traces, group)
    try:
        return s.csv()
    finally:
        s.close()
