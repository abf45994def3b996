"""The 32-bit simulated-clock bound (esim_time32_ok, csrc/capi.cu): the
common-path replay kernels run their clock in int32 when the host proves
events x compute_us + (demands + predictions) x transfer_us < 2^31 us. The
bound must hold for every run the oracle replays (the clock only ever waits
on the transfer channel, whose busy time is at most one working-precision
transfer per queued fetch), and the library must agree with its restatement
here. CPU only: esim_time32_ok is host arithmetic."""
import ctypes as C

import numpy as np

LIM = (1 << 31) - 1


def _bound(cfg, pk):
    bw, nb = cfg.hardware.bandwidth_bytes_per_sec, cfg.model.expert_bytes(cfg.working_precision)
    dur = 0 if bw == 0 or nb == 0 else -(-nb * 1_000_000 // bw)
    ev, E = pk.n_events, pk.experts
    dem = min(int(pk.row_offset[-1]) * pk.top_k, ev * E)
    return ev * cfg.hardware.per_layer_compute_us + (dem + ev * E) * dur


def _common_cases(n, seed):
    from test_gpu_fuzz import _random_cases
    return [(c, t) for c, t in _random_cases(n, seed) if c.miss == "fetch" and c.routing == "standard"]


def test_bound_covers_the_oracle_clock(oracle_lib):
    cases = _common_cases(160, 11)
    assert len(cases) > 40
    for cfg, tr in cases:
        o = oracle_lib.run(cfg, tr, full_log=False)
        assert int(o.counters.status) == 0
        assert int(o.counters.total_us) <= _bound(cfg, tr.packed())


def test_library_agrees_with_the_restatement():
    import dataclasses
    from paper_2602_03921_b200 import _abi, _device
    from paper_2602_03921_b200.models import HardwareSpec
    L = _device.lib()
    seen = set()
    for cfg, tr in _common_cases(120, 12):
        pk = tr.packed()
        desc, keep = _abi.trace_desc_host(pk)
        for cu in (cfg.hardware.per_layer_compute_us, 10**6, LIM // max(1, pk.n_events), 2 * 10**9):
            hw = HardwareSpec(capacity_bytes=cfg.hardware.capacity_bytes,
                              bandwidth_bytes_per_sec=cfg.hardware.bandwidth_bytes_per_sec, per_layer_compute_us=cu)
            c2 = dataclasses.replace(cfg, hardware=hw)
            cc = c2.to_c(0, False)
            want = _bound(c2, pk) < LIM
            got = bool(L.esim_time32_ok(C.addressof(cc), C.addressof(desc)))
            assert got == want, (cu, _bound(c2, pk))
            seen.add(want)
    assert seen == {True, False}
