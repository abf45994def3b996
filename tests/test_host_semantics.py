"""Host-interpreter semantics the bit-exact path depends on (SURVEY.md
Appendix A; VERDICT r1 "portability guards"): CPython <= 3.11 builtin
sum() is a plain left fold, >= 3.12 is Neumaier-compensated. Goldens made
by the REAL reference under a restated 3.10 sum() (tests/golden/
make_py310_golden.py) pin the oracle's and the device's plain-sum mode; the
same cases under 3.12 semantics pin the default. The device additionally
checks its float32 exp / pairwise-sum restatement against this host's numpy
before its first computation (_device.ensure_host_semantics)."""
import gzip
import json
import os

import pytest

from golden_cases import GOLDEN, config_from, trace_from
from paper_2602_03921_b200.records import canon_reference_record, digest_records

PY310 = json.load(gzip.open(os.path.join(GOLDEN, "cases_py310.json.gz"), "rt"))


def test_py310_goldens_exercise_the_difference():
    assert sum(c["differs_from_312"] for c in PY310) >= 10


def test_oracle_plain_sum_mode_matches_reference_py310(oracle_lib):
    oracle_lib.set_host_sum(False)
    try:
        for c in PY310:
            res = oracle_lib.run(config_from(c), trace_from(c["trace"]), full_log=True)
            assert json.dumps(res.report) == json.dumps(c["report"]), c["name"]
            assert digest_records([canon_reference_record(r) for r in res.log]) == c["log_sha256"], c["name"]
    finally:
        oracle_lib.set_host_sum(True)
    # and the default (this interpreter, CPython >= 3.12) differs exactly where the goldens say
    for c in PY310:
        res = oracle_lib.run(config_from(c), trace_from(c["trace"]))
        assert (json.dumps(res.report) != json.dumps(c["report"])) == c["differs_from_312"], c["name"]


@pytest.mark.gpu
def test_device_plain_sum_mode_matches_reference_py310():
    from paper_2602_03921_b200._device import ensure_host_semantics, lib, run_simulations
    ensure_host_semantics()
    assert lib().esim_get_host_sum() == 1
    cfgs = [config_from(c) for c in PY310]
    trs = [trace_from(c["trace"]) for c in PY310]
    assert lib().esim_set_host_sum(0) == 0
    try:
        res = run_simulations(cfgs, trs)
        for c, r in zip(PY310, res):
            assert json.dumps(r.report) == json.dumps(c["report"]), c["name"]
    finally:
        assert lib().esim_set_host_sum(1) == 0
    res = run_simulations(cfgs, trs)
    for c, r in zip(PY310, res):
        assert (json.dumps(r.report) != json.dumps(c["report"])) == c["differs_from_312"], c["name"]


@pytest.mark.gpu
def test_device_softmax_selfcheck_against_host_numpy():
    """The startup check passes on this host and catches a perturbed reference."""
    import numpy as np
    from paper_2602_03921_b200 import _device
    _device._host_checked = False
    _device.ensure_host_semantics()           # raises if this host's numpy differs
    assert _device._host_checked
    real_exp = np.exp
    try:
        np.exp = lambda x, dtype=None: np.nextafter(real_exp(x, dtype=dtype), np.float32(np.inf))
        _device._host_checked = False
        with pytest.raises(RuntimeError, match="host numpy float32 softmax differs"):
            _device.ensure_host_semantics()
    finally:
        np.exp = real_exp
        _device._host_checked = False
        _device.ensure_host_semantics()
