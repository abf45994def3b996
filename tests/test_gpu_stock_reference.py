"""On-box parity against the unmodified reference: the stock `expertsim`
(pip-installed offline into baseline/_ref, which travels with the repo; the
test skips without it) runs a slice of the C5 grid on the host, and its own
emit(report, "csv") rows must equal, byte for byte, the rows the C-ABI sweep
plan (router + replay kernels on the GPU) produces for the same points."""
import importlib
import os
import sys
import tempfile
from itertools import product

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _stock():
    if not os.path.isdir(os.path.join(REF, "expertsim")):
        pytest.skip("baseline/_ref not installed")
    sys.path.insert(0, REF)
    try:
        return {m: importlib.import_module(f"expertsim.{m}") for m in ("engine", "models", "trace", "metrics")}
    finally:
        sys.path.remove(REF)


@pytest.mark.parametrize("model,seed", [("olmoe", 3), ("mixtral", 4), ("qwen15moe", 5), ("phi35moe", 6)])
def test_device_sweep_csv_equals_stock_reference(model, seed):
    es = _stock()
    from paper_2602_03921_b200.models import builtin_spec
    from paper_2602_03921_b200.sweep import C5_BANDWIDTHS, C5_CAPACITIES, C5_EVICTIONS, HostGrid, csv_text, grid
    from paper_2602_03921_b200.trace import generate_synthetic
    pts = list(product(C5_EVICTIONS, C5_CAPACITIES, C5_BANDWIDTHS))[::4]          # 7 of the 27 points
    tr = generate_synthetic(builtin_spec(model), seed=seed, prefill_tokens=64, decode_tokens=64, affinity=0.6,
                            skew=1.0)
    cfgs = [c for c, p in zip(grid(model), product(C5_EVICTIONS, C5_CAPACITIES, C5_BANDWIDTHS)) if p in pts]
    g = HostGrid(cfgs, [tr] * len(cfgs))
    cs, pl = g.run()
    dev = csv_text(cfgs, list(cs), pl)
    g.close()
    spec = es["models"].builtin_spec(model)
    rtr = es["trace"].generate_synthetic(spec, seed=seed, prefill_tokens=64, decode_tokens=64, affinity=0.6,
                                         skew=1.0)
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "ref.csv")
        for ev, cap, bw in pts:
            hw = es["models"].HardwareSpec(capacity_fraction=cap, bandwidth_bytes_per_sec=bw)
            cfg = es["engine"].SimConfig(model=spec, hardware=hw, eviction=ev, working_precision="int4",
                                         prefetch="score", percentile=80.0, miss="fetch", seed=0)
            es["metrics"].emit(es["engine"].run_simulation(cfg, rtr), "csv", path)
        with open(path, newline="") as fh:
            ref = fh.read()
    assert dev == ref
