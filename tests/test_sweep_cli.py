"""The sweep CLI (paper_2602_03921_b200.cli, reference cli.py:322-495)
against goldens made by running the reference CLI (tests/golden/
make_sweep_golden.py): the regenerated trace file is byte-identical, the
grid rows (product order, presets, `original` eviction, config errors) match
on CPU, and on the GPU the whole sweep -- exit code, stdout, the FAILED
lines on stderr and the CSV file -- is identical."""
import contextlib
import gzip
import hashlib
import io
import json
import os

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(gzip.open(os.path.join(HERE, "golden", "sweep_cli.json.gz"), "rt"))


def _run(argv):
    from paper_2602_03921_b200.cli import main
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = main(argv)
    return rc, out.getvalue(), err.getvalue()


def _trace(tmp_path, case):
    p = tmp_path / (case["name"] + ".trace")
    rc, out, _ = _run(["gen-trace", *case["gen"], "--out", str(p)])
    assert rc == 0 and out.startswith(f"wrote {p}: ")
    return p


@pytest.mark.parametrize("case", GOLD, ids=[c["name"] for c in GOLD])
def test_gen_trace_file_is_byte_identical(tmp_path, case):
    p = _trace(tmp_path, case)
    assert hashlib.sha256(p.read_bytes()).hexdigest() == case["trace_sha256"]


@pytest.mark.parametrize("case", GOLD, ids=[c["name"] for c in GOLD])
def test_sweep_rows_and_config_errors(tmp_path, case):
    """Row tags in product order and the config-error rows, without a GPU."""
    from paper_2602_03921_b200.cli import Settings, build_parser, flag_overrides, AXIS_KEYS, sweep_axes, sweep_rows
    from paper_2602_03921_b200.trace import read_trace
    p = _trace(tmp_path, case)
    args = build_parser().parse_args(["sweep", "--trace", str(p), *case["sweep"]])
    rows = sweep_rows(Settings(), flag_overrides(args, skip=AXIS_KEYS), sweep_axes(args), read_trace(p).spec)
    want_lines = [ln for ln in case["stdout"].splitlines() + case["stderr"].splitlines() if ln.startswith("[")]
    want = {int(ln[1:4]): ln for ln in want_lines}
    assert sorted(want) == [r["idx"] for r in rows]
    for r in rows:
        tag = want[r["idx"]].split(": ", 1)[0][6:]
        assert r["tag"] == tag
        if r["error"] is not None:
            assert want[r["idx"]] == f"[{r['idx']:3d}] {r['tag']}: FAILED: {r['error']}"
        else:
            assert ": FAILED: " not in want[r["idx"]]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD, ids=[c["name"] for c in GOLD])
def test_sweep_cli_matches_reference_byte_for_byte(tmp_path, case):
    p = _trace(tmp_path, case)
    out_csv = tmp_path / (case["name"] + ".csv")
    rc, out, err = _run(["sweep", "--trace", str(p), *case["sweep"], "--out", str(out_csv), "--jobs", "1"])
    d = str(tmp_path)
    assert rc == case["rc"]
    assert out.replace(d, "<DIR>") == case["stdout"]
    fails = [ln for ln in err.replace(d, "<DIR>").splitlines() if ": FAILED: " in ln]
    assert fails == [ln for ln in case["stderr"].splitlines() if ": FAILED: " in ln]
    got_csv = open(out_csv, newline="").read() if out_csv.exists() else None
    assert got_csv == case["csv"]


@pytest.mark.gpu
def test_sweep_cli_sharded_under_torchrun_matches_reference(tmp_path):
    """`torchrun --nproc-per-node 2 -m paper_2602_03921_b200.cli sweep ...`: the
    rows sharded over two ranks (gloo: they share the test box's one GPU),
    results all-gathered, rank 0 writes -- stdout and CSV identical to the
    reference CLI's single-process sweep."""
    import socket
    import subprocess
    import sys
    case = next(c for c in GOLD if c["name"] == "presets_olmoe")
    p = _trace(tmp_path, case)
    out_csv = tmp_path / (case["name"] + ".csv")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    root = os.path.dirname(HERE)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "-m", "paper_2602_03921_b200.cli",
           "sweep", "--trace", str(p), *case["sweep"], "--out", str(out_csv), "--jobs", "1"]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "PYTHONPATH": root, "OMP_NUM_THREADS": "1"})
    assert r.returncode == case["rc"], r.stderr[-2000:]
    assert r.stdout.replace(str(tmp_path), "<DIR>") == case["stdout"]
    assert open(out_csv, newline="").read() == case["csv"]
