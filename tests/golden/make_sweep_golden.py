"""Golden fixtures for the sweep CLI, made by running the REAL reference CLI
(`expertsim gen-trace` + `expertsim sweep --jobs 1`, cli.py:322-495).

Run in the build container only (imports the read-only reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_sweep_golden.py

Output: sweep_cli.json.gz -- per case the gen-trace argv and the sha256 of
the trace file it wrote (this repo's generator + writer must reproduce it
byte for byte), the sweep argv, exit code, stdout, stderr and the CSV.
The mixed-axis grids cover presets with `original` eviction, every
eviction / prefetch / miss token kind, cache-aware routing with an
out-of-range lambda (config-error rows), an expert larger than the cache
(runtime-error rows) and prediction noise.
"""
from __future__ import annotations

import contextlib
import gzip
import hashlib
import io
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))

from expertsim.cli import main as ref_main  # noqa: E402  (reference, read-only)

CASES = [
    {"name": "presets_olmoe",
     "gen": ["--model", "olmoe", "--seed", "3", "--prefill", "12", "--decode", "6"],
     "sweep": ["--preset", "config1,config2,config3,config4,config5", "--eviction", "original,ls,lfu",
               "--capacity", "0.02,0.1", "--bandwidth", "1e9,25e9"]},
    {"name": "tokens_qwen_cache_aware",
     "gen": ["--model", "qwen15moe", "--seed", "4", "--prefill", "10", "--decode", "5"],
     "sweep": ["--eviction", "lru,sb,fld", "--prefetch", "none,topk:1.5,score:70,oracle",
               "--miss", "fetch,drop:2,subst:0.05,fetch_low,fetch_priority", "--lam", "0.3,20",
               "--routing", "cache_aware", "--working", "int8"]},
    {"name": "tiny_cache_mixtral",
     "gen": ["--model", "mixtral", "--seed", "5", "--prefill", "8", "--decode", "6", "--drift", "0.2"],
     "sweep": ["--capacity", "0.001,0.05", "--eviction", "ls,lru,lhu", "--miss", "fetch,fetch_low,fetch_priority",
               "--working", "fp16", "--bandwidth", "0,5e9"]},
    {"name": "noise_phi",
     "gen": ["--model", "phi35moe", "--seed", "6", "--prefill", "6", "--decode", "8", "--affinity", "0.3"],
     "sweep": ["--prefetch", "score:80,topk", "--eviction", "ls,lhu,sb", "--prefetch-noise", "0.2", "--seed", "3",
               "--miss", "fetch_priority", "--degrade-percentile", "40", "--sb-decay", "0.7"]},
]


def run(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = ref_main(argv)
    return rc, out.getvalue(), err.getvalue()


def main():
    res = []
    with tempfile.TemporaryDirectory() as d:
        for c in CASES:
            tpath = os.path.join(d, c["name"] + ".trace")
            rc, _, _ = run(["gen-trace", *c["gen"], "--out", tpath])
            assert rc == 0
            sha = hashlib.sha256(open(tpath, "rb").read()).hexdigest()
            opath = os.path.join(d, c["name"] + ".csv")
            argv = ["sweep", "--trace", tpath, *c["sweep"], "--out", opath, "--jobs", "1"]
            rc, out, err = run(argv)
            csv_text = open(opath, newline="").read() if os.path.exists(opath) else None
            res.append({"name": c["name"], "gen": c["gen"], "trace_sha256": sha, "sweep": c["sweep"], "rc": rc,
                        "stdout": out.replace(d, "<DIR>"), "stderr": err.replace(d, "<DIR>"), "csv": csv_text})
            print(c["name"], "rc", rc, "rows", out.count("\n"), "errors", err.count("\n"))
    with gzip.open(os.path.join(HERE, "sweep_cli.json.gz"), "wt") as fh:
        json.dump(res, fh)


if __name__ == "__main__":
    sys.exit(main())
