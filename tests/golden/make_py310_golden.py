"""Golden cases under CPython <= 3.11 builtin sum() semantics, made by running
the REAL reference with builtins.sum replaced by a restatement of CPython
3.10's builtin_sum_impl (bltinmodule.c): int fast path, then a float fast
path that is a plain left fold (3.12 added Neumaier compensation), then the
generic PyNumber_Add loop. The reference's own log ran Python 3.10.12
(pkg/test_output.txt:2); these pin the device's plain-sum mode
(esim_set_host_sum(0)) where the two semantics differ: RouteRec masses
(engine.py:630-631, cache-aware routing and drop/subst rows) and the
prefetch precision/recall macro sums (metrics.py:168-180).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_py310_golden.py
"""
from __future__ import annotations

import builtins
import gzip
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

_sum312 = builtins.sum


def sum310(iterable, start=0, /):
    """CPython 3.10 builtin_sum_impl: the float path adds without compensation."""
    it = iter(iterable)
    result = start
    if type(result) is int:
        for item in it:
            if type(item) is int or type(item) is bool:
                result += item
                continue
            result = result + item
            break
        else:
            return result
    if type(result) is float:
        f = result
        for item in it:
            if type(item) is float:
                f += item
                continue
            if type(item) is int and abs(item) < 2 ** 53:
                f += float(item)
                continue
            result = f + item
            break
        else:
            return f
    for item in it:
        result = result + item
    return result


def main():
    from make_golden import GB, builtin_spec, hw, run_case, synth  # noqa: E402  (imports the reference)
    olmoe, qwen, phi = builtin_spec("olmoe"), builtin_spec("qwen15moe"), builtin_spec("phi35moe")
    cases = []
    i = 0
    for spec, seed in ((olmoe, 31), (qwen, 32), (phi, 33)):
        for routing in ({"routing": "standard"}, {"routing": "cache_aware", "lam": 0.7}):
            for miss in ({"miss": "fetch"}, {"miss": "drop", "drop_rank_threshold": 2},
                         {"miss": "subst", "subst_tolerance": 0.05}):
                for pf in ({"prefetch": "score", "percentile": 70.0}, {"prefetch": "topk", "overfetch": 2.0}):
                    cfg = {"hardware": hw(capacity_fraction=0.05, bw=5 * GB), "working_precision": "int4",
                           "eviction": ("ls", "lru", "sb")[i % 3], **routing, **miss, **pf}
                    cases.append({"name": f"py310_{i:03d}", "trace": synth(spec, seed, 24, 24, affinity=0.5),
                                  "config": cfg, "full_log": False})
                    i += 1
    builtins.sum = sum310
    try:
        out = [run_case(c) for c in cases]
    finally:
        builtins.sum = _sum312
    # keep only cases whose report differs from 3.12 semantics (the ones that pin the mode)
    same = 0
    for c, o in zip(cases, out):
        o["differs_from_312"] = run_case(c)["report"] != o["report"]
        same += not o["differs_from_312"]
    print(f"{len(out)} cases, {len(out) - same} differ from CPython 3.12 sum() semantics")
    with gzip.open(os.path.join(HERE, "cases_py310.json.gz"), "wt") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
