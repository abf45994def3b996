"""The CPU oracle against the REAL reference's outputs (tests/golden, written
by tests/golden/make_golden.py): reports byte-identical, event logs
digest-identical, full logs record-identical where stored. This pins the
oracle before it is trusted as the GPU path's checker."""
import json

import numpy as np
import pytest

from golden_cases import cases, config_from, trace_from
from paper_2602_03921_b200.metrics import build_report
from paper_2602_03921_b200.records import canon_reference_record, digest_records

ALL = cases()
GROUPS = sorted({c["name"].split("_")[0] for c in ALL})


@pytest.mark.parametrize("group", GROUPS)
def test_oracle_matches_reference(group, oracle_lib):
    bad = []
    for c in ALL:
        if c["name"].split("_")[0] != group:
            continue
        cfg, tr = config_from(c), trace_from(c["trace"])
        res = oracle_lib.run(cfg, tr, full_log=True)
        canon = [canon_reference_record(r) for r in res.log]
        if json.dumps(res.report) != json.dumps(c["report"]):
            bad.append((c["name"], "report"))
        if digest_records(canon) != c["log_sha256"]:
            bad.append((c["name"], "log digest"))
        if "log" in c and [list(t) for t in canon] != c["log"]:
            bad.append((c["name"], "log records"))
        # the log-driven report path gives the same bytes as the counter path
        rep2 = build_report(cfg.echo(), cfg.model.num_layers, cfg.hardware.per_layer_compute_us, res.log)
        if json.dumps(rep2) != json.dumps(c["report"]):
            bad.append((c["name"], "report-from-log"))
        if c["ls_counters"] is not None:
            got = [res.counters.ls_forced, res.counters.ls_unforced, res.counters.ls_refusals]
            if got != c["ls_counters"]:
                bad.append((c["name"], f"ls counters {got} != {c['ls_counters']}"))
    assert not bad, bad[:10]


def test_generator_matches_reference_traces():
    import hashlib
    with open(__import__("golden_cases").GOLDEN + "/traces.json") as fh:
        recs = json.load(fh)
    assert len(recs) >= 10
    for r in recs:
        tr = trace_from(r["recipe"])
        h = hashlib.sha256()
        for fp in tr.passes:
            for ev in fp.events:
                h.update(np.ascontiguousarray(ev.logits, np.float32).tobytes())
        assert h.hexdigest() == r["sha256"], r["recipe"]


def test_hand_walkthrough_table(oracle_lib):
    """test_engine.py:120-188 hand table, restated."""
    expect = {"lru": ([(0, 0), (0, 2), (1, 1)], [6000, 11000, 17000], 1, (4, 0, 1)),
              "ls": ([(0, 0), (0, 2), (1, 1)], [6000, 11000, 17000], 1, (4, 0, 1)),
              "fld": ([(1, 1), (0, 0), (1, 1), (0, 0)], [6000, 12000, 18000], 0, (4, 1, 1)),
              "sb": ([(1, 1), (0, 0), (1, 1), (0, 0)], [6000, 12000, 18000], 0, (4, 1, 1))}
    for ev, (victims, ends, hits, classes) in expect.items():
        c = next(x for x in ALL if x["name"] == f"hand_{ev}")
        res = oracle_lib.run(config_from(c), trace_from(c["trace"]))
        got_v = [(r.victim_layer, r.victim_expert) for r in res.log if type(r).__name__ == "EvictRec"]
        got_e = [r.end_us for r in res.log if type(r).__name__ == "PassRec"]
        t = res.report["totals"]
        assert got_v == victims and got_e == ends and t["hits"] == hits
        assert (t["compulsory_misses"], t["collision_misses"], t["capacity_misses"]) == classes
