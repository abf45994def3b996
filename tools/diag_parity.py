"""Parity diagnostics: every golden case (tests/golden) through one device
batch, digests vs the C oracle and reports vs the reference's goldens;
prints the mismatching cases grouped by eviction policy (with status)."""
import json, sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from test_gpu_replay import ALL, _batch
from oracle import oracle
bad = []
cfgs, trs, res = _batch(ALL, full_log=False)
for c, cfg, tr, r in zip(ALL, cfgs, trs, res):
    o = oracle.run(cfg, tr, full_log=False)
    if o.counters.digest != r.counters.digest or json.dumps(r.report) != json.dumps(c["report"]):
        bad.append((c["name"], cfg.eviction, cfg.miss, cfg.prefetch, cfg.capacity_bytes() // cfg.model.expert_bytes(cfg.working_precision), r.counters.status))
print(len(ALL), "cases", len(bad), "bad")
from collections import Counter
print(Counter(b[1] for b in bad))
for b in bad[:12]: print(b)
