"""Eviction-policy plug-in objects on the device vs op sequences recorded from
the REAL reference classes (tests/golden/policy_ops.json, written by
tests/golden/make_policy_golden.py): every select_victim result and the LS
structural counters must match."""
import json
import os

import pytest

from paper_2602_03921_b200.eviction import AccessContext, LSPolicy, make_eviction_policy

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "policy_ops.json")))


@pytest.mark.parametrize("name", ["lru", "lfu", "lhu", "fld", "sb", "ls"])
def test_policy_objects_match_reference(name):
    for seq in (s for s in GOLD if s["policy"] == name):
        pol = make_eviction_policy(name, num_layers=3, highest_precision="fp16", sb_decay=0.75)
        pass_id = 0
        for op in seq["ops"]:
            if op[0] == "pass":
                pass_id = op[1]
                pol.begin_pass(pass_id)
            elif op[0] == "admit":
                pol.note_admit(tuple(op[1]), AccessContext(op[2], pass_id, None, op[3]))
            elif op[0] == "access":
                pol.note_access(tuple(op[1]), AccessContext(op[2], pass_id, op[4], op[3]))
            elif op[0] == "prefetch_hit":
                pol.note_prefetch_hit(tuple(op[1]), AccessContext(op[2], pass_id, None, "fp16"))
            else:
                got = pol.select_victim(AccessContext(op[2], pass_id, None, None), forced=op[1])
                want = None if op[3] is None else tuple(op[3])
                assert got == want, (name, seq["seed"], op)
        if name == "ls":
            assert isinstance(pol, LSPolicy)
            assert [pol.forced_current_evictions, pol.unforced_current_evictions, pol.refusals,
                    pol.stale_size(), pol.current_size()] == seq["ls"]


def test_begin_pass_ids_must_increase():
    pol = make_eviction_policy("ls", 2, "fp16")
    pol.begin_pass(0)
    with pytest.raises(RuntimeError, match="strictly increase"):
        pol.begin_pass(0)
