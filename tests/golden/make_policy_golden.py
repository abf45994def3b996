"""Golden op sequences for the eviction-policy plug-in objects, recorded from
the REAL reference classes (expertsim/eviction.py). Run in the build
container:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_policy_golden.py
Output: tests/golden/policy_ops.json (ops + every select_victim result + LS counters)."""
import json
import os
import random

import expertsim
from expertsim.eviction import AccessContext, make_eviction_policy

assert "/root/reference" in expertsim.__file__
HERE = os.path.dirname(os.path.abspath(__file__))
KEYS = [(l, e) for l in range(3) for e in range(3)]
PRECS = ["fp16", "int8", "int4"]


def run(name, seed, n_ops):
    rnd = random.Random(seed)
    pol = make_eviction_policy(name, num_layers=3, highest_precision="fp16", sb_decay=0.75)
    resident = set()
    pass_id = 0
    pol.begin_pass(pass_id)
    ops = [["pass", 0]]
    for _ in range(n_ops):
        r = rnd.random()
        if r < 0.3:
            k = rnd.choice(KEYS)
            if k in resident:
                continue
            c = AccessContext(k[0], pass_id, None, rnd.choice(PRECS))
            pol.note_admit(k, c)
            resident.add(k)
            ops.append(["admit", list(k), c.layer, c.precision])
        elif r < 0.6:
            if not resident:
                continue
            k = rnd.choice(sorted(resident))
            gate = None if rnd.random() < 0.2 else round(rnd.random(), 6)
            c = AccessContext(k[0], pass_id, gate, rnd.choice(PRECS))
            pol.note_access(k, c)
            ops.append(["access", list(k), c.layer, c.precision, gate])
        elif r < 0.7:
            if not resident:
                continue
            k = rnd.choice(sorted(resident))
            c = AccessContext(k[0], pass_id, None, "fp16")
            pol.note_prefetch_hit(k, c)
            ops.append(["prefetch_hit", list(k), c.layer])
        elif r < 0.92:
            forced = rnd.random() < 0.6
            layer = rnd.randrange(3)
            got = pol.select_victim(AccessContext(layer, pass_id, None, None), forced=forced)
            if got is not None:
                resident.discard(got)
            ops.append(["select", forced, layer, None if got is None else list(got)])
        else:
            pass_id += 1
            pol.begin_pass(pass_id)
            ops.append(["pass", pass_id])
    extra = None
    if name == "ls":
        extra = [pol.forced_current_evictions, pol.unforced_current_evictions, pol.refusals,
                 pol.stale_size(), pol.current_size()]
    return {"policy": name, "seed": seed, "ops": ops, "ls": extra}


def main():
    out = []
    for name in ("lru", "lfu", "lhu", "fld", "sb", "ls"):
        for seed in range(40):
            out.append(run(name, seed, 60))
    with open(os.path.join(HERE, "policy_ops.json"), "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(len(out), "sequences")


if __name__ == "__main__":
    main()
