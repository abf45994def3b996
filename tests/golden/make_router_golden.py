"""Known answers for routing.route_event(policy=cache_aware) from the REAL
reference (a DeltaAvgState carried across events, random cached sets and
lambda). PYTHONPATH=/root/reference/pkg/src python tests/golden/make_router_golden.py"""
import json
import os

import numpy as np

import expertsim
from expertsim.routing import DeltaAvgState, route_event

assert "/root/reference" in expertsim.__file__
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(77)
    out = []
    for E, k, T in ((64, 8, 6), (60, 4, 3), (8, 2, 5), (16, 2, 1), (200, 8, 2)):
        for lam in (0.0, 0.3, 2.5):
            delta = DeltaAvgState()
            seqs = []
            for ev in range(4):
                layer = int(rng.integers(0, 2))
                x = (rng.standard_normal((T, E)) * rng.uniform(0.5, 4.0) + rng.uniform(-1, 1)).astype(np.float32)
                cached = sorted(int(e) for e in rng.choice(E, size=int(rng.integers(0, E // 2 + 1)), replace=False))
                dec = route_event(x, k, "cache_aware", lam, set(cached), delta, layer)
                seqs.append({"layer": layer, "logits": [[float(v).hex() for v in r] for r in x], "cached": cached,
                             "selected": [d.selected for d in dec], "original": [d.original_selected for d in dec],
                             "weights": [[float(w).hex() for w in d.weights] for d in dec],
                             "modified": [d.modified for d in dec],
                             "delta": [float(delta.sums[layer]).hex(), delta.counts[layer]]})
            out.append({"E": E, "k": k, "lam": lam, "events": seqs})
    json.dump(out, open(os.path.join(HERE, "router_cache_aware.json"), "w"), separators=(",", ":"))
    print(len(out))


if __name__ == "__main__":
    main()
