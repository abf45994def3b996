"""Sweep grid order (the reference CLI's product order, cli.py:446) and the
multi-rank shard + all-gather protocol on CPU ranks (gloo, world size 2),
checked against a single-process run of the oracle."""
import os
import socket

import numpy as np
import pytest

from golden_cases import cases
from paper_2602_03921_b200.sweep import C5_MODELS, RECORD_BYTES, grid, point_costs, shard_bounds


def test_grid_order_matches_the_reference_sweep():
    names = [c["name"] for c in cases() if c["name"].startswith("sweep_olmoe_")]
    g = grid("olmoe")
    mine = [f"sweep_olmoe_{c.eviction}_{c.hardware.capacity_fraction}_{c.hardware.bandwidth_bytes_per_sec // 10**9}g"
            for c in g]
    assert mine == names and len(g) == 27


def test_shard_bounds_cover_and_balance():
    costs = list(np.random.default_rng(0).integers(1, 100, size=108))
    for world in (1, 2, 4, 8):
        b = [shard_bounds(costs, r, world) for r in range(world)]
        assert b[0][0] == 0 and b[-1][1] == 108
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
        loads = [sum(costs[lo:hi]) for lo, hi in b]
        assert max(loads) <= sum(costs) / world + max(costs)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from oracle import oracle
    from paper_2602_03921_b200.models import builtin_spec
    from paper_2602_03921_b200.sweep import c5_points, gather_counter_records
    from paper_2602_03921_b200.trace import generate_synthetic
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    trs = {m: [generate_synthetic(builtin_spec(m), seed=2, prefill_tokens=8, decode_tokens=4)] for m in C5_MODELS}
    cfgs, tl = c5_points(trs)
    bounds = [shard_bounds(point_costs(cfgs, tl), r, world) for r in range(world)]
    lo, hi = bounds[rank]
    local = b"".join(bytes(oracle.run(c, t, full_log=False).counters) for c, t in zip(cfgs[lo:hi], tl[lo:hi]))
    allrec = gather_counter_records(local, bounds)
    if rank == 0:
        q.put(allrec)
    dist.destroy_process_group()


def test_two_rank_gloo_gather_equals_single_process():
    import multiprocessing as mp
    from oracle import oracle
    from paper_2602_03921_b200.models import builtin_spec
    from paper_2602_03921_b200.sweep import c5_points
    from paper_2602_03921_b200.trace import generate_synthetic
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    allrec = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    trs = {m: [generate_synthetic(builtin_spec(m), seed=2, prefill_tokens=8, decode_tokens=4)] for m in C5_MODELS}
    cfgs, tl = c5_points(trs)
    want = b"".join(bytes(oracle.run(c, t, full_log=False).counters) for c, t in zip(cfgs, tl))
    assert len(allrec) == len(cfgs) * RECORD_BYTES
    assert allrec == want
