"""The sharded sweep entry point (sweep.run_sharded)
on the DEVICE path: two ranks (gloo; they share the one GPU of the test box)
each replay their cost-balanced block of the C5 grid through the C-ABI plan,
all-gather the result records and rank 0 formats the reference sweep CSV.
It must equal the single-process device sweep byte for byte, and every
point's log digest must equal the C oracle's."""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu

SEEDS = (1, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _grid():
    from paper_2602_03921_b200.models import builtin_spec
    from paper_2602_03921_b200.sweep import C5_MODELS, c5_points
    from paper_2602_03921_b200.trace import generate_synthetic
    trs = {m: [generate_synthetic(builtin_spec(m), seed=s, prefill_tokens=16, decode_tokens=8) for s in SEEDS]
           for m in C5_MODELS}
    return c5_points(trs)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2602_03921_b200.sweep import ShardedSweep
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfgs, tl = _grid()
    s = ShardedSweep(cfgs, tl)
    text = s.csv()
    cs, _ = s.run()
    q.put((rank, s.bounds[rank], text, [int(c.digest) for c in cs]))
    s.close()
    dist.destroy_process_group()


def test_two_rank_sharded_device_sweep_equals_single_process():
    import multiprocessing as mp
    from oracle import oracle
    from paper_2602_03921_b200.sweep import csv_text, run_grid_host
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    import queue
    import time
    got, t_end = [], time.time() + 600
    while len(got) < len(procs):            # fail fast when a rank dies instead of waiting out the queue
        try:
            got.append(q.get(timeout=5))
        except queue.Empty:
            assert all(p.is_alive() or p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
            assert time.time() < t_end, "sharded sweep ranks timed out"
    got.sort(key=lambda g: g[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfgs, tl = _grid()
    (b0, b1) = got[0][1], got[1][1]
    assert b0[0] == 0 and b0[1] == b1[0] and b1[1] == len(cfgs) and 0 < b0[1] < len(cfgs)   # both ranks replay
    assert got[1][2] is None                                   # only rank 0 emits
    cs, pl = run_grid_host(cfgs, tl)
    assert got[0][2] == csv_text(cfgs, cs, pl)                 # byte-identical CSV
    assert got[0][3] == got[1][3] == [int(c.digest) for c in cs]
    want = [int(oracle.run(c, t, full_log=False).counters.digest) for c, t in zip(cfgs, tl)]
    assert got[0][3] == want
