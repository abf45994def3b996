"""Perf probe: oracle CPU timing vs device router+replay on the C5 grid."""
import sys, time, os, json
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2602_03921_b200.sweep import c5_points, DeviceSweep, run_grid_host
from paper_2602_03921_b200.trace import generate_synthetic
from paper_2602_03921_b200.models import builtin_spec
from oracle import oracle
out = {}
def traces(seeds):
    return {m: [generate_synthetic(builtin_spec(m), seed=s, prefill_tokens=64, decode_tokens=64) for s in seeds]
            for m in ("olmoe", "mixtral", "qwen15moe", "phi35moe")}
t1 = traces([1])
cfgs, trs = c5_points(t1)
ccfg = []
ids = {}
tl = []
for c, t in zip(cfgs, trs):
    if id(t) not in ids: ids[id(t)] = len(tl); tl.append(t)
    ccfg.append(c.to_c(ids[id(t)], False))
t0 = time.perf_counter(); cs, pl = oracle.run_batch(ccfg, tl, 1); dt1 = time.perf_counter() - t0
acc = sum(c.totals[0] for c in cs)
out["oracle_1thr_s"] = dt1; out["accesses_seed1"] = acc; out["oracle_1thr_acc_s"] = acc / dt1
t0 = time.perf_counter(); cs16, _ = oracle.run_batch(ccfg, tl, os.cpu_count()); dtn = time.perf_counter() - t0
out["oracle_nthr_s"] = dtn; out["oracle_nthr_acc_s"] = acc / dtn; out["threads"] = os.cpu_count()
for S, dg in ((1, True), (16, True), (48, True), (48, False), (96, True)):
    tt = traces(list(range(1, S + 1)))
    cfgs, trs = c5_points(tt)
    ds = DeviceSweep(cfgs, trs, digest=dg)
    st = torch.cuda.current_stream()
    for _ in range(2): ds.step()
    torch.cuda.synchronize()
    e0, e1, e2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e0.record(); ds.route(); e1.record(); ds.replay(); e2.record(); torch.cuda.synchronize()
    res = ds.results()
    a = sum(r.counters.totals[0] for r in res)
    out[f"S{S}{dg}"] = {"points": len(cfgs), "accesses": a, "route_ms": e0.elapsed_time(e1), "replay_ms": e1.elapsed_time(e2),
                    "acc_per_s": a / (e0.elapsed_time(e2) / 1e3)}
    print(S, dg, out[f"S{S}{dg}"], flush=True)
# digest check vs oracle for S=1
ds = DeviceSweep(*c5_points(t1)); ds.step(); res = ds.results()
out["digest_match_seed1"] = all(r.counters.digest == c.digest for r, c in zip(res, cs))
# e2e C-ABI
cfgs, trs = c5_points(t1)
t0 = time.perf_counter(); c2, p2 = run_grid_host(cfgs, trs); out["e2e_s_seed1"] = time.perf_counter() - t0
t0 = time.perf_counter(); c2, p2 = run_grid_host(cfgs, trs); out["e2e_s_seed1_warm"] = time.perf_counter() - t0
out["e2e_digest_match"] = all(a.digest == b.digest for a, b in zip(c2, cs))
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/probe_perf.json", "w"), indent=1)
