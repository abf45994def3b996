import sys, time, cProfile, pstats
sys.path.insert(0, ".")
from bench import make_traces
from paper_2602_03921_b200.sweep import c5_points, run_grid_host
cfgs, trs = c5_points(make_traces(list(range(1, 49))))
from paper_2602_03921_b200.sweep import pin_traces; pin_traces(trs); run_grid_host(cfgs, trs)
t0 = time.perf_counter(); run_grid_host(cfgs, trs); print("e2e s", time.perf_counter() - t0)
pr = cProfile.Profile(); pr.enable(); run_grid_host(cfgs, trs); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
