import sys, time
sys.path.insert(0, '.')
import bench, torch
wl = bench.WORKLOADS["C4"]
cfg, tg, cp = bench.build_plan(1, wl["kw"], 32, family="gpt")
t0 = time.time()
r = bench.gemm_roofline(cfg, 1, 24, 2268.0, 1571.8, 32)
print(r["frac"], time.time() - t0)
