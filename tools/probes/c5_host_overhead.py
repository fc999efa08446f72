import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
from paper_1812_06635_b200 import fastl1 as F
a, Y, lams = bench.make_c5(5)
n, k = a.shape; B = Y.shape[1]
d = F.DenseDictionary(a); L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L])
orig = F._collect_results
tc = []
def timed(lib, hs, B):
    t = time.perf_counter(); r = orig(lib, hs, B); tc.append(time.perf_counter() - t); return r
F._collect_results = timed
for i in range(6):
    t = time.perf_counter()
    rs = F.run_lasso_batched(seq, Y, lams, cfg, opts, 0)
    tot = time.perf_counter() - t
    print(f"host-Y call {tot*1e3:.2f} ms: device {rs[0].batch_device_ms:.2f} ms, collect {tc[-1]*1e3:.2f} ms")
