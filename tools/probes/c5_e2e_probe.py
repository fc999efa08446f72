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
print("collect_trace", opts.collect_trace, "Y fortran", Y.flags.f_contiguous)
for i in range(6):
    t0 = time.perf_counter()
    r = F.run_lasso_batched(seq, Y, lams, cfg, opts, 0)
    t1 = time.perf_counter()
    print(f"e2e {1e3*(t1-t0):.2f} ms device {r[0].batch_device_ms:.2f}")
with bench.ClockSampler(0) as clk:
    for i in range(3):
        t0 = time.perf_counter()
        r = F.run_lasso_batched(seq, Y, lams, cfg, opts, 0)
        t1 = time.perf_counter()
        print(f"sampled e2e {1e3*(t1-t0):.2f} ms device {r[0].batch_device_ms:.2f}")
