"""Host cost of collecting a 512-signal batched result in Python (cProfile of _collect_results)."""
import os, sys, time, cProfile, pstats
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np, torch
import bench
from paper_1812_06635_b200 import fastl1 as F
a, Y, lams = bench.make_c5(5)
n, k = a.shape; B = Y.shape[1]
d = F.DenseDictionary(a); L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L])
for _ in range(3):
    F.run_lasso_batched(seq, Y, lams, cfg, opts, 0)
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    F.run_lasso_batched(seq, Y, lams, cfg, opts, 0)
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(12)
