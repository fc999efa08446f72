"""Single-solve device time, grid vs one 16-CTA cluster, across dictionary sizes."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
import bench
cases = [("c1", syn.dense_instance("c1"))]
a5, Y5, l5 = bench.make_c5(5)
cases.append(("c5-signal0", (a5, Y5[:, 0], l5[0])))
rng = np.random.default_rng(3)
for n, k in ((1024, 8192), (2048, 4096)):
    a = syn.gaussian_dictionary(rng, n, k)
    y = syn.observe(rng, a @ syn.sparse_signal(rng, k, 40), None, 30.0)
    cases.append((f"{n}x{k}", (a, y, 0.25 * float(np.max(np.abs(a.T @ y))))))
for name, inst in cases:
    if isinstance(inst, tuple):
        a, y, lam = inst
    else:
        a, y, lam = inst.a, inst.y, inst.lam
    d = F.DenseDictionary(a)
    L = F.lipschitz_bound(d)
    seq = F.ApproxSequence([F.make_exact_approx(d)])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L])
    for mode, env in (("grid", "0"), ("cl16", "1")):
        os.environ["FL1_SINGLE_CLUSTER"] = env
        os.environ["FL1_SINGLE_CLUSTER_MB"] = "100000"
        F.run_lasso(seq, y, lam, cfg, opts)
        ms = [F.run_lasso(seq, y, lam, cfg, opts).device_ms for _ in range(3)]
        print(f"{name:12s} {a.nbytes/2**20:7.1f} MiB {mode}: {np.mean(ms):7.3f} ms")
