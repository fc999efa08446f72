import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np
import bench
from paper_1812_06635_b200 import fastl1 as F
a, Y, lams = bench.make_c5(5)
n, k = a.shape
d = F.DenseDictionary(a)
L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L])
NB = int(os.environ.get('NB', '512'))
modes = [int(v) for v in os.environ.get('MODES', '4,-1,-2,-4,-8,-16').split(',')]
for M in modes:
    F.run_lasso_batched(seq, Y[:, :NB], lams[:NB], cfg, opts, M)
    t = time.perf_counter()
    rs = F.run_lasso_batched(seq, Y[:, :NB], lams[:NB], cfg, opts, M)
    wall = time.perf_counter() - t
    dm = np.array([r.device_ms for r in rs])
    it = np.array([r.iterations for r in rs]); pw = np.array([r.power_iterations for r in rs])
    pr = np.array([r.profile for r in rs])
    print(f"M={M:3d} wall={wall*1e3:8.1f} ms  mean dev_ms/solve={dm.mean():7.2f}    its={it.mean():.0f} power_steps={pw.mean():.0f} "
          f"A={pr[:,0].mean()/1e6:.2f} B={pr[:,1].mean()/1e6:.2f} E={pr[:,2].mean()/1e6:.2f} pw={pr[:,3].mean()/1e6:.2f} ms")
