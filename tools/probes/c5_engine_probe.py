"""c5 signals on the per-signal engines only (FL1_BATCH_PREFIX=0; cluster size from argv):
per-signal device time against iterations and power steps -> cost per iteration."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
os.environ['FL1_BATCH_PREFIX'] = '0'
import numpy as np, torch
import bench
from paper_1812_06635_b200 import fastl1 as F
cs = int(sys.argv[1]) if len(sys.argv) > 1 else 1
a, Y, lams = bench.make_c5(5)
n, k = a.shape; B = Y.shape[1]
d = F.DenseDictionary(a); L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], collect_trace=True)
Yd = torch.from_numpy(np.ascontiguousarray(Y.T)).cuda()
for _ in range(2):
    rs = F.run_lasso_batched(seq, (n, B), lams, cfg, opts, -cs, y_dev_ptr=Yd.data_ptr())
its = np.array([r.iterations for r in rs]); pw = np.array([r.power_iterations for r in rs]); dev = np.array([r.device_ms for r in rs])
S = np.array([r.trace['active_size'].mean() for r in rs])
print(f"cluster {cs}: batch {rs[0].batch_device_ms:.2f} ms; per signal: its {its.mean():.1f} power {pw.mean():.1f} "
      f"mean|S| {S.mean():.0f} device {dev.mean():.3f} ms -> {dev.mean() * 1e3 / (its.mean() + pw.mean()):.1f} us per (iteration + power step)")
A = np.vstack([its, pw]).T
coef, *_ = np.linalg.lstsq(A, dev * 1e3, rcond=None)
print(f"  least squares: {coef[0]:.1f} us per iteration, {coef[1]:.1f} us per power step")
