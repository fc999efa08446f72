"""Lockstep batched engine: per-step occupancy / time (FL1_STEP_LOG diagnostics)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
os.environ['FL1_STEP_LOG'] = '/tmp/fl1_steps.txt'
import numpy as np, torch
import bench
from paper_1812_06635_b200 import fastl1 as F
a, Y, lams = bench.make_c5(5)
n, k = a.shape; B = Y.shape[1]
d = F.DenseDictionary(a); L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L])
Yd = torch.from_numpy(np.ascontiguousarray(Y.T)).cuda()
for _ in range(2):
    rs = F.run_lasso_batched(seq, (n, B), lams, cfg, opts, -2, y_dev_ptr=Yd.data_ptr())
lg = np.loadtxt('/tmp/fl1_steps.txt')
t = lg[:, 2] / 1e6
dt = np.diff(t)
gn = (lg[:, 3] - lg[:, 2]) / 1e3   # us: power contraction W = A V + combine
gt = (lg[:, 4] - lg[:, 3]) / 1e3   # us: A^T R contraction
print('batch ms', rs[0].batch_device_ms, 'steps', len(lg), 'lockstep ms', t[-1])
if lg.shape[1] >= 9:  # stream-K route: CTA 0's own completion times inside the step (us from the step start)
    st = lg[:, 2]
    rel = lambda c: np.where(lg[:, c] > 0, (lg[:, c] - st) / 1e3, np.nan)
    stg, wd, wb, cd, cb, pd = rel(5), rel(6), rel(3), rel(7), rel(4), rel(8)
    nxt = np.append((lg[1:, 2] - st[:-1]) / 1e3, np.nan)
    for lo, hi in [(0, 40), (40, 80), (80, 120), (120, 160), (160, 200), (200, 240)]:
        sel = slice(lo, min(hi, len(lg) - 1))
        m = lambda x: np.nanmean(x[sel])
        print(f"  steps {lo:3d}-{hi:3d}: staged {m(stg):6.1f} | CTA0 W done {m(wd):6.1f} W barrier {m(wb):6.1f} | "
              f"CTA0 Corr done {m(cd):6.1f} Corr barrier {m(cb):6.1f} | CTA0 per-signal done {m(pd):6.1f} next step {m(nxt):6.1f}")
for lo, hi in [(0, 40), (40, 80), (80, 120), (120, 160), (160, 200), (200, 240), (240, 300)]:
    sel = slice(lo, min(hi, len(dt)))
    if lo >= len(dt): break
    print(f"steps {lo:3d}-{hi:3d}: n_act {lg[sel,0].mean():6.1f} n_pow {lg[sel,1].mean():6.1f} us/step {dt[sel].mean()*1e3:7.1f} "
          f"[W=AV {gn[sel].mean():6.1f}  A^T R {gt[sel].mean():6.1f}  per-signal {dt[sel].mean()*1e3-gn[sel].mean()-gt[sel].mean():6.1f}] total ms {dt[sel].sum():6.2f}")
