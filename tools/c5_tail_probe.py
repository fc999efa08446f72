"""c5 default route: per-iteration wall-clock increments of a few signals after their
hand-off to the per-signal engines (trace wall_ms), to see the per-iteration cost at
small preserved sets."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
import numpy as np, torch
import bench
from paper_1812_06635_b200 import fastl1 as F
a, Y, lams = bench.make_c5(5)
n, k = a.shape; B = Y.shape[1]
d = F.DenseDictionary(a); L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], collect_trace=True)
Yd = torch.from_numpy(np.ascontiguousarray(Y.T)).cuda()
for _ in range(2):
    rs = F.run_lasso_batched(seq, (n, B), lams, cfg, opts, 0, y_dev_ptr=Yd.data_ptr())
pr = rs[0].profile
print('batch', rs[0].batch_device_ms, 'lockstep ms', pr[0])
ends = np.array([r.trace['wall_ms'][-1] for r in rs])
print('signal end wall_ms: min %.2f p50 %.2f p90 %.2f max %.2f' % (ends.min(), np.median(ends), np.percentile(ends, 90), ends.max()))
for b in list(np.argsort(-ends)[:3]) + [0]:
    tr = rs[b].trace
    w = tr['wall_ms']; dw = np.diff(w) * 1e3
    big = np.argmax(dw)
    print(f"signal {b}: its {rs[b].iterations} power {rs[b].power_iterations} end {w[-1]:.2f} ms; largest gap {dw[big]:.0f} us at it {big+1}")
    tail = dw[big + 1:]
    print("   after it: us per iteration", np.round(tail[:40]).astype(int).tolist(), "S", tr['active_size'][big+1:big+6].tolist())
