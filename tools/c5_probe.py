"""c5 per-signal shape: iterations, preserved-set sizes, power steps, and where the batch's
time goes (lockstep launch vs the per-signal cluster engines)."""
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
for _ in range(3):
    rs = F.run_lasso_batched(seq, (n, B), lams, cfg, opts, 0, y_dev_ptr=Yd.data_ptr())
pr = rs[0].profile
print('batch ms %.2f lockstep ms %.2f steps %d sum_act %d sum_pow %d' % (rs[0].batch_device_ms, pr[0], pr[3], pr[1], pr[2]))
its = np.array([r.iterations for r in rs]); pw = np.array([r.power_iterations for r in rs])
s10 = np.array([r.trace['active_size'][min(11, len(r.trace) - 1)] for r in rs])
send = np.array([r.trace['active_size'][-1] for r in rs]); dev = np.array([r.device_ms for r in rs])
for name, v in (('iterations', its), ('power steps', pw), ('|S| after first screen', s10), ('|S| final', send), ('device ms', dev)):
    print('%-24s min %8.1f p50 %8.1f p90 %8.1f max %8.1f' % (name, v.min(), np.median(v), np.percentile(v, 90), v.max()))
o = np.argsort(-dev)[:10]
for b in o:
    print('slow signal %3d: its %4d power %4d S11 %5d Send %5d dev_ms %.2f' % (b, its[b], pw[b], s10[b], send[b], dev[b]))
