"""Per-call wall time of the batched cluster path, device vs host Y, alternating."""
import os, sys, time
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
Yd = torch.from_numpy(np.ascontiguousarray(Y.T)).cuda()
M = int(os.environ.get('M', '0'))
for rep in range(6):
    for mode in ('dev', 'host'):
        torch.cuda.synchronize(); t = time.perf_counter()
        if mode == 'dev':
            rs = F.run_lasso_batched(seq, (n, B), lams, cfg, opts, M, y_dev_ptr=Yd.data_ptr())
        else:
            rs = F.run_lasso_batched(seq, Y, lams, cfg, opts, M)
        w = time.perf_counter() - t
        dm = np.array([r.device_ms for r in rs])
        print(f"rep {rep} {mode}: wall {w*1e3:7.1f} ms  sum dev {dm.sum():8.1f}  max dev {dm.max():6.2f} its {sum(r.iterations for r in rs)}")
