"""Per-phase time of CTA 0's per-signal FISTA steps in the lockstep (FL1_SIGPROF build)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
os.environ['FL1_SIGPROF_OUT'] = '/tmp/sigprof.txt'
import numpy as np, torch
sys.argv = [sys.argv[0]]
from paper_1812_06635_b200 import _abi
_abi.PRODUCT_ONLY.pop("build_sukro_sequence", None) if False else None
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
    rs = F.run_lasso_batched(seq, (n, B), lams, cfg, opts, 0, y_dev_ptr=Yd.data_ptr())
v = np.loadtxt('/tmp/sigprof.txt')
cnt = v[13]
names = ['sum_parts+max', 'scalars', 'prox+lists+sum3', 'fix apply', 'u = A x', 'bookkeeping+rho']
print('CTA 0 FISTA steps:', int(cnt), 'batch ms', rs[0].batch_device_ms)
for i, nm in enumerate(names):
    print(f'  {nm:18s} {v[i] / cnt / 1e3:7.2f} us per step')
