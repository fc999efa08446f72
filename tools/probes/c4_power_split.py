import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np, torch
import bench
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
At, y = bench.make_c4_device(4, "cuda")
k, n = At.shape
d = F.DenseDictionaryDevice(At.data_ptr(), n, k); del At; torch.cuda.empty_cache()
lmax = F.lambda_max(d, y); L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
yd = torch.from_numpy(y).cuda()
for rep in range(2):
    x = None; tot = np.zeros(14)
    for r in syn.CONFIGS["c4"]["lam_ratios"]:
        res = F.run_lasso_device(seq, yd.data_ptr(), r * lmax, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], x_init=x))
        x = res.x; tot += res.profile
pb = tot[7]
print("power ms %.1f: apply %.1f combine %.1f adjoint %.1f reduce %.1f ms; power bytes %.1f GB -> apply+adjoint %.2f TB/s"
      % (tot[3] / 1e6, tot[8] / 1e6, tot[9] / 1e6, tot[10] / 1e6, tot[11] / 1e6, pb / 1e9, pb / ((tot[8] + tot[10]) * 1e-9) / 1e12))
print("apply alone %.2f TB/s, adjoint alone %.2f TB/s (half the bytes each)" % (pb / 2 / (tot[8] * 1e-9) / 1e12, pb / 2 / (tot[10] * 1e-9) / 1e12))
