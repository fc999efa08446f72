"""c4 path: per-lambda phase split (A pass, B, D/E, power) against the iteration count,
mean preserved-set size and mean nnz of x (where the apply u = A x_next spends)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch
import bench
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
At, y = bench.make_c4_device(4, "cuda")
k, n = At.shape
d = F.DenseDictionaryDevice(At.data_ptr(), n, k)
del At
torch.cuda.empty_cache()
lmax = F.lambda_max(d, y); L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
yd = torch.from_numpy(y).cuda()
for rep in range(2):
    x = None
    for i, r in enumerate(syn.CONFIGS["c4"]["lam_ratios"]):
        res = F.run_lasso_device(seq, yd.data_ptr(), r * lmax, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], x_init=x))
        x = res.x
        if rep == 1:
            p = res.profile; tr = res.trace
            print(f"lam{i}: its {res.iterations:4d} S_mean {tr['active_size'].mean():8.0f} nnz_mean {tr['x_nnz'].mean():6.0f} "
                  f"A {p[0]/1e6:6.1f} B {p[1]/1e6:5.1f} DE {p[2]/1e6:5.1f} ({p[2]/1e3/res.iterations:5.1f} us/it, apply GB {p[6]/1e9:5.1f}) power {p[3]/1e6:6.1f} ms")
