"""Round-2 code paths for compute-sanitizer: physical compaction + column-split apply
(grid route, N >= 4096), SuKro sequence construction on the device, device-side
ingestion (host and device input), lockstep width tiles / narrow steps / split budget."""
import os, sys
os.environ["FL1_COMPACT"] = "1"
os.environ["FL1_COLSPLIT"] = "1"
os.environ["FL1_SINGLE_CLUSTER"] = "0"
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np, torch
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn, harness as H

inst = syn.dense_instance("c1", seed=31, n=8192, k=600, nnz=12)
d = F.DenseDictionary(inst.a)
At = torch.from_numpy(np.ascontiguousarray(inst.a.T)).cuda()
dd = F.DenseDictionaryDevice(At.data_ptr(), inst.a.shape[0], inst.a.shape[1])
assert np.array_equal(d.atom_norms2(), dd.atom_norms2())
L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=5, max_iterations=2000, rel_tolerance=1e-6)
r = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L]))
assert r.converged
print("compact + colsplit ok", r.iterations, r.power_iterations)
a = syn.dense_instance("c1", seed=5, n=64, k=256, nnz=5).a
lv = H.build_sukro_levels(a, [1, 2, 4])
print("sukro build ok", [round(float(x.op_err), 6) for x in lv])
rng = np.random.default_rng(3)
n, k, B = 256, 512, 40
A2 = syn.gaussian_dictionary(rng, n, k)
Y = np.empty((n, B), order="F")
for b in range(B):
    Y[:, b] = syn.observe(rng, A2 @ syn.sparse_signal(rng, k, 3 + b % 5), None, 30.0)
lams = 0.25 * np.max(np.abs(A2.T @ Y), axis=0)
d2 = F.DenseDictionary(A2)
L2 = F.lipschitz_bound(d2)
rs = F.run_lasso_batched(F.ApproxSequence([F.make_exact_approx(d2)]), Y, lams, cfg,
                         F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L2]), 0)
assert all(x.converged for x in rs)
print("batched ok", sum(x.iterations for x in rs))
