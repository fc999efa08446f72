"""Small solves over every engine route, for compute-sanitizer (memcheck / racecheck /
synccheck): grid mode (bulk-ring power iterations), single cluster, SuKro switching,
Gram mode, lockstep batched + cluster hand-off. Each result is checked for convergence."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn

cfg = F.SwitchConfig(screening_interval=10, max_iterations=3000, rel_tolerance=1e-6)
inst = syn.dense_instance("c1", seed=21, n=300, k=1200, nnz=20)
d = F.DenseDictionary(inst.a)
L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
for route in ("grid", "cluster"):
    os.environ["FL1_SINGLE_CLUSTER"] = "0" if route == "grid" else "1"
    r = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L],
                                                                collect_trace=True))
    assert r.converged, route
    print(route, "ok", r.iterations, r.power_iterations)
os.environ["FL1_SINGLE_CLUSTER"] = "0"
g = F.gram_matrix(d)
r = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], exact_gram=g))
assert r.converged
print("gram ok", r.iterations)
si = syn.sukro_instance(seed=4, m=16, q=32, terms=4, levels=(1, 2), nnz=30)
sseq = syn.sukro_sequence(si)
Ls = [F.lipschitz_bound(dd.op) for dd in sseq.dicts]
r = F.run_lasso(sseq, si.y, si.lam, F.SwitchConfig(screening_interval=10, max_iterations=3000, rel_tolerance=1e-6,
                                                   gamma_threshold=0.5),
                F.RunOptions(variant=F.VARIANT_MULTI_DICT, full_lipschitz=Ls))
assert r.converged
print("sukro ok", r.iterations, r.switches)
rng = np.random.default_rng(3)
B = 24
Y = inst.a[:, rng.choice(inst.a.shape[1], 8)] @ rng.standard_normal((8, B)) + 0.01 * rng.standard_normal((inst.a.shape[0], B))
lams = 0.25 * np.max(np.abs(inst.a.T @ Y), axis=0)
rs = F.run_lasso_batched(seq, Y, lams, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L]), -2)
assert all(x.converged for x in rs)
print("batched ok", sum(x.iterations for x in rs))
