"""Batched call beyond the lockstep's shared memory (6,000 small signals): convergence and
oracle agreement of the per-signal engine route."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np
from pathlib import Path
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn, _abi
B = int(sys.argv[1]) if len(sys.argv) > 1 else 6000
rng = np.random.default_rng(43)
n, k = 48, 96
a = syn.gaussian_dictionary(rng, n, k)
X0 = np.zeros((k, B))
for b in range(B):
    X0[rng.choice(k, 3, replace=False), b] = rng.standard_normal(3)
Y = np.asfortranarray(a @ X0 + 0.01 * rng.standard_normal((n, B)))
lams = 0.3 * np.max(np.abs(a.T @ Y), axis=0)
d = F.DenseDictionary(a)
L = F.lipschitz_bound(d)
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L])
res = F.run_lasso_batched(F.ApproxSequence([F.make_exact_approx(d)]), Y, lams, cfg, opts, concurrency=0)
bad = [b for b, r in enumerate(res) if not r.converged]
print('B', B, 'not converged', len(bad), bad[:10], 'iterations of the first', [res[b].iterations for b in bad[:5]],
      'gaps', [res[b].final_gap for b in bad[:5]], 'launches', res[0].kernel_launches)
orc = F.Backend(_abi.Library(Path(__file__).resolve().parents[2] / 'oracle/_build/libfl1oracle.so', 'orc_', extra=_abi.ORACLE_ONLY))
seq_o = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=orc))])
for b in bad[:3]:
    o = F.run_lasso(seq_o, Y[:, b], lams[b], cfg, opts)
    print('oracle', b, o.converged, o.iterations, o.final_gap, '| gpu', res[b].iterations, res[b].final_gap)
