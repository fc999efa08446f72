"""c1 per-iteration wall time on the grid route vs the single-cluster route (trace wall_ms)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import subprocess
code = r'''
import os, sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
inst = syn.dense_instance("c1")
d = F.DenseDictionary(inst.a); L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], collect_trace=True)
for _ in range(3): r = F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
w = r.trace["wall_ms"]; dw = np.diff(np.concatenate([[0.0], w])) * 1e3
print(os.environ.get("FL1_SINGLE_CLUSTER", "1"), "device %.3f ms" % r.device_ms, "power steps", r.power_iterations,
      "profile", np.round(r.profile[:5] / 1e3, 1))
print("  us per iteration:", np.round(dw).astype(int).tolist())
print("  S:", r.trace["active_size"].tolist())
'''
root = os.path.join(os.path.dirname(__file__), '..', '..')
for v in ("1", "0"):
    env = dict(os.environ, FL1_SINGLE_CLUSTER=v)
    print(subprocess.run([sys.executable, "-c", code, root], env=env, capture_output=True, text=True).stdout)
