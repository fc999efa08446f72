"""Direct vs Gram-backed exact phase on BASELINE c1 / c2 (device time per solve)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
for name in ("c1", "c2"):
    inst = syn.dense_instance(name)
    d = F.DenseDictionary(inst.a)
    L = F.lipschitz_bound(d)
    seq = F.ApproxSequence([F.make_exact_approx(d)])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    t = time.perf_counter(); g = F.gram_matrix(d); tg = time.perf_counter() - t
    for label, gram in (("direct", None), ("gram", g)):
        opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], exact_gram=gram)
        F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
        ms = [F.run_lasso(seq, inst.y, inst.lam, cfg, opts).device_ms for _ in range(5)]
        r = F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
        print(f"{name} {label:6s} device {np.mean(ms):7.3f} ms  its {r.iterations}  gap {r.final_gap:.3e}  (G build {tg*1e3:.1f} ms wall)")
