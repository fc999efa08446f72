"""GPU (fused single-read power steps forced by FL1_FUSED_POWER_MB=1) vs the oracle on tall dictionaries (4096 < n <= 8192)."""
import os, sys, time
ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), '..', '..')
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'tests'))
import numpy as np
import _fuzz
from _parity import assert_parity
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
gpu, orc = F.default_backend(), _fuzz.oracle_backend()
CASES = ((4200, 1500, 40, 0.3), (8192, 1200, 60, 0.2), (5000, 3000, 100, 0.1), (6001, 2000, 30, 0.5))
if len(sys.argv) > 1 and sys.argv[1] == "edges":  # unit-count and padding edges: 9 units with a 16-double tail, 8191, 4609, few columns
    CASES = ((4097, 900, 20, 0.3), (8191, 700, 25, 0.2), (4609, 1100, 30, 0.15), (7777, 150, 10, 0.4), (4608, 2000, 50, 0.25))
for n, k, nnz, ratio in CASES:
    inst = syn.dense_instance("c1", seed=n, n=n, k=k, nnz=nnz)
    lam = ratio * inst.lam_max if hasattr(inst, "lam_max") else inst.lam
    res = {}
    for tag, b in (("gpu", gpu), ("orc", orc)):
        d = F.DenseDictionary(inst.a, backend=b)
        seq = F.ApproxSequence([F.make_exact_approx(d)])
        cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
        t = time.time()
        res[tag] = F.run_lasso(seq, inst.y, lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED))
        el = time.time() - t
        if tag == "gpu":
            L = F.lipschitz_bound(d)
    g, o = res["gpu"], res["orc"]
    assert_parity(g, o, inst.a, inst.y, lam, case="fused-power", gap_ulps=_fuzz.FUZZ_GAP_ULPS)
    print(f"ok n {n} k {k}: iterations {g.iterations} power steps {g.power_iterations} final |S| {g.final_active.size} "
          f"device {g.device_ms:.2f} ms L {L!r}", flush=True)
