"""Cold restricted power iteration on dense 2500 x K dictionaries: per-step phase times (FL1_UTIL_LOG)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
os.environ['FL1_UTIL_LOG'] = '1'
import numpy as np
from paper_1812_06635_b200 import fastl1 as F
rng = np.random.default_rng(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2500
for k in [10000, 5000, 2876, 1000, 643]:
    a = rng.standard_normal((n, k)); a /= np.linalg.norm(a, axis=0)
    d = F.DenseDictionary(a)
    for r in range(3):
        t0 = time.perf_counter(); L = F.lipschitz_bound(d); t1 = time.perf_counter()
    print(f"n={n} k={k} L={L:.6f} wall {1e3*(t1-t0):.3f} ms", flush=True)
