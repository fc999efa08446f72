"""L = 1.05 sigma_max^2 through the power-iteration utility launch, fused (single-read) steps against numpy."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np
from paper_1812_06635_b200 import fastl1 as F
n, k = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(1)
a = rng.standard_normal((n, k)); a /= np.linalg.norm(a, axis=0); a = np.asfortranarray(a)
d = F.DenseDictionary(a)
t = time.time(); L = F.lipschitz_bound(d); el = time.time() - t
ref = 1.05 * np.linalg.norm(a, 2) ** 2
print(f"n {n} k {k} FUSED_MB {os.environ.get('FL1_FUSED_POWER_MB')} L {L!r} ref {ref!r} rel {abs(L - ref) / ref:.2e} time {el:.3f}s", flush=True)
