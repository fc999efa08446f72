"""Power phase in isolation: the engine's power iteration (utility launch, fl1_lipschitz_bound) over a
2500 x S column subset of c2's dictionary -- the restricted power steps of a c2 solve at |S| = S
(L2-resident for S <= ~6000).  FL1_UTIL_LOG=1 prints the sub-phase times of every launch; under ncu
(-k regex:engine_kernel --launch-skip 2 --launch-count 1) the capture holds the power phase alone."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
import numpy as np
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
S = int(sys.argv[1]) if len(sys.argv) > 1 else 2876
inst = syn.dense_instance('c2')
rng = np.random.default_rng(7)
cols = np.sort(rng.choice(inst.a.shape[1], S, replace=False))
d = F.DenseDictionary(np.asfortranarray(inst.a[:, cols]))
for rep in range(4):
    t0 = time.perf_counter()
    L = F.lipschitz_bound(d)
    print(f"S {S} rep {rep}: L bound {L:.12f} host {1e3 * (time.perf_counter() - t0):.3f} ms", flush=True)
