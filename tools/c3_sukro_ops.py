"""Isolated SuKro products of config 3 (Kronecker-sum levels of 1 / 2 / 4 terms, 4096 x
16384): the adjoint Z = sum_t C_t^T R B_t and the apply on the device, one engine launch
each (utility modes), for an ncu capture of the DMMA contraction alone; prints the
launch times and the SURVEY 8(d) flops (2 * matvec_flops per product)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_1812_06635_b200 import fastl1 as F, synthetic as syn  # noqa: E402

inst = syn.sukro_instance(seed=3)
seq = syn.sukro_sequence(inst)
rng = np.random.default_rng(0)
r = rng.standard_normal(inst.a.shape[0])
x = np.zeros(inst.a.shape[1])
x[rng.choice(x.size, 400, replace=False)] = rng.standard_normal(400)
for lv in seq.dicts[:-1]:
    op = lv.op
    for _ in range(3):
        op.apply_adjoint(r)
        op.apply(x)
    t = time.perf_counter()
    for _ in range(20):
        op.apply_adjoint(r)
    ta = (time.perf_counter() - t) / 20
    print(f"terms {len(op._keep[0])}: matvec_flops {op.matvec_flops()} "
          f"adjoint host-timed {ta * 1e6:.1f} us/call (incl. launch + copies)")
