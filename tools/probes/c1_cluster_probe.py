"""c1 single solve: full cooperative grid vs one thread-block cluster (batched entry, B = 1)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
os.environ["FL1_BATCH_PREFIX"] = "0"
for name in ("c1", "c2"):
    inst = syn.dense_instance(name)
    d = F.DenseDictionary(inst.a)
    L = F.lipschitz_bound(d)
    seq = F.ApproxSequence([F.make_exact_approx(d)])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L])
    F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
    print(name, "grid  ", np.mean([F.run_lasso(seq, inst.y, inst.lam, cfg, opts).device_ms for _ in range(5)]))
    Y = inst.y.reshape(-1, 1)
    for cs in (4, 8, 16):
        try:
            F.run_lasso_batched(seq, Y, [inst.lam], cfg, opts, concurrency=-cs)
            r = [F.run_lasso_batched(seq, Y, [inst.lam], cfg, opts, concurrency=-cs)[0] for _ in range(3)]
            print(name, f"cl{cs:2d} ", np.mean([x.device_ms for x in r]), "batch", np.mean([x.batch_device_ms for x in r]))
        except Exception as e:
            print(name, cs, "ERR", e)
