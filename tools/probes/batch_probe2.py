"""c5 batched path: wall vs batch device time vs Python collection, per mode."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np, torch
import bench
from paper_1812_06635_b200 import fastl1 as F
a, Y, lams = bench.make_c5(5)
n, k = a.shape; B = Y.shape[1]
d = F.DenseDictionary(a); L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L])
Yd = torch.from_numpy(np.ascontiguousarray(Y.T)).cuda()
for M in [int(v) for v in os.environ.get('MODES', '-2,-4').split(',')]:
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        rs = F.run_lasso_batched(seq, (n, B), lams, cfg, opts, M, y_dev_ptr=Yd.data_ptr())
        w = time.perf_counter() - t
        dm = np.array([r.device_ms for r in rs])
        print(f"M={M} rep {rep}: wall {w*1e3:7.1f} ms  batch_device {rs[0].batch_device_ms:7.1f} ms  "
              f"mean signal dev {dm.mean():6.2f} max {dm.max():6.2f}  its {sum(r.iterations for r in rs)} "
              f"power {np.mean([r.power_iterations for r in rs]):.0f}")
order = np.argsort([-r.device_ms for r in rs])[:6]
for b in order:
    r = rs[b]
    print(f"slow signal {b}: dev {r.device_ms:.2f} ms its {r.iterations} power {r.power_iterations} "
          f"final_active {len(r.final_active)} nnz {np.count_nonzero(r.x)} profile(ms) {np.round(r.profile[:4]/1e6,2)}")
its = np.array([r.iterations for r in rs]); pw = np.array([r.power_iterations for r in rs])
print("iterations pct 50/90/99/max", np.percentile(its, [50, 90, 99, 100]), "power", np.percentile(pw, [50, 90, 99, 100]))
