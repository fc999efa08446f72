"""c5: work done by the per-signal engines after the lockstep hand-off (policy 3), from the
trace wall clock: per signal, the iterations from the first one after its cold power
iteration (the largest wall-clock gap) with |S| <= FL1_HANDOFF_S, their summed time and
preserved-set sizes."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np, torch
import bench
from paper_1812_06635_b200 import fastl1 as F
a, Y, lams = bench.make_c5(5)
n, k = a.shape; B = Y.shape[1]
d = F.DenseDictionary(a); L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], collect_trace=True)
Yd = torch.from_numpy(np.ascontiguousarray(Y.T)).cuda()
for _ in range(2):
    rs = F.run_lasso_batched(seq, (n, B), lams, cfg, opts, 0, y_dev_ptr=Yd.data_ptr())
pr = rs[0].profile
print('batch', rs[0].batch_device_ms, 'lockstep ms', pr[0])
its_after, t_after, s_first, s_mean = [], [], [], []
for r in rs:
    w = r.trace['wall_ms']; S = r.trace['active_size']
    if len(w) < 2:
        continue
    dw = np.diff(w)
    g0 = int(np.argmax(dw)) + 1  # the first (cold) power iteration ends here
    hs = np.nonzero(S[g0:] <= int(os.environ.get("FL1_HANDOFF_S", "512")))[0]
    if len(hs) == 0:
        continue
    g = g0 + int(hs[0])  # hand-off: the first iteration after it with |S| <= the threshold
    its_after.append(len(w) - g)
    t_after.append(w[-1] - w[g])
    s_first.append(S[g]); s_mean.append(S[g:].mean())
its_after, t_after, s_first = map(np.array, (its_after, t_after, s_first))
print(f"signals {len(t_after)}: iterations after hand-off mean {its_after.mean():.1f} (max {its_after.max()}), "
      f"engine time per signal mean {t_after.mean():.3f} ms (p90 {np.percentile(t_after, 90):.3f}, max {t_after.max():.3f}), "
      f"sum {t_after.sum():.1f} ms -> /148 = {t_after.sum() / 148:.2f} ms")
print(f"S at the first engine iteration: p10 {np.percentile(s_first, 10):.0f} p50 {np.median(s_first):.0f} "
      f"p90 {np.percentile(s_first, 90):.0f} max {s_first.max()}; us per engine iteration mean "
      f"{1e3 * t_after.sum() / max(its_after.sum(), 1):.1f}")
