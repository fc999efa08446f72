"""Per-phase timeline of a dense solve (c1 on the single-cluster route, or c2 with FL1_SINGLE_CLUSTER=0), instrumented build."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
import numpy as np
os.environ['FL1_LIB'] = os.path.join(os.path.dirname(__file__), '..', 'paper_1812_06635_b200/_build/libfl1cuda_timeline.so')
os.environ['FL1_TIMELINE_OUT'] = '/tmp/fl1_timeline.bin'
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
name = sys.argv[1] if len(sys.argv) > 1 else 'c1'
inst = syn.dense_instance(name)
d = F.DenseDictionary(inst.a); L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], collect_trace=True)
F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
out = F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
raw = np.fromfile('/tmp/fl1_timeline.bin', dtype=np.uint64)
G = raw.size // (4096 * 8)
tl = raw.reshape(4096, G, 8).astype(np.float64)
its = out.iterations
names = ['A', 'sync1', 'Bscal', 'Bapply', 'sync2', 'E', 'sync3', 'tail']
print(f"{name}: {its} iterations, CTAs {G}, device {out.device_ms:.3f} ms, power steps {out.power_iterations}, "
      f"profile {np.round(out.profile[:5]/1e6,3)}")
tot = np.zeros(8)
for t in range(its - 1):
    m = tl[t]
    nxt = tl[t + 1, :, 0]
    seg = [m[:, 1] - m[:, 0], m[:, 2] - m[:, 1], m[:, 3] - m[:, 2], m[:, 4] - m[:, 3], m[:, 5] - m[:, 4],
           m[:, 6] - m[:, 5], nxt - m[:, 6]]
    # wall-clock segment lengths: max over CTAs of the end mark minus max of the start mark
    mx = [np.max(m[:, 1]) - np.max(m[:, 0]), np.max(m[:, 2]) - np.max(m[:, 1]), np.max(m[:, 7]) - np.max(m[:, 2]),
          np.max(m[:, 3]) - np.max(m[:, 7]),
          np.max(m[:, 4]) - np.max(m[:, 3]), np.max(m[:, 5]) - np.max(m[:, 4]), np.max(m[:, 6]) - np.max(m[:, 5]),
          np.max(nxt) - np.max(m[:, 6])]
    tot += np.array(mx)
    if t < 12 or t % 10 == 9 or t > its - 6:
        print(f"it {t:3d} S {out.trace['active_size'][t]:6d} " + " ".join(
            f"{nm}={v/1e3:6.1f}" for nm, v in zip(names, mx)) + "  | mean CTA A work %.1f" % (seg[0].mean() / 1e3))
print("totals ms:", " ".join(f"{nm}={v/1e6:.3f}" for nm, v in zip(names, tot)))
