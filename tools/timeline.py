"""Analyse a per-CTA phase timeline dump (instrumented build, FL1_TIMELINE_OUT)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
import numpy as np
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
os.environ['FL1_LIB'] = os.path.join(os.path.dirname(__file__), '..', 'paper_1812_06635_b200/_build/libfl1cuda_timeline.so')
os.environ['FL1_TIMELINE_OUT'] = '/tmp/fl1_timeline.bin'
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
inst = syn.dense_instance(name)
d = F.DenseDictionary(inst.a)
L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
out = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L]))
G = 148
tl = np.fromfile('/tmp/fl1_timeline.bin', dtype=np.uint64).reshape(4096, G, 8).astype(np.float64)
its = out.iterations
tl = tl[:its]
names = ['A work', 'sync1', 'B work', 'sync2', 'E work', 'sync3', 'tail(power/switch)->next A']
print(f"{name}: {its} iterations, device {out.device_ms:.3f} ms")
rows = []
for t in range(its - 1):
    m = tl[t]
    nxt = tl[t + 1, :, 0]
    seg = [m[:, 1] - m[:, 0], m[:, 2] - m[:, 1], m[:, 3] - m[:, 2], m[:, 4] - m[:, 3], m[:, 5] - m[:, 4],
           m[:, 6] - m[:, 5], nxt - m[:, 6]]
    rows.append([(s.mean(), s.max(), s.min()) for s in seg])
rows = np.array(rows)  # its-1 x 7 x 3
S = out.trace['active_size'][:its - 1]
for label, mask in (('full set', S == S.max()), ('shrunk', S < S.max())):
    if mask.sum() == 0:
        continue
    r = rows[mask]
    print(f"  {label}: {mask.sum()} iterations; per-iteration us (mean over iters of [CTA mean / CTA max]):")
    for j, nm in enumerate(names):
        print(f"    {nm:28s} mean {r[:, j, 0].mean()/1e3:7.2f}  max {r[:, j, 1].mean()/1e3:7.2f}  min {r[:, j, 2].mean()/1e3:7.2f}")
