"""Per-phase timeline of c4's lambda_9 solve (instrumented build: python
paper_1812_06635_b200/build.py --timeline). Wall-clock segment lengths per iteration:
max over CTAs of the end mark minus max of the start mark."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
import numpy as np
os.environ['FL1_LIB'] = os.path.join(os.path.dirname(__file__), '..', 'paper_1812_06635_b200/_build/libfl1cuda_timeline.so')
os.environ['FL1_TIMELINE_OUT'] = '/tmp/fl1_timeline.bin'
import torch
import bench
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
At, y = bench.make_c4_device(4, "cuda")
k, n = At.shape
d = F.DenseDictionaryDevice(At.data_ptr(), n, k)
del At
torch.cuda.empty_cache()
lmax = F.lambda_max(d, y); L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
x = None
for r in syn.CONFIGS["c4"]["lam_ratios"]:
    out = F.run_lasso(seq, y, r * lmax, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], x_init=x))
    x = out.x
raw = np.fromfile('/tmp/fl1_timeline.bin', dtype=np.uint64)
G = raw.size // (4096 * 8)
tl = raw.reshape(4096, G, 8).astype(np.float64)
its = out.iterations
names = ['A', 'sync1', 'Bscal', 'Bapply', 'sync2', 'E', 'sync3', 'tail']
print(f"lambda_9: {its} iterations, device {out.device_ms:.3f} ms, profile {np.round(out.profile[:5]/1e6,3)}")
tot = np.zeros(8)
for t in range(its - 1):
    m = tl[t]; nxt = tl[t + 1, :, 0]
    mx = [np.max(m[:, 1]) - np.max(m[:, 0]), np.max(m[:, 2]) - np.max(m[:, 1]), np.max(m[:, 7]) - np.max(m[:, 2]),
          np.max(m[:, 3]) - np.max(m[:, 7]), np.max(m[:, 4]) - np.max(m[:, 3]), np.max(m[:, 5]) - np.max(m[:, 4]),
          np.max(m[:, 6]) - np.max(m[:, 5]), np.max(nxt) - np.max(m[:, 6])]
    e_work = m[:, 5] - m[:, 4]
    tot += np.array(mx)
    if t % 20 == 9 or t > its - 4:
        print(f"it {t:3d} S {out.trace['active_size'][t]:6d} nnz {out.trace['x_nnz'][t]:5d} " + " ".join(
            f"{nm}={v/1e3:6.1f}" for nm, v in zip(names, mx)) + f" | E per-CTA min/mean/max {e_work.min()/1e3:.1f}/{e_work.mean()/1e3:.1f}/{e_work.max()/1e3:.1f}")
print("totals ms:", " ".join(f"{nm}={v/1e6:.3f}" for nm, v in zip(names, tot)))
