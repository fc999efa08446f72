"""One c5 signal solved on a one-CTA engine (single-cluster route forced, cluster size 1),
instrumented build: per-phase times at small preserved sets."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
os.environ['FL1_LIB'] = os.path.join(os.path.dirname(__file__), '..', '..', 'paper_1812_06635_b200/_build/libfl1cuda_timeline.so')
os.environ['FL1_TIMELINE_OUT'] = '/tmp/fl1_timeline.bin'
os.environ['FL1_SINGLE_CLUSTER_MB'] = '64'
os.environ['FL1_SINGLE_CLUSTER_SIZE'] = sys.argv[1] if len(sys.argv) > 1 else '1'
import numpy as np
import bench
from paper_1812_06635_b200 import fastl1 as F
a, Y, lams = bench.make_c5(5)
d = F.DenseDictionary(a); L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], collect_trace=True)
b = 0
out = F.run_lasso(seq, Y[:, b], lams[b], cfg, opts)
out = F.run_lasso(seq, Y[:, b], lams[b], cfg, opts)
raw = np.fromfile('/tmp/fl1_timeline.bin', dtype=np.uint64)
G = raw.size // (4096 * 8)
tl = raw.reshape(4096, G, 8).astype(np.float64)
names = ['A', 'sync1', 'Bscal', 'Bapply', 'sync2', 'E', 'sync3', 'tail']
print(f"signal {b}: {out.iterations} its, CTAs {G}, device {out.device_ms:.3f} ms, power {out.power_iterations}, profile {np.round(out.profile[:5]/1e6,3)}")
for t in range(out.iterations - 1):
    m = tl[t]; nxt = tl[t + 1, :, 0]
    mx = [np.max(m[:, 1]) - np.max(m[:, 0]), np.max(m[:, 2]) - np.max(m[:, 1]), np.max(m[:, 7]) - np.max(m[:, 2]),
          np.max(m[:, 3]) - np.max(m[:, 7]), np.max(m[:, 4]) - np.max(m[:, 3]), np.max(m[:, 5]) - np.max(m[:, 4]),
          np.max(m[:, 6]) - np.max(m[:, 5]), np.max(nxt) - np.max(m[:, 6])]
    if t in (1, 5, 9, 15, 25, 35, 45, 50) or t > out.iterations - 3:
        print(f"it {t:3d} S {out.trace['active_size'][t]:5d} nnz {out.trace['x_nnz'][t]:4d} " + " ".join(f"{nm}={v/1e3:6.1f}" for nm, v in zip(names, mx)))
