"""Per-CTA timeline of one lockstep step's stream-K products (FL1_SK_TRACE diagnostics):
for W and Corr, each CTA's start, end of its units and end of its reductions, relative to
the earliest start (us)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
step = int(sys.argv[1]) if len(sys.argv) > 1 else 200
os.environ['FL1_SK_TRACE'] = str(step)
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
for _ in range(2):
    F.run_lasso_batched(seq, (n, B), lams, cfg, opts, -2, y_dev_ptr=Yd.data_ptr())
raw = np.loadtxt('fl1_sk_trace.txt').reshape(-1)
t = raw[:2 * 256 * 4].reshape(2, 256, 4)
units = raw[2 * 256 * 4:].reshape(2, 4, 128, 2)  # [product][CTA 0-3][unit][before wait, after wait]
for w, name in ((0, 'W'), (1, 'Corr')):
    x = t[w, :148]
    if not x[:, 0].any():
        print(name, 'not run at step', step); continue
    t0 = x[:, 0].min()
    st, ud, en = (x[:, 0] - t0) / 1e3, (x[:, 1] - t0) / 1e3, (x[:, 2] - t0) / 1e3
    fl = np.where(x[:, 3] > 0, (x[:, 3] - t0) / 1e3, np.nan)  # flags waited (CTAs that reduce a shared tile)
    print(f"{name} step {step}: start max {st.max():.1f} us | units done min {ud.min():.1f} p50 {np.median(ud):.1f} max {ud.max():.1f} "
          f"| flags waited p50 {np.nanmedian(fl):.1f} max {np.nanmax(fl):.1f} | end min {en.min():.1f} p50 {np.median(en):.1f} max {en.max():.1f}")
    for g in range(2):
        u = units[w, g]
        m = u[:, 0] > 0
        if m.sum() > 1:
            aft = u[m, 1]
            per = np.diff(aft) / 1e3
            waits = (u[m, 1] - u[m, 0]) / 1e3
            print(f"   CTA {g}: {m.sum()} units, unit period p50 {np.median(per):.2f} us (min {per.min():.2f}, max {per.max():.2f}), "
                  f"full-barrier wait p50 {np.median(waits):.2f} us, first wait {waits[0]:.2f} us after start {(u[0, 0] - x[g, 0]) / 1e3:.2f} us")
    worst = np.argsort(-en)[:5]
    print('   slowest CTAs', worst.tolist(), 'units done', np.round(ud[worst], 1).tolist(), 'flags',
          np.round(fl[worst], 1).tolist(), 'end', np.round(en[worst], 1).tolist())
