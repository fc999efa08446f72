import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
os.environ['FL1_LIB'] = '/root/repo/paper_1812_06635_b200/_build/libfl1cuda_timeline.so'
os.environ['FL1_TIMELINE_OUT'] = '/tmp/fl1_timeline.bin'
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
name = sys.argv[1]
if name == 'c3':
    inst = syn.sukro_instance(seed=3)
    seq = syn.sukro_sequence(inst)
    Ls = [F.lipschitz_bound(dd.op) for dd in seq.dicts]
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6, gamma_threshold=0.5)
    opts = F.RunOptions(variant=F.VARIANT_MULTI_DICT, full_lipschitz=Ls, collect_trace=True)
    its = range(22, 40)
else:
    inst = syn.dense_instance(name)
    d = F.DenseDictionary(inst.a); L = F.lipschitz_bound(d)
    seq = F.ApproxSequence([F.make_exact_approx(d)])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], collect_trace=True)
    its = range(2, 60)
F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
out = F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
raw = np.fromfile('/tmp/fl1_timeline.bin', dtype=np.uint64); G = raw.size // (4096 * 8)
tl = raw.reshape(4096, G, 8).astype(np.float64)
W = np.array([tl[t, :, 1] - tl[t, :, 0] for t in its]) / 1e3   # per-CTA A work, us
print(name, "A work per CTA: mean %.1f  min %.1f  max %.1f  (per-iteration max-min avg %.1f)" % (
    W.mean(), W.min(axis=1).mean(), W.max(axis=1).mean(), (W.max(axis=1) - W.min(axis=1)).mean()))
cm = W.mean(axis=0)
order = np.argsort(cm)
print("slowest CTAs (mean us):", [(int(i), round(cm[i], 1)) for i in order[-8:]])
print("fastest CTAs (mean us):", [(int(i), round(cm[i], 1)) for i in order[:8]])
a, b = W[::2].mean(axis=0), W[1::2].mean(axis=0)
print("corr(even its, odd its) of per-CTA time: %.3f" % np.corrcoef(a, b)[0, 1])
# start skew: per-CTA start mark relative to the earliest
st = np.array([tl[t, :, 0] - tl[t, :, 0].min() for t in its]) / 1e3
print("start skew mean %.2f max %.2f" % (st.mean(), st.max(axis=1).mean()))
