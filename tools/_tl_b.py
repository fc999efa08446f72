import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
os.environ['FL1_LIB'] = '/root/repo/paper_1812_06635_b200/_build/libfl1cuda_timeline.so'
os.environ['FL1_TIMELINE_OUT'] = '/tmp/fl1_timeline.bin'
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
inst = syn.dense_instance('c2')
d = F.DenseDictionary(inst.a); L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], collect_trace=True)
F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
out = F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
raw = np.fromfile('/tmp/fl1_timeline.bin', dtype=np.uint64); G = raw.size // (4096 * 8)
tl = raw.reshape(4096, G, 8).astype(np.float64)
for t in [5, 20, 69, 80, 90, 95]:
    m = tl[t]; b = lambda k: m[:, k].max()
    print(t, "gridred %.2f scal %.2f prox %.2f blockred %.2f apply %.2f" % ((b(4)-b(2))/1e3, (b(5)-b(4))/1e3, (b(6)-b(5))/1e3, (b(7)-b(6))/1e3, (b(3)-b(7))/1e3),
          " mean: gridred %.2f scal %.2f prox %.2f" % ((m[:,4]-m[:,2]).mean()/1e3, (m[:,5]-m[:,4]).mean()/1e3, (m[:,6]-m[:,5]).mean()/1e3))
