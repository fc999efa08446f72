"""Per-phase timeline of the c3 (SuKro switching) solve, instrumented build."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
import numpy as np
os.environ['FL1_LIB'] = os.path.join(os.path.dirname(__file__), '..', 'paper_1812_06635_b200/_build/libfl1cuda_timeline.so')
os.environ['FL1_TIMELINE_OUT'] = '/tmp/fl1_timeline.bin'
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
inst = syn.sukro_instance(seed=3)
seq = syn.sukro_sequence(inst)
Ls = [F.lipschitz_bound(dd.op) for dd in seq.dicts]
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6, gamma_threshold=0.5)
opts = F.RunOptions(variant=F.VARIANT_MULTI_DICT, full_lipschitz=Ls, collect_trace=True)
F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
out = F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
G = 148
tl = np.fromfile('/tmp/fl1_timeline.bin', dtype=np.uint64).reshape(4096, G, 8).astype(np.float64)
its = out.iterations
names = ['A work', 'sync1', 'B work', 'sync2', 'E work', 'sync3', 'tail->next A']
print(f"c3: {its} iterations, device {out.device_ms:.3f} ms, power steps {out.power_iterations}, profile {np.round(out.profile[:5]/1e6,3)}")
di = out.trace['dict_index']
for t in range(min(its - 1, 40)):
    m = tl[t]
    nxt = tl[t + 1, :, 0]
    seg = [m[:, 1] - m[:, 0], m[:, 2] - m[:, 1], m[:, 3] - m[:, 2], m[:, 4] - m[:, 3], m[:, 5] - m[:, 4],
           m[:, 6] - m[:, 5], nxt - m[:, 6]]
    print(f"it {t:3d} lvl {di[t]} S {out.trace['active_size'][t]:6d} " + " ".join(f"{nm.split()[0]}={s.max()/1e3:7.1f}" for nm, s in zip(names, seg)))
