import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
inst = syn.sukro_instance(seed=3)
seq = syn.sukro_sequence(inst)
Ls = [F.lipschitz_bound(dd.op) for dd in seq.dicts]
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6, gamma_threshold=0.5)
for fl in (Ls, None):
    opts = F.RunOptions(variant=F.VARIANT_MULTI_DICT, full_lipschitz=fl)
    for _ in range(2):
        r = F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
    p = r.profile
    tr = r.trace
    print('full_lipschitz' if fl else 'no cached L', 'device', round(r.device_ms, 3), 'its', r.iterations, 'power steps', r.power_iterations,
          'phases A/B/D/power/switch ms', np.round(p[:5] / 1e6, 3), 'power sub (apply, combine, adjoint, reduce) ms', np.round(p[8:12] / 1e6, 3))
    print('  switches', [(int(e['iter']), int(e['from']), int(e['to'])) for e in r.switches], 'S at switches', [int(tr['active_size'][int(e['iter'])]) for e in r.switches])
    print('  S trajectory', tr['active_size'][::5].tolist())
