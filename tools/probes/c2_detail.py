import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
inst = syn.dense_instance(name)
d = F.DenseDictionary(inst.a); L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
for rep in range(3):
    out = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], collect_trace=True))
pr = out.profile
print(f"{name} it={out.iterations} dev_ms={out.device_ms:.3f} setup_ms={out.setup_ms:.3f} A={pr[0]/1e6:.3f} B={pr[1]/1e6:.3f} D={pr[2]/1e6:.3f} "
      f"power={pr[3]/1e6:.3f} ({out.power_iterations} steps) pw[apply,comb,adj,red]_ms={[round(v/1e6,3) for v in pr[8:12]]}")
s = out.trace['active_size']; print('active every 10:', s[::10].tolist())
print('wall_ms every 10:', np.round(out.trace['wall_ms'][::10], 3).tolist())
