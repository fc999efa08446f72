"""One c3 (SuKro switching) solve on the CUDA library, after the per-level L cache."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
inst = syn.sukro_instance(seed=3)
seq = syn.sukro_sequence(inst)
Ls = [F.lipschitz_bound(dd.op) for dd in seq.dicts]   # 4 utility launches
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6, gamma_threshold=0.5)
r = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(variant=F.VARIANT_MULTI_DICT, full_lipschitz=Ls))
print(f"c3 it={r.iterations} dev_ms={r.device_ms:.3f} converged={r.converged}")
