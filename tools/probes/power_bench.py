"""Per-step cost of the cold restricted power iteration vs working-set size."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np
import torch
from paper_1812_06635_b200 import fastl1 as F

for n, k in [(500, 96), (500, 2000), (2500, 1000), (2500, 2876), (2500, 6000), (2500, 10000), (8192, 4000), (8192, 16000)]:
    g = torch.Generator(device='cuda').manual_seed(0)
    A = torch.randn(k, n, device='cuda', dtype=torch.float64, generator=g)
    A /= A.norm(dim=1, keepdim=True)
    d = F.DenseDictionaryDevice(A.data_ptr(), n, k)
    seq = F.ApproxSequence([F.make_exact_approx(d)])
    y = np.random.default_rng(1).standard_normal(n)
    cfg = F.SwitchConfig(max_iterations=1, tolerance=1e-30)
    F.run_lasso(seq, y, 1e-3, cfg, F.RunOptions(variant=F.VARIANT_PLAIN))
    out = F.run_lasso(seq, y, 1e-3, cfg, F.RunOptions(variant=F.VARIANT_PLAIN))
    pr = out.profile
    st = out.power_iterations
    mb = 8 * n * k / 1e6
    print(f"n={n} k={k} MB={mb:.1f} steps={st} setup_ms={out.setup_ms:.3f} us/step={1e3*out.setup_ms/st:.1f} "
          f"apply={pr[8]/st/1e3:.1f} comb={pr[9]/st/1e3:.1f} adj={pr[10]/st/1e3:.1f} red={pr[11]/st/1e3:.1f} us "
          f"eff_GBps={2*mb*1e6/(out.setup_ms*1e-3/st)/1e9:.0f}")
    del d, seq, A
