"""Streaming-pass bandwidth probe: a few unscreened iterations at a given shape,
read back the device phase profile (A^T r bytes / phase-A time)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np
import torch
from paper_1812_06635_b200 import fastl1 as F

n, k, its = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 65536, 6)))
g = torch.Generator(device='cuda').manual_seed(0)
A = torch.randn(k, n, device='cuda', dtype=torch.float64, generator=g)
A /= A.norm(dim=1, keepdim=True)
d = F.DenseDictionaryDevice(A.data_ptr(), n, k)  # A row j = column j (column-major N x K)
y = torch.randn(n, dtype=torch.float64, generator=torch.Generator().manual_seed(1)).numpy()
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(max_iterations=its, tolerance=1e-30)
opts = F.RunOptions(variant=F.VARIANT_PLAIN, full_lipschitz=[float(k) / n * 4.0])
F.run_lasso(seq, y, 0.1, cfg, opts)  # warm
out = F.run_lasso(seq, y, 0.1, cfg, opts)
pr = out.profile
print(f"lib={os.environ.get('FL1_LIB','default')} n={n} k={k} its={out.iterations} phaseA_ms={pr[0]/1e6:.3f} "
      f"bytes={pr[5]:.3e} GB/s={pr[5]/pr[0]:.1f} per_iter_ms={pr[0]/1e6/its:.4f} B_ms={pr[1]/1e6:.3f} D_ms={pr[2]/1e6:.3f} dev_ms={out.device_ms:.3f}")
