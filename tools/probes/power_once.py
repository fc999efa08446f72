"""One cold lipschitz_bound (200-step power iteration) on an n x k Gaussian dictionary."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import torch
from paper_1812_06635_b200 import fastl1 as F
n, k = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator(device='cuda').manual_seed(0)
A = torch.randn(k, n, device='cuda', dtype=torch.float64, generator=g)
A /= A.norm(dim=1, keepdim=True)
d = F.DenseDictionaryDevice(A.data_ptr(), n, k)
print(F.lipschitz_bound(d))
