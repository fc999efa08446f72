"""c4 (8192 x 65536, 10-lambda warm-started path) under ncu: the engine launches of the
lambdas selected by --lams (default: all) run between cudaProfilerStart / Stop, so
`ncu --profile-from-start off` captures exactly those solve launches (one launch per lambda).
Also prints each solve's algorithmic bytes for the traffic comparison."""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lams", default="0,1,2,3,4,5,6,7,8,9")
args = ap.parse_args()
sel = {int(v) for v in args.lams.split(",")}
At, y = bench.make_c4_device(4, "cuda")
k, n = At.shape
d = F.DenseDictionaryDevice(At.data_ptr(), n, k)
del At
torch.cuda.empty_cache()
lmax = F.lambda_max(d, y)
L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
y_dev = torch.from_numpy(y).cuda()
x = None
out = []
for i, r in enumerate(syn.CONFIGS["c4"]["lam_ratios"]):
    opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], x_init=x)
    if i in sel:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
    res = F.run_lasso_device(seq, y_dev.data_ptr(), r * lmax, cfg, opts)
    if i in sel:
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    out.append({"lambda": i, "iterations": res.iterations, "device_ms": res.device_ms,
                "launches": res.kernel_launches, "alg_bytes": bench.algorithmic_bytes(res, n)})
    x = res.x
print(json.dumps(out))
