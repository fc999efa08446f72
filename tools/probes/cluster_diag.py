"""Where does a cluster-mode solve first differ from the oracle / the grid-mode solve?"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', 'tests'))
import numpy as np
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn, _abi
from paper_1812_06635_b200.fastl1 import Backend, default_backend
from test_parity_gpu import _sukro_seq
from conftest import _ensure_oracle
cuda = default_backend()
orc = Backend(_abi.Library(_ensure_oracle(), "orc_", extra=_abi.ORACLE_ONLY))
inst = syn.sukro_instance(seed=3, m=16, q=32, nnz=30)
rng = np.random.default_rng(11)
B = 6
Y = np.empty((inst.a.shape[0], B), order="F"); lams = np.empty(B)
for b in range(B):
    Y[:, b] = syn.observe(rng, inst.a @ syn.sparse_signal(rng, inst.a.shape[1], 20 + 3 * b), None, 30.0)
    lams[b] = (0.2 + 0.05 * b) * np.max(np.abs(inst.a.T @ Y[:, b]))
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6, gamma_threshold=0.5)
opts = F.RunOptions(collect_trace=True)
sg = _sukro_seq(inst, cuda); so = _sukro_seq(inst, orc)
modes = {m: F.run_lasso_batched(sg, Y, lams, cfg, opts, concurrency=m) for m in (1, -1, -2, -8)}
for b in range(B):
    o = F.run_lasso(so, Y[:, b], lams[b], cfg, opts)
    for m, rs in modes.items():
        g = rs[b]
        ta, tb = g.trace, o.trace
        n = min(len(ta), len(tb))
        bad = [i for i in range(n) if any(ta[f][i] != tb[f][i] for f in ("dict_index", "active_size", "x_nnz", "flops_cum"))]
        print(f"b={b} mode={m:3d} its g={g.iterations} o={o.iterations} first_diff={bad[:1]} "
              f"sw_g={g.switches.tolist()} sw_o={o.switches.tolist()}")
        if bad:
            i = bad[0]
            for f in ta.dtype.names:
                print("   ", f, ta[f][max(0,i-1):i+2], tb[f][max(0,i-1):i+2])
