"""GPU parity of the alternative code paths behind the run-time switches (DESIGN.md
§7b): every non-default setting must reproduce the oracle exactly as the default
does (identical trajectories, ledgers and supports; objective and gap within 1e-9).

The switches are read when a workspace is set up, so each setting runs in its own
process; the child solves through the C-ABI and returns the result fields as .npz.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1812_06635_b200 import fastl1 as F, synthetic as syn

from test_parity_gpu import assert_parity

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1812_06635_b200 import fastl1 as F, synthetic as syn
name, out = sys.argv[2], sys.argv[3]
if name == "sukro":
    inst = syn.sukro_instance(seed=int(sys.argv[4]), m=16, q=32, nnz=int(sys.argv[7]))
    seq = syn.sukro_sequence(inst)
    L = 0.0
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6, gamma_threshold=0.5)
    r = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(collect_trace=True))
else:
    inst = syn.dense_instance(name, seed=int(sys.argv[4]), n=int(sys.argv[5]), k=int(sys.argv[6]), nnz=int(sys.argv[7]))
    d = F.DenseDictionary(inst.a)
    L = F.lipschitz_bound(d)
    seq = F.ApproxSequence([F.make_exact_approx(d)])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    r = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L],
                                                              collect_trace=True))
np.savez(out, x=r.x, it=r.iterations, conv=r.converged, gap=r.final_gap, flops=r.total_flops,
         active=r.final_active, L=L, sw=r.switches, **{"t_" + k: r.trace[k] for k in r.trace.dtype.names})
"""

# (switch, value): each one selects a different code path than the default
SWITCHES = [
    ("FL1_EARLY_PROX", "0"),       # prox after the first barrier on every iteration
    ("FL1_LIST_APPLY", "0"),       # chunked apply partials instead of the phase-B lists
    ("FL1_LD_ALIGN", "4"),         # 32-byte instead of 128-byte leading dimension
    ("FL1_BULK_STAGES", "0"),      # register ring for the power-iteration adjoints
    ("FL1_SINGLE_CLUSTER", "0"),   # small dictionaries on the full grid
    ("FL1_POWER_ONCHIP", "0"),     # cluster-mode power iterations streamed, not resident
    ("FL1_SINGLE_CLUSTER_SIZE", "16"),  # the single-cluster route on 16 CTAs (default 12 up to 8 MiB)
    ("FL1_COMPACT", "1"),          # preserved columns physically compacted (ActiveOp::maybe_compact)
    ("FL1_COLSPLIT", "1"),         # phase-E apply by column split on every iteration
    ("FL1_FUSED_POWER_MB", "1"),   # single-read power steps from 1 MiB sets (default: beyond L2, 192 MiB)
]

CASES = {  # name, seed, n, k, nnz: c1 (single-cluster route) and a full-grid dense solve
    "small": ("c1", 1, 500, 2000, 50),
    "grid": ("c2", 2, 1500, 6000, 150),
    "sukro": ("sukro", 3, 256, 1024, 30),
    "long": ("c2", 4, 8192, 2000, 300),  # long columns: the phase-E column split applies (ld >= 8192)
    "tall": ("c2", 5, 5000, 1500, 120),  # 10 units per column, the last one partial (single-read power steps)
    "edge": ("c2", 6, 4097, 300, 20),    # 9 units, a 16-double tail unit; preserved sets below the CTA count
}


def child_solve(tmp_path, case, env_extra):
    name, seed, n, k, nnz = CASES[case]
    out = tmp_path / f"{case}_{'_'.join(f'{a}{b}' for a, b in env_extra.items()) or 'default'}.npz"
    env = dict(os.environ, **env_extra)
    subprocess.run([sys.executable, "-c", CHILD, str(ROOT), name, str(out), str(seed), str(n), str(k), str(nnz)],
                   check=True, env=env, timeout=600)
    return np.load(out)


class _Res:  # the fields assert_parity reads
    def __init__(self, z):
        self.x = z["x"]
        self.iterations = int(z["it"])
        self.converged = bool(z["conv"])
        self.final_gap = float(z["gap"])
        self.total_flops = int(z["flops"])
        self.final_active = z["active"]
        self.switches = z["sw"]
        names = [k[2:] for k in z.files if k.startswith("t_")]
        self.trace = {k: z["t_" + k] for k in names}


# the SuKro case covers the compaction's rebase path, the long case the column split
# (single-read power steps need 4096 < n <= 8192: the long, tall and edge cases)
PARAMS = [(c, sw, v) for c in sorted(CASES) for sw, v in SWITCHES
          if (c != "sukro" or sw == "FL1_COMPACT") and (c != "long" or sw in ("FL1_COLSPLIT", "FL1_FUSED_POWER_MB"))
          and (c not in ("tall", "edge") or sw == "FL1_FUSED_POWER_MB")
          and (sw != "FL1_FUSED_POWER_MB" or c in ("long", "tall", "edge"))]


@pytest.mark.parametrize("case,switch,value", PARAMS)
def test_switch_matches_oracle(tmp_path, oracle, case, switch, value):
    name, seed, n, k, nnz = CASES[case]
    if name == "sukro":  # multi-level: the switch to the exact level rebases (and compacts) the column view
        inst = syn.sukro_instance(seed=seed, m=16, q=32, nnz=nnz)
        g = _Res(child_solve(tmp_path, case, {switch: value}))
        cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6, gamma_threshold=0.5)
        o = F.run_lasso(syn.sukro_sequence(inst, oracle), inst.y, inst.lam, cfg, F.RunOptions(collect_trace=True))
        assert g.switches.size >= 1
        assert_parity(g, o, inst.a, inst.y, inst.lam)
        return
    inst = syn.dense_instance(name, seed=seed, n=n, k=k, nnz=nnz)
    z = child_solve(tmp_path, case, {switch: value})
    g = _Res(z)
    d = F.DenseDictionary(inst.a, backend=oracle)
    seq = F.ApproxSequence([F.make_exact_approx(d)])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    L = float(z["L"])  # the cached full Lipschitz constant the GPU solve used (as the harness passes it)
    o = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L],
                                                              collect_trace=True))
    assert_parity(g, o, inst.a, inst.y, inst.lam)
