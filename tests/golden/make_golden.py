"""Generate tests/golden/solves.npz: end-to-end solve fixtures of the pinned oracle.

The reference cannot be built here (Eigen3 absent), so its engine
outputs cannot be recorded directly. The oracle (oracle/fl1_oracle.cpp) is pinned to
every known-answer vector of the reference's suites (tests/golden/reference_kats.json,
tests/test_kats_*.py, incl. the bit-exact first-gamma regression), and this script
freezes its outputs on small seeded instances covering the solver / rule / variant
space, so that

* the CPU suite checks the oracle still reproduces them bit for bit, and
* the GPU suite checks libfl1cuda.so against them without running the oracle.

Inputs are regenerated from seeds by paper_1812_06635_b200.synthetic (numpy PCG64);
an input checksum guards against generator drift. Run from the repo root:
    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from paper_1812_06635_b200 import _abi, fastl1 as F, synthetic as syn  # noqa: E402

TRACE_FIELDS = ("iter", "dict_index", "active_size", "x_nnz", "flops_cum", "gap", "gamma")


def oracle_backend():
    import conftest

    return F.Backend(_abi.Library(conftest._ensure_oracle(), "orc_", extra=_abi.ORACLE_ONLY))


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()[:16]


def cases():
    """name -> dict(kind, params). Every case is small enough for the oracle in < 1 s."""
    dense = dict(kind="dense", inst=dict(name="c2", seed=11, n=120, k=400, nnz=12))  # lambda = 0.2 lambda_max
    ragged = dict(kind="dense", inst=dict(name="c2", seed=12, n=97, k=333, nnz=9))
    c1_style = dict(kind="dense", inst=dict(name="c1", seed=13, n=150, k=600, nnz=15))  # sigma 0.01, 0.5 lambda_max
    base_cfg = dict(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    return {
        "fista_gap_screened": {**dense, "cfg": base_cfg, "opts": dict(variant=F.VARIANT_SCREENED)},
        "fista_gap_cached_l": {**dense, "cfg": base_cfg, "opts": dict(variant=F.VARIANT_SCREENED), "cached_l": True},
        "ista_gap_screened": {**dense, "cfg": base_cfg, "opts": dict(variant=F.VARIANT_SCREENED, solver=F.SOLVER_ISTA)},
        "fista_dynamic_aty": {**dense, "cfg": {**base_cfg, "precompute_aty": True},
                              "opts": dict(variant=F.VARIANT_SCREENED, rule=F.RULE_DYNAMIC)},
        "fista_plain": {**dense, "cfg": base_cfg, "opts": dict(variant=F.VARIANT_PLAIN)},
        "fista_ragged": {**ragged, "cfg": base_cfg, "opts": dict(variant=F.VARIANT_SCREENED)},
        "fista_c1_style": {**c1_style, "cfg": base_cfg, "opts": dict(variant=F.VARIANT_SCREENED)},
        "fista_cap": {**dense, "cfg": {**base_cfg, "max_iterations": 7}, "opts": dict(variant=F.VARIANT_SCREENED)},
        "fista_abs_tol": {**dense, "cfg": dict(screening_interval=5, max_iterations=5000, tolerance=1e-8),
                          "opts": dict(variant=F.VARIANT_SCREENED)},
        "fista_gram": {**dense, "cfg": base_cfg, "opts": dict(variant=F.VARIANT_SCREENED), "cached_l": True,
                       "gram": True},
        "sukro_multi_dict": dict(kind="sukro", inst=dict(seed=4, m=16, q=32, terms=4, levels=(1, 2), nnz=30),
                                 cfg={**base_cfg, "gamma_threshold": 0.5},
                                 opts=dict(variant=F.VARIANT_MULTI_DICT)),
    }


def build(case, backend):
    """(seq, y, lam, cfg, opts, a_dense) for a case on a backend."""
    if case["kind"] == "dense":
        inst = syn.dense_instance(**case["inst"])
        d = F.DenseDictionary(inst.a, backend=backend)
        seq = F.ApproxSequence([F.make_exact_approx(d)])
        a, y, lam = inst.a, inst.y, inst.lam
        opts = dict(case["opts"])
        if case.get("cached_l"):
            opts["full_lipschitz"] = [F.lipschitz_bound(d)]
        if case.get("gram"):
            opts["exact_gram"] = F.gram_matrix(d)
    else:
        si = syn.sukro_instance(**case["inst"])
        seq = syn.sukro_sequence(si, backend)
        a, y, lam = si.a, si.y, si.lam
        opts = dict(case["opts"])
    cfg = F.SwitchConfig(**case["cfg"])
    return seq, y, lam, cfg, F.RunOptions(collect_trace=True, **opts), a


def record(res) -> dict:
    out = {"x": res.x, "iterations": np.int64(res.iterations), "converged": np.int64(res.converged),
           "final_gap": np.float64(res.final_gap), "total_flops": np.uint64(res.total_flops),
           "final_active": np.asarray(res.final_active, dtype=np.int32),
           "switches": np.asarray([tuple(s)[:3] for s in res.switches], dtype=np.int64).reshape(-1, 3)}
    for f in TRACE_FIELDS:
        out["trace_" + f] = np.asarray(res.trace[f])
    return out


def batched_case(backend):
    """8 signals on one dictionary (BASELINE c5's shape of problem, reduced): the GPU runs
    them as one batched call (lockstep engine + cluster hand-off); each equals its own
    single solve. Returns (seq, Y (N x B), lambdas, cfg, opts, a)."""
    inst = syn.dense_instance("c2", seed=21, n=128, k=512, nnz=10)
    rng = np.random.default_rng(22)
    B = 8
    Y = np.empty((inst.a.shape[0], B), order="F")
    for b in range(B):
        Y[:, b] = syn.observe(rng, inst.a @ syn.sparse_signal(rng, inst.a.shape[1], 6 + b), None, 30.0)
    lams = 0.25 * np.max(np.abs(inst.a.T @ Y), axis=0)
    d = F.DenseDictionary(inst.a, backend=backend)
    seq = F.ApproxSequence([F.make_exact_approx(d)])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[F.lipschitz_bound(d)], collect_trace=True)
    return seq, Y, lams, cfg, opts, inst.a


def main():
    orc = oracle_backend()
    store, meta = {}, {}
    seq, Y, lams, cfg, opts, a = batched_case(orc)
    for b in range(Y.shape[1]):
        res = F.run_lasso(seq, Y[:, b], lams[b], cfg, opts)
        for key, v in record(res).items():
            store[f"batched{b}/{key}"] = v
    meta["_batched"] = {"input_digest": digest(a, Y), "signals": int(Y.shape[1])}
    for name, case in cases().items():
        seq, y, lam, cfg, opts, a = build(case, orc)
        res = F.run_lasso(seq, y, lam, cfg, opts)
        for key, v in record(res).items():
            store[f"{name}/{key}"] = v
        meta[name] = {"case": {k: v for k, v in case.items()}, "input_digest": digest(a, y), "lambda": lam}
        print(f"{name}: {res.iterations} iterations, converged {res.converged}, nnz {int(np.sum(res.x != 0))}")
    store["_meta"] = np.frombuffer(json.dumps(meta, default=list).encode(), dtype=np.uint8)
    np.savez_compressed(Path(__file__).with_name("solves.npz"), **store)


if __name__ == "__main__":
    main()
