"""Golden vectors (tests/golden/): the reference's known-answer vectors
(reference_kats.json) and the frozen end-to-end solves of the pinned oracle
(solves.npz, made by tests/golden/make_golden.py). The CPU suite checks the
oracle reproduces them bit for bit; -m gpu checks libfl1cuda.so against them
(integer fields identical, floating point within the parity tolerances)."""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1812_06635_b200 import fastl1 as F

GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(GOLDEN))
import make_golden as MG  # noqa: E402
import _parity as P  # noqa: E402

KATS = json.loads((GOLDEN / "reference_kats.json").read_text())
SOLVES = np.load(GOLDEN / "solves.npz")
META = json.loads(bytes(SOLVES["_meta"]).decode())
OBJ_RTOL = 1e-9


@pytest.mark.parametrize("fn", ["soft_threshold", "gap_ratio", "switch_dictionary", "flops_plain", "flops_screened",
                                "flops_stable", "stable_gap_delta", "sphere_test"])
def test_reference_scalar_kats(backend, fn):
    s = F.scalars(backend)
    for args, want in KATS[fn]["cases"]:
        got = getattr(s, fn)(*args)
        assert got == pytest.approx(want, rel=1e-15, abs=0.0), (fn, args, got, want, KATS[fn]["cite"])


def test_reference_operator_kats(backend):
    for case, want in KATS["lambda_max"]["cases"]:
        d = F.DenseDictionary(np.asarray(case["a"]), backend=backend)
        assert F.lambda_max(d, case["y"]) == want
    for case, (lo, hi) in KATS["lipschitz_bound"]["cases"]:
        d = F.DenseDictionary(case["a_scale"] * np.eye(case["n"]), backend=backend)
        assert lo <= F.lipschitz_bound(d) <= hi
    dd = KATS["dense_diagonal"]
    d = F.DenseDictionary(np.asarray(dd["a"]), backend=backend)
    for x, want in dd["apply"]:
        assert np.array_equal(d.apply(x), want)
    for r, want in dd["apply_adjoint"]:
        assert np.array_equal(d.apply_adjoint(r), want)


def _primal(a, y, lam, x):
    r = y - a @ x
    return 0.5 * float(r @ r) + lam * float(np.sum(np.abs(x)))


@pytest.mark.parametrize("name", sorted(n for n in META if not n.startswith("_")))
def test_golden_solve(backend, name):
    case = MG.cases()[name]
    seq, y, lam, cfg, opts, a = MG.build(case, backend)
    assert MG.digest(a, y) == META[name]["input_digest"], "instance generator drifted"
    g = {k.split("/", 1)[1]: SOLVES[k] for k in SOLVES.files if k.startswith(name + "/")}
    check(MG.record(F.run_lasso(seq, y, lam, cfg, opts)), g, a, y, lam, exact=backend.lib.prefix == "orc_")


def test_golden_batched(backend):
    """The oracle solves each signal alone; the GPU takes all of them in one batched call."""
    seq, Y, lams, cfg, opts, a = MG.batched_case(backend)
    assert MG.digest(a, Y) == META["_batched"]["input_digest"], "instance generator drifted"
    exact = backend.lib.prefix == "orc_"
    if exact:
        results = [F.run_lasso(seq, Y[:, b], lams[b], cfg, opts) for b in range(Y.shape[1])]
    else:
        results = F.run_lasso_batched(seq, Y, lams, cfg, opts)
    for b, r in enumerate(results):
        g = {k.split("/", 1)[1]: SOLVES[k] for k in SOLVES.files if k.startswith(f"batched{b}/")}
        check(MG.record(r), g, a, Y[:, b], lams[b], exact)


def check(res, g, a, y, lam, exact):
    for key in ("iterations", "converged", "total_flops", "final_active", "switches", "trace_iter",
                "trace_dict_index", "trace_active_size", "trace_x_nnz", "trace_flops_cum"):
        assert np.array_equal(res[key], g[key]), key
    if exact:  # the oracle itself: frozen bit for bit
        for key in ("x", "final_gap", "trace_gap", "trace_gamma"):
            assert np.array_equal(res[key], g[key], equal_nan=True), key
        return
    p_ref = _primal(a, y, lam, g["x"])
    assert abs(_primal(a, y, lam, res["x"]) - p_ref) <= OBJ_RTOL * abs(p_ref)
    assert np.max(np.abs(res["x"] - g["x"])) <= 1e-9 * max(1.0, np.max(np.abs(g["x"])))
    assert np.array_equal(res["trace_gamma"] == -1.0, g["trace_gamma"] == -1.0)
    assert np.array_equal(res["trace_gap"] == -1.0, g["trace_gap"] == -1.0)
    m = (g["trace_gap"] != -1.0) & (g["trace_gap"] != 0.0)
    tg = float(np.max(np.abs(res["trace_gap"][m] - g["trace_gap"][m]) / np.abs(g["trace_gap"][m]))) if m.any() else 0.0
    dgap = (abs(float(res["final_gap"]) - float(g["final_gap"])) / abs(float(g["final_gap"]))
            if g["converged"] and float(g["final_gap"]) != 0 else None)
    P.RECORDS.append({"case": P.os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], "P": p_ref,
                      "dP_rel": abs(_primal(a, y, lam, res["x"]) - p_ref) / abs(p_ref), "dgap_rel": dgap,
                      "dx_rel": float(np.max(np.abs(res["x"] - g["x"]))) / max(float(np.max(np.abs(g["x"]))), 1e-300),
                      "trace_gap_rel_max": tg, "iterations": int(g["iterations"])})
    if P.MEASURE_ONLY:
        return
    if dgap is not None:
        assert abs(float(res["final_gap"]) - float(g["final_gap"])) <= P.gap_bar(float(g["final_gap"]), p_ref,
                                                                                 P.ulp_bar(a.shape[0]))
    bar = np.maximum(P.GAP_RTOL * np.abs(g["trace_gap"][m]), P.ulp_bar(a.shape[0]) * P.EPS * (abs(p_ref) + np.abs(g["trace_gap"][m])))
    assert np.all(np.abs(res["trace_gap"][m] - g["trace_gap"][m]) <= bar)
    assert np.allclose(res["trace_gamma"], g["trace_gamma"], rtol=1e-6, atol=1e-12)
