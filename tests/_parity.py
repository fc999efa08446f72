"""Shared parity bar (BASELINE north_star) and the discrepancy recorder.

Every GPU-vs-oracle comparison goes through `assert_parity`, which asserts

* integer trajectory identical: iterations, preserved-set size and x support size at
  every iteration, dictionary index, ledger (`flops_cum`, `total_flops`), switch
  events, final preserved set and final support (fastl1.cpp:459-645, 611-623);
* final objective P(x) within OBJ_RTOL = 1e-9 relative (P recomputed here in fp64 from
  each x, fastl1.cpp:473);
* final duality gap within GAP_RTOL relative to the oracle's gap (fastl1.cpp:476-483);
* every logged gap and gamma within GAP_RTOL / GAMMA_RTOL relative;
* x within 1e-9 of max|x|;

and records the achieved discrepancies (max |dP|/P, |dgap|/gap, |dx|/|x|, trace gap and
gamma) so a GPU run can commit them (FL1_PARITY_OUT=path: JSON written at session end,
see conftest.py).

Why the gap bar has an ulp floor. The gap is P - D of two O(P) numbers computed from
the same iterate; at the stop it is ~1e-6 P. Each of P and D is a sum over N terms
whose rounding error depends on the summation order: ~sqrt(N) ulp(P) for a sequential
loop (the oracle, and Eigen's GEMV/dot in the reference), less for the GPU's shuffle
trees. So the gap is only determined to ~sqrt(N) * 1e-16 P / 1e-6 P ~ 1e-8 relative by
the reference's own fp64 arithmetic (N = 8192), and two correct implementations
summing in different orders differ by that much; 1e-9 relative is below the
reference's own precision there. The bar is therefore

    |gap_gpu - gap_oracle| <= max(1e-9 * gap, GAP_ULPS(N) * eps * P),
    GAP_ULPS(N) = max(64, 2 sqrt(N)),

where the second term binds whenever gap < ~1e-5 P. Measured on the B200 over the whole
GPU suite (profiles/r02_parity_metrics.json, 919 comparisons): at most 71 ulp(P) at
N = 8192 (c4, lambda_9 trace; bar 181), 26 at N = 1024 (c5; bar 64), 31 at N = 2500 (c2;
bar 100), 23 at N = 230 (bar 64); P itself agrees to <= 3.9e-16 relative and x to
<= 1.8e-14 of max|x|. The logged per-iteration gaps use the same bar with P_t <= P_final
+ gap_t as the ulp scale.
"""
from __future__ import annotations

import json
import os

import numpy as np

OBJ_RTOL = 1e-9
GAP_RTOL = 1e-9   # north_star: duality gap within 1e-9 relative ...
GAP_ULPS = 64.0   # ... or within max(GAP_ULPS, 2 sqrt(N)) ulp of P (summation-order rounding)
MEASURE_ONLY = os.environ.get("FL1_PARITY_MEASURE", "0") == "1"  # record, do not assert the gap bars

EPS = float(np.finfo(np.float64).eps)
RECORDS: list = []


def primal(a, y, lam, x) -> float:
    nz = np.flatnonzero(x)
    r = y - a[:, nz] @ x[nz] if nz.size else np.asarray(y, dtype=np.float64).copy()
    return 0.5 * float(r @ r) + lam * float(np.abs(x).sum())


def _rel(a, b):
    return abs(a - b) / abs(b) if b != 0 else abs(a - b)


def gap_bar(gap: float, p: float, ulps: float = GAP_ULPS) -> float:
    """Allowed |gap_gpu - gap_oracle|: 1e-9 relative, floored at `ulps` ulp of P."""
    return max(GAP_RTOL * abs(gap), ulps * EPS * abs(p))


def trace_rel(g, o, field: str, p: float | None = None, ulps: float = GAP_ULPS) -> float:
    """max over logged iterations of |g - o| / |o| (entries logged as -1 excluded); with p,
    of |g - o| / gap_bar(o, p) instead (<= 1 passes)."""
    gv, ov = np.asarray(g.trace[field], np.float64), np.asarray(o.trace[field], np.float64)
    m = (ov != -1.0) & np.isfinite(ov) & (ov != 0.0)
    if not np.any(m):
        return 0.0
    # P(x_t) = D_t + gap_t <= P* + gap_t <= P_final + gap_t bounds the ulp scale at iteration t
    den = (np.abs(ov[m]) if p is None
           else np.maximum(GAP_RTOL * np.abs(ov[m]), ulps * EPS * (abs(p) + np.abs(ov[m]))))
    return float(np.max(np.abs(gv[m] - ov[m]) / den))


def ulp_bar(n: int, floor: float = GAP_ULPS) -> float:
    return max(floor, 2.0 * float(np.sqrt(n)))


def record(case: str, g, o, a, y, lam, ulps: float = GAP_ULPS) -> dict:
    if case == "?" or case.startswith("+"):
        case = os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0] + (case[1:] if case != "?" else "")
    pg, po = primal(a, y, lam, g.x), primal(a, y, lam, o.x)
    xo = float(np.max(np.abs(o.x))) if o.x.size else 0.0
    rec = {"case": case, "n": int(a.shape[0]), "iterations": int(o.iterations), "converged": bool(o.converged),
           "P": po, "dP_rel": _rel(pg, po),
           "final_gap": float(o.final_gap) if o.converged else None,
           "gap_over_P": float(o.final_gap) / po if o.converged and po else None,
           "dgap_rel": _rel(float(g.final_gap), float(o.final_gap)) if o.converged else None,
           "dgap_ulpP": abs(float(g.final_gap) - float(o.final_gap)) / (EPS * abs(po)) if o.converged and po else None,
           "dx_rel": float(np.max(np.abs(g.x - o.x))) / max(xo, 1e-300) if o.x.size else 0.0,
           "trace_gap_rel_max": trace_rel(g, o, "gap") if len(o.trace) else None,
           "trace_gap_over_bar": trace_rel(g, o, "gap", po, ulps) if len(o.trace) else None,
           "trace_gamma_rel_max": trace_rel(g, o, "gamma") if len(o.trace) else None}
    RECORDS.append(rec)
    return rec


def assert_parity(g, o, a, y, lam, x_atol=1e-9, case: str = "?", gap_ulps: float = GAP_ULPS):
    """gap_ulps: the floor of the gap bar's ulp term (see the module docstring)."""
    ulps = ulp_bar(a.shape[0], gap_ulps)
    rec = record(case, g, o, a, y, lam, ulps)
    rec["gap_ulps_bar"] = ulps
    assert g.converged == o.converged
    assert g.iterations == o.iterations
    for f in ("dict_index", "active_size", "x_nnz", "flops_cum", "iter"):
        assert np.array_equal(g.trace[f], o.trace[f]), f
    assert np.array_equal(g.final_active, o.final_active)
    assert np.array_equal(g.x != 0, o.x != 0), "support differs"
    assert np.array_equal(g.switches, o.switches)
    assert g.total_flops == o.total_flops
    assert rec["dP_rel"] <= OBJ_RTOL, rec
    gm, om = g.trace["gamma"], o.trace["gamma"]
    assert np.array_equal(gm == -1.0, om == -1.0)
    assert np.max(np.abs(g.x - o.x)) <= x_atol * max(1.0, np.max(np.abs(o.x)))
    if MEASURE_ONLY:
        return rec
    if o.converged:
        assert abs(g.final_gap - o.final_gap) <= gap_bar(o.final_gap, rec["P"], ulps), rec
    if rec["trace_gap_over_bar"] is not None:
        assert rec["trace_gap_over_bar"] <= 1.0, rec
        # gamma = gap~ / gap' is a ratio of two such gaps (fastl1.cpp:26-30): 1e-6 relative, plus the
        # gaps' own bar relative to the logged gap where that is larger (a gap at the rounding
        # floor, e.g. lambda >= lambda_max, makes gamma a ratio of noise)
        og = np.asarray(o.trace["gap"], np.float64)
        lg = (om != -1.0) & np.isfinite(om)
        with np.errstate(divide="ignore", invalid="ignore"):
            noise = np.where(og > 0, 4.0 * ulps * EPS * (abs(rec["P"]) + np.abs(og)) / np.abs(og), np.inf)
        with np.errstate(invalid="ignore", over="ignore"):
            tol = np.where(np.isfinite(noise), np.abs(om) * (1e-6 + noise) + 1e-12, np.inf)
        assert np.all(np.abs(gm[lg] - om[lg]) <= tol[lg]), rec
    return rec


def write_records(path: str) -> None:
    if not RECORDS:
        return
    keys = ("dP_rel", "dgap_ulpP", "trace_gap_over_bar", "dx_rel", "trace_gap_rel_max", "trace_gamma_rel_max")
    summary = {k: max((r[k] for r in RECORDS if r.get(k) is not None), default=None) for k in keys}
    out = {"cases": len(RECORDS), "max": summary, "records": RECORDS}
    if os.path.exists(path):  # several pytest processes append to one file
        try:
            prev = json.loads(open(path).read())
            out["records"] = prev.get("records", []) + RECORDS
            out["cases"] = len(out["records"])
            out["max"] = {k: max((r[k] for r in out["records"] if r.get(k) is not None), default=None)
                          for k in keys}
        except Exception:
            pass
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
