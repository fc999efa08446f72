"""Engine-level tests ported from test_fastl1.cpp and acceptance.cpp (paths
relative to /root/reference/proj/tests), run on the oracle (CPU suite) and on
libfl1cuda.so (-m gpu) through the same Python API.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_1812_06635_b200 import fastl1 as F

from _refgen import make_sequence, perturbed_approx, solve_oracle

P = lambda a: np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731


def degenerate(backend, a):
    return F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=backend))])


def test_plain_engine_reproduces_stepper(backend, oracle, refgen):  # test_fastl1.cpp:72-104
    a, y, lmax = refgen.square_instance(36, 64, 5)
    seq = degenerate(backend, a)
    lam = 0.3 * lmax
    L = F.lipschitz_bound(F.DenseDictionary(a, backend=oracle))
    od = F.DenseDictionary(a, backend=oracle)
    for solver in (F.SOLVER_ISTA, F.SOLVER_FISTA):
        cfg = F.SwitchConfig(tolerance=1e-9, max_iterations=60)
        res = F.run_lasso(seq, y, lam, cfg, F.RunOptions(solver=solver, variant=F.VARIANT_PLAIN, full_lipschitz=[L]))
        steps = res.iterations - 1 if res.converged else res.iterations
        x = np.zeros(64)
        x_prev = np.zeros(64)
        t_k, ready = C.c_double(1.0), C.c_int32(0)
        for _ in range(steps):
            xn = np.empty(64)
            if solver == F.SOLVER_ISTA:
                oracle.lib.check(oracle.lib.ista_step(od._h, P(y), lam, 1.0 / L, P(x), P(xn), None, None))
            else:
                oracle.lib.check(oracle.lib.fista_step(od._h, P(y), lam, 1.0 / L, P(x),
                                                       x_prev.ctypes.data_as(C.POINTER(C.c_double)), C.byref(t_k),
                                                       C.byref(ready), P(xn), None, None))
            x = xn
        assert np.max(np.abs(res.x - x)) <= 1e-9


@pytest.mark.parametrize("rule", [F.RULE_GAP, F.RULE_DYNAMIC])
def test_degenerate_sequence_equals_screened(backend, refgen, rule):  # test_fastl1.cpp:106-137
    a, y, lmax = refgen.square_instance(36, 100, 7)
    seq = degenerate(backend, a)
    cfg = F.SwitchConfig(tolerance=1e-8, max_iterations=5000)
    ra = F.run_lasso(seq, y, 0.25 * lmax, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, rule=rule))
    rb = F.run_lasso(seq, y, 0.25 * lmax, cfg, F.RunOptions(variant=F.VARIANT_MULTI_DICT, rule=rule))
    assert ra.converged and rb.converged
    assert ra.trace.size == rb.trace.size
    assert np.max(np.abs(ra.x - rb.x)) == 0.0
    for f in ("dict_index", "active_size", "gap", "gamma", "flops_cum", "x_nnz"):
        assert np.array_equal(ra.trace[f], rb.trace[f]), f


@pytest.mark.parametrize("trial", range(5))
def test_multi_dict_matches_oracle_solution(backend, oracle, refgen, trial):  # test_fastl1.cpp:139-165
    a, y, lmax = refgen.square_instance(36, 100, 40 + trial, support=2)
    levels = refgen.build_sukro_sequence(a, [1, 3])
    seq = make_sequence(F, backend, a, levels)
    lam = (0.25 + 0.05 * trial) * lmax
    cfg = F.SwitchConfig(tolerance=1e-8, gamma_threshold=0.5, max_iterations=200000)
    res = F.fastl1_solve(seq, y, lam, cfg, F.SOLVER_FISTA, F.RULE_GAP)
    assert res.converged and res.final_gap <= cfg.tolerance
    sol = solve_oracle(a, y, lam, 1e-12)
    assert np.max(np.abs(res.x - sol.x)) <= 2.0 * np.sqrt(2.0 * cfg.tolerance)
    od = F.DenseDictionary(a, backend=oracle)
    theta = np.empty(36)
    oracle.lib.check(oracle.lib.dual_scale(od._h, P(sol.theta), theta.ctypes.data_as(C.POINTER(C.c_double))))
    gap = oracle.lib.duality_gap(od._h, P(y), lam, P(res.x), P(theta), None)
    assert gap <= cfg.tolerance * (1 + 1e-9)


@pytest.mark.parametrize("solver", [F.SOLVER_ISTA, F.SOLVER_FISTA])
@pytest.mark.parametrize("rule", [F.RULE_GAP, F.RULE_DYNAMIC])
def test_trace_invariants(backend, refgen, solver, rule):  # test_fastl1.cpp:167-201
    a, y, lmax = refgen.square_instance(64, 144, 77)
    seq = make_sequence(F, backend, a, refgen.build_sukro_sequence(a, [1, 2, 4]))
    cfg = F.SwitchConfig(tolerance=1e-7, gamma_threshold=0.4, max_iterations=100000)
    res = F.run_lasso(seq, y, 0.2 * lmax, cfg, F.RunOptions(solver=solver, rule=rule))
    assert res.converged
    tr = res.trace
    assert np.all(np.diff(tr["active_size"]) <= 0) and tr["active_size"][0] <= 144
    assert np.all(np.diff(tr["dict_index"]) >= 0)
    g = tr["gamma"][tr["gamma"] != -1.0]
    assert np.all((g >= 0.0) & (g <= 1.0))
    last = seq.levels() - 1
    first_exact = np.argmax(tr["dict_index"] == last)
    assert np.all(tr["dict_index"][first_exact:] == last)


@pytest.mark.parametrize("variant", [F.VARIANT_PLAIN, F.VARIANT_SCREENED, F.VARIANT_MULTI_DICT])
def test_ledger_audit(backend, refgen, variant):  # test_fastl1.cpp:203-217
    a, y, lmax = refgen.square_instance(49, 121, 91)
    seq = make_sequence(F, backend, a, refgen.build_sukro_sequence(a, [1, 3]))
    cfg = F.SwitchConfig(tolerance=1e-7, max_iterations=100000)
    res = F.run_lasso(seq, y, 0.3 * lmax, cfg, F.RunOptions(variant=variant))
    assert res.converged
    total, rows_match = F.recompute_flops(res.trace, seq, variant, 49, 121)
    assert total == res.total_flops and rows_match
    assert int(res.trace["flops_cum"][-1]) == res.total_flops


def test_gamma_regression_kat(backend, refgen):  # test_fastl1.cpp:243-268
    a, y, lmax = refgen.square_instance(36, 100, 113, 4, "easy")
    seq = make_sequence(F, backend, a, refgen.build_sukro_sequence(a, [2]))
    cfg = F.SwitchConfig(gamma_threshold=0.5, tolerance=1e-10, max_iterations=100000)
    res = F.run_lasso(seq, y, 0.2 * lmax, cfg, F.RunOptions(rule=F.RULE_GAP))
    g = res.trace["gamma"][res.trace["gamma"] != -1.0]
    assert g.size > 0
    assert g[0] >= 0.9
    assert g[0] == pytest.approx(0.95470658293002786, rel=1e-9)  # the reference's regression value
    assert g[-1] <= g[0]


def test_iteration_cap(backend, refgen):  # test_fastl1.cpp:270-283
    a, y, lmax = refgen.square_instance(36, 64, 131)
    res = F.run_lasso(degenerate(backend, a), y, 0.3 * lmax, F.SwitchConfig(tolerance=1e-14, max_iterations=5),
                      F.RunOptions(variant=F.VARIANT_SCREENED))
    assert not res.converged and res.iterations == 5 and res.trace.size == 5 and res.x.size == 64
    assert np.isnan(res.final_gap)


def test_immediate_convergence_at_lambda_max(backend, refgen):  # test_fastl1.cpp:306-320
    a, y, lmax = refgen.square_instance(36, 64, 171)
    res = F.run_lasso(degenerate(backend, a), y, lmax, F.SwitchConfig(tolerance=1e-10),
                      F.RunOptions(variant=F.VARIANT_SCREENED))
    assert res.converged and res.iterations == 1 and res.trace.size == 1
    assert np.max(np.abs(res.x)) == 0.0 and res.final_gap <= 1e-10 and res.total_flops > 0


@pytest.mark.parametrize("trial", range(3))
def test_precompute_aty_dynamic_rule_safe(backend, refgen, trial):  # test_fastl1.cpp:322-350
    a, y, lmax = refgen.square_instance(36, 100, 181 + trial)
    seq = make_sequence(F, backend, a, refgen.build_sukro_sequence(a, [1, 3]))
    lam = 0.3 * lmax
    sol = solve_oracle(a, y, lam, 1e-12)
    supp = set(np.nonzero(sol.x)[0])
    violations = []

    def obs(ev):
        if not supp <= set(ev.kept.tolist()):
            violations.append(ev.iter)

    cfg = F.SwitchConfig(tolerance=1e-8, max_iterations=300000, precompute_aty=True)
    res = F.run_lasso(seq, y, lam, cfg, F.RunOptions(rule=F.RULE_DYNAMIC, variant=F.VARIANT_MULTI_DICT, observer=obs))
    assert res.converged and not violations
    assert np.max(np.abs(res.x - sol.x)) <= 2.0 * np.sqrt(2.0 * cfg.tolerance)


def test_screening_interval_nesting(backend, refgen):  # test_fastl1.cpp:352-371
    a, y, lmax = refgen.square_instance(36, 100, 191)
    seq = make_sequence(F, backend, a, refgen.build_sukro_sequence(a, [1, 3]))
    cfg = F.SwitchConfig(tolerance=1e-8, screening_interval=5, max_iterations=300000)
    res = F.run_lasso(seq, y, 0.3 * lmax, cfg, F.RunOptions(variant=F.VARIANT_MULTI_DICT))
    assert res.converged
    prev = 100
    for row in res.trace:
        if row["iter"] % 5 != 1:
            assert row["active_size"] == prev
        assert row["active_size"] <= prev
        prev = row["active_size"]


@pytest.mark.parametrize("rule", [F.RULE_GAP, F.RULE_DYNAMIC])
def test_safety_against_oracle_support(backend, refgen, rule):  # acceptance.cpp:149-262 (criteria 1-2), reduced
    """Stable screening with perturbed-dense approximations never drops the support,
    and the certified sphere always contains the dual optimum."""
    for trial, ratio in enumerate((0.1, 0.3, 0.7, 0.95)):
        a, y, lam, _ = refgen.random_instance(50, 120, ratio, 900 + trial)
        sol = solve_oracle(a, y, lam, 1e-12)
        supp = set(np.nonzero(sol.x)[0])
        coarse, _ = perturbed_approx(F, backend, refgen, a, 0.05, 950 + trial, rc=0.3)
        fine, _ = perturbed_approx(F, backend, refgen, a, 0.01, 970 + trial, rc=0.6)
        fine.atom_error_bounds = np.minimum(fine.atom_error_bounds, coarse.atom_error_bounds)
        exact = F.make_exact_approx(F.DenseDictionary(a, backend=backend))
        seq = F.ApproxSequence([coarse, fine, exact])
        bad = []

        def obs(ev):
            if not supp <= set(ev.kept.tolist()):
                bad.append(("support", ev.iter))
            if rule == F.RULE_GAP and np.linalg.norm(sol.theta - ev.center) > ev.radius + 1e-9:
                bad.append(("sphere", ev.iter))

        cfg = F.SwitchConfig(tolerance=1e-9, screening_interval=1, max_iterations=200000)
        res = F.run_lasso(seq, y, lam, cfg, F.RunOptions(rule=rule, observer=obs))
        assert res.converged
        assert not bad, bad[:5]


def test_invalid_arguments(backend, refgen):  # fastl1.cpp:268-273, dictionary.cpp:227-251
    a, y, lmax = refgen.square_instance(36, 64, 5)
    seq = degenerate(backend, a)
    with pytest.raises(F.InvalidArgument):
        F.run_lasso(seq, y, 0.0, F.SwitchConfig(), F.RunOptions())
    with pytest.raises(F.InvalidArgument):
        F.run_lasso(seq, y, 0.1, F.SwitchConfig(gamma_threshold=1.0), F.RunOptions())
    with pytest.raises(F.InvalidArgument):
        F.run_lasso(seq, y, 0.1, F.SwitchConfig(screening_interval=0), F.RunOptions())
    with pytest.raises(F.InvalidArgument):
        F.run_lasso(seq, y[:-1], 0.1, F.SwitchConfig(), F.RunOptions())
    d = F.DenseDictionary(a, backend=backend)
    ex = F.make_exact_approx(d)
    bad_rc = F.ApproxDictionary(d, np.zeros(64), 0.0, 0.5, np.ones(64), np.ones(64))
    with pytest.raises(F.InvalidArgument):  # last level must be exact with RC 1
        F.ApproxSequence([bad_rc])
    with pytest.raises(F.InvalidArgument):  # RC must strictly increase
        F.ApproxSequence([F.ApproxDictionary(d, np.full(64, 0.1), 0.1, 1.0, np.ones(64), np.ones(64)), ex])
    with pytest.raises(F.InvalidArgument):  # eps must be non-increasing
        F.ApproxSequence([F.ApproxDictionary(d, np.full(64, 0.1), 0.1, 0.3, np.ones(64), np.ones(64)),
                          F.ApproxDictionary(d, np.full(64, 0.2), 0.2, 0.6, np.ones(64), np.ones(64)), ex])
    with pytest.raises(F.InvalidArgument):
        F.ApproxSequence([F.ApproxDictionary(d, np.full(64, -0.1), 0.1, 0.3, np.ones(64), np.ones(64)), ex])
    with pytest.raises(F.InvalidArgument):
        F.ApproxSequence([])


def test_exact_fit_zero_signal(backend, refgen):  # fastl1.cpp:428-449 (ray = y fallback)
    a, _, _ = refgen.square_instance(36, 64, 5)
    res = F.run_lasso(degenerate(backend, a), np.zeros(36), 0.1, F.SwitchConfig(screening_interval=10),
                      F.RunOptions(variant=F.VARIANT_SCREENED))
    assert res.converged and res.iterations == 1 and np.all(res.x == 0.0)


def test_warm_start_and_relative_tolerance_extensions(backend, refgen):
    """x_init / rel_tolerance extensions (BASELINE configs 1-4); defaults are the reference."""
    a, y, lmax = refgen.square_instance(36, 100, 7)
    seq = degenerate(backend, a)
    cfg = F.SwitchConfig(tolerance=1e-12, rel_tolerance=1e-6, screening_interval=10, max_iterations=20000)
    r1 = F.run_lasso(seq, y, 0.4 * lmax, cfg, F.RunOptions(variant=F.VARIANT_SCREENED))
    assert r1.converged
    primal_gap_ok = r1.final_gap <= 1e-6 * (0.5 * np.sum((y - a @ r1.x) ** 2) + 0.4 * lmax * np.abs(r1.x).sum()) * (1 + 1e-9)
    assert primal_gap_ok
    # warm start from the converged point of the same lambda: certified within a few iterations
    # (r1.x passed the test with the dual ray at the extrapolated point, so the restart re-certifies)
    r2 = F.run_lasso(seq, y, 0.4 * lmax, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, x_init=r1.x))
    assert r2.converged and r2.iterations <= max(5, r1.iterations // 4)
    # warm start along a lambda path reaches the same solution as a cold start
    r3 = F.run_lasso(seq, y, 0.3 * lmax, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, x_init=r1.x))
    r4 = F.run_lasso(seq, y, 0.3 * lmax, cfg, F.RunOptions(variant=F.VARIANT_SCREENED))
    assert r3.converged and r4.converged
    assert np.max(np.abs(r3.x - r4.x)) <= 2.0 * np.sqrt(2.0 * 1e-6 * 0.5 * (y @ y))


@pytest.mark.gpu
def test_gamma_regression_kat_device_sequence(cuda, refgen):  # test_fastl1.cpp:243-268
    """The reference's first-gamma regression on a SuKro sequence built by the device
    construction (fl1_build_sukro_sequence) instead of the LAPACK restatement."""
    from paper_1812_06635_b200 import harness as H

    a, y, lmax = refgen.square_instance(36, 100, 113, 4, "easy")
    seq = H.sukro_sequence(a, [2], backend=cuda)
    cfg = F.SwitchConfig(gamma_threshold=0.5, tolerance=1e-10, max_iterations=100000)
    res = F.run_lasso(seq, y, 0.2 * lmax, cfg, F.RunOptions(rule=F.RULE_GAP))
    g = res.trace["gamma"][res.trace["gamma"] != -1.0]
    assert g.size > 0 and g[0] >= 0.9 and g[-1] <= g[0]
    assert g[0] == pytest.approx(0.95470658293002786, rel=1e-9)


@pytest.mark.gpu
def test_build_sukro_sequence_abi_errors(cuda):
    """fl1_build_sukro_sequence's own argument checks return FL1_EINVAL with the
    reference's messages (dictionary.cpp:19-33, 284-296)."""
    import ctypes as C

    lib = cuda.lib
    P = C.POINTER(C.c_double)
    out = [np.zeros(4096) for _ in range(6)]

    def call(a, ranks):
        d = F.DenseDictionary(a, backend=cuda)
        rk = np.asarray(ranks, dtype=np.int32)
        lib.check(lib.build_sukro_sequence(d._h, rk.ctypes.data_as(C.POINTER(C.c_int32)), len(ranks),
                                           *[o.ctypes.data_as(P) for o in out]))

    rng = np.random.default_rng(1)
    with pytest.raises(F.InvalidArgument, match="N must be a perfect square, got 35"):
        call(rng.standard_normal((35, 64)), [1])
    with pytest.raises(F.InvalidArgument, match="ranks must be positive and strictly increasing"):
        call(rng.standard_normal((36, 64)), [2, 2])
    with pytest.raises(F.InvalidArgument, match="rank exceeds rearranged dimension"):
        call(rng.standard_normal((36, 64)), [49])
    with pytest.raises(F.InvalidArgument, match="relative complexity >= 1"):
        call(rng.standard_normal((36, 64)), [4])
