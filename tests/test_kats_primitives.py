"""Known-answer tests of the path's primitives, ported from the reference's own
suites (paths relative to /root/reference/proj/tests). Oracle-only primitives
(steppers, dual points, vector-form screening) pin the oracle; scalar formulas
and operators also run on libfl1cuda.so (-m gpu, or host-side where no device
is needed).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_1812_06635_b200 import fastl1 as F

from _refgen import perturbed_approx, solve_oracle

P = lambda a: np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731


def _dense(b, a):
    return F.DenseDictionary(np.asarray(a, dtype=np.float64), backend=b)


# ----------------------------------------------------------------- test_solver.cpp
def test_soft_threshold(oracle):  # test_solver.cpp:11-16
    s = F.scalars(oracle)
    assert s.soft_threshold(0.5, 1.0) == 0.0
    assert s.soft_threshold(2.0, 1.0) == 1.0
    assert s.soft_threshold(-2.0, 0.5) == -1.5
    assert s.soft_threshold(0.0, 0.0) == 0.0


def _ista(oracle, d, y, lam, step, x):
    n, k = d.shape
    xn, res, corr = np.empty(k), np.empty(n), np.empty(k)
    oracle.lib.check(oracle.lib.ista_step(d._h, P(y), lam, step, P(x), P(xn), P(res), P(corr)))
    return xn, res, corr


class Fista:
    def __init__(self, oracle, d, y, lam, step):
        self.o, self.d, self.y, self.lam, self.step = oracle, d, np.asarray(y, float), lam, step
        self.x_prev = np.zeros(d.cols())
        self.t_k = C.c_double(1.0)
        self.ready = C.c_int32(0)

    def __call__(self, x):
        k = self.d.cols()
        xn, res, corr = np.empty(k), np.empty(self.d.rows()), np.empty(k)
        x = np.ascontiguousarray(x, dtype=np.float64)
        self.o.lib.check(self.o.lib.fista_step(self.d._h, P(self.y), self.lam, self.step, P(x),
                                               self.x_prev.ctypes.data_as(C.POINTER(C.c_double)), C.byref(self.t_k),
                                               C.byref(self.ready), P(xn), P(res), P(corr)))
        return xn


def test_ista_identity_one_step(oracle):  # test_solver.cpp:29-38
    d = _dense(oracle, np.eye(2))
    xn, res, corr = _ista(oracle, d, np.array([1.0, 0.0]), 0.5, 1.0, np.zeros(2))
    assert xn[0] == pytest.approx(0.5) and xn[1] == 0.0
    assert res[0] == 1.0 and corr[0] == 1.0


def test_ista_zero_fixed_point_above_lambda_max(oracle, refgen):  # test_solver.cpp:40-48
    a, y, _, lmax = refgen.random_instance(8, 16, 1.0, 3)
    d = _dense(oracle, a)
    xn, _, _ = _ista(oracle, d, y, 1.1 * lmax, 0.25, np.zeros(16))
    assert np.max(np.abs(xn)) == 0.0


def test_ista_fixed_point_kkt(oracle, refgen):  # test_solver.cpp:50-67
    a, y, lam, _ = refgen.random_instance(8, 16, 0.3, 11)
    d = _dense(oracle, a)
    step = 1.0 / F.lipschitz_bound(d)
    x = np.zeros(16)
    for _ in range(100000):
        x, _, _ = _ista(oracle, d, y, lam, step, x)
    corr = a.T @ ((y - a @ x) / lam)
    assert np.all(np.abs(corr) <= 1.0 + 1e-8)
    nz = x != 0
    assert np.allclose(corr[nz], np.sign(x[nz]), rtol=1e-8, atol=1e-8)


def test_fista_first_step_equals_ista(oracle, refgen):  # test_solver.cpp:69-76
    a, y, lam, _ = refgen.random_instance(8, 16, 0.4, 17)
    d = _dense(oracle, a)
    x0 = refgen.random_vector(16, 2)
    xi, _, _ = _ista(oracle, d, y, lam, 0.2, x0)
    xf = Fista(oracle, d, y, lam, 0.2)(x0)
    assert np.max(np.abs(xi - xf)) == 0.0


def test_fista_stays_at_zero_above_lambda_max(oracle, refgen):  # test_solver.cpp:78-87
    a, y, _, lmax = refgen.random_instance(8, 16, 1.0, 19)
    d = _dense(oracle, a)
    f = Fista(oracle, d, y, 1.5 * lmax, 0.3)
    x = np.zeros(16)
    for _ in range(5):
        x = f(x)
    assert np.max(np.abs(x)) == 0.0


def test_fista_beats_ista(oracle, refgen):  # test_solver.cpp:89-101
    a, y, lam, _ = refgen.random_instance(8, 16, 0.1, 23)
    d = _dense(oracle, a)
    inv_l = 1.0 / F.lipschitz_bound(d)
    f = Fista(oracle, d, y, lam, inv_l)
    xi = np.zeros(16)
    xf = np.zeros(16)
    for _ in range(200):
        xi, _, _ = _ista(oracle, d, y, lam, inv_l, xi)
        xf = f(xf)
    pv = lambda x: oracle.lib.primal_value(d._h, P(y), lam, P(x))  # noqa: E731
    assert pv(xf) <= pv(xi) + 1e-12


def test_ista_monotone(oracle, refgen):  # test_solver.cpp:103-117
    a, y, lam, _ = refgen.random_instance(10, 24, 0.2, 29)
    d = _dense(oracle, a)
    step = 1.0 / F.lipschitz_bound(d)
    x = np.zeros(24)
    prev = oracle.lib.primal_value(d._h, P(y), lam, P(x))
    for _ in range(200):
        x, _, _ = _ista(oracle, d, y, lam, step, x)
        cur = oracle.lib.primal_value(d._h, P(y), lam, P(x))
        assert cur <= prev + 1e-12
        prev = cur


def test_objective_values(oracle, refgen):  # test_solver.cpp:119-144
    d = _dense(oracle, np.eye(2))
    y = np.array([1.0, 0.0])
    L = oracle.lib
    assert L.primal_value(d._h, P(y), 1.0, P(np.zeros(2))) == pytest.approx(0.5)
    assert L.primal_value(d._h, P(y), 1.0, P(np.array([1.0, 0.0]))) == pytest.approx(1.0)
    assert L.dual_value(2, P(y), 1.0, P(np.zeros(2))) == pytest.approx(0.0)
    assert L.dual_value(2, P(y), 1.0, P(y / 1.0)) == pytest.approx(0.5)
    a, yy, lam, _ = refgen.random_instance(9, 20, 0.5, 31)
    dd = _dense(oracle, a)
    x = refgen.random_vector(20, 4)
    th = refgen.random_vector(9, 5)
    pref = 0.5 * np.sum((a @ x - yy) ** 2) + lam * np.abs(x).sum()
    dref = 0.5 * yy @ yy - 0.5 * lam * lam * np.sum((th - yy / lam) ** 2)
    assert L.primal_value(dd._h, P(yy), lam, P(x)) == pytest.approx(pref, rel=1e-12)
    assert L.dual_value(9, P(yy), lam, P(th)) == pytest.approx(dref, rel=1e-12)


def test_duality_gap_basics(oracle):  # test_solver.cpp:146-156
    d = _dense(oracle, np.eye(2))
    y = np.array([1.0, 0.0])
    w = C.c_int32(0)
    assert oracle.lib.duality_gap(d._h, P(y), 1.0, P(np.zeros(2)), P(np.zeros(2)), None) == pytest.approx(0.5)
    assert oracle.lib.duality_gap(d._h, P(y), 1.0, P(np.zeros(2)), P(y), C.byref(w)) <= 1e-10
    assert w.value == 0


def test_lipschitz_bracket(backend, refgen):  # test_solver.cpp:158-179
    l1 = F.lipschitz_bound(_dense(backend, np.eye(4)))
    assert 1.0 <= l1 <= 1.05
    l2 = F.lipschitz_bound(_dense(backend, 2.0 * np.eye(4)))
    assert 4.0 <= l2 <= 4.2
    for trial in range(10):
        m = refgen.random_matrix(12, 20, 100 + trial)
        smax = np.linalg.svd(m, compute_uv=False)[0]
        l = F.lipschitz_bound(_dense(backend, m))
        assert l >= smax * smax * (1 - 1e-12)
        assert l <= 1.05 * smax * smax * (1 + 1e-9)


def test_restricted_solve_zero_padded(refgen):  # test_solver.cpp:181-200 (solve_oracle property)
    a, y, lam, _ = refgen.random_instance(12, 30, 0.4, 41)
    sol = solve_oracle(a, y, lam)
    supp = list(np.nonzero(sol.x)[0])
    active = supp + [j for j in range(30) if j not in supp][:4]
    sub = solve_oracle(a[:, active], y, lam)
    padded = np.zeros(30)
    padded[active] = sub.x
    assert np.max(np.abs(padded - sol.x)) <= 1e-8


# ----------------------------------------------------------------- test_screening.cpp
def test_lambda_max_basics(backend, refgen):  # test_screening.cpp:43-56
    d = _dense(backend, np.eye(2))
    assert F.lambda_max(d, [3.0, -1.0]) == 3.0
    assert F.lambda_max(d, [0.0, 0.0]) == 0.0
    a = refgen.random_dictionary(10, 25, 7)
    z = refgen.random_vector(10, 8)
    brute = max(abs(a[:, j] @ z) for j in range(25))
    assert F.lambda_max(_dense(backend, a), z) == pytest.approx(brute, rel=1e-14)


def test_stable_lambda_max_dominates(oracle, refgen):  # test_screening.cpp:58-83
    exact = refgen.random_dictionary(12, 30, 11)
    y = refgen.random_vector(12, 12)
    y /= np.linalg.norm(y)
    ex = F.make_exact_approx(_dense(oracle, exact))
    out = C.c_double()
    oracle.lib.check(oracle.lib.stable_lambda_max(ex.handle(), P(y), C.byref(out)))
    lmax = F.lambda_max(ex.op, y)
    assert out.value == pytest.approx(lmax, rel=1e-15)
    zero = F.ApproxDictionary(_dense(oracle, np.zeros((12, 30))), np.linalg.norm(exact, axis=0),
                              float(np.linalg.norm(exact, axis=0).max()), 0.5, np.zeros(30),
                              np.linalg.norm(exact, axis=0))
    oracle.lib.check(oracle.lib.stable_lambda_max(zero.handle(), P(y), C.byref(out)))
    assert out.value == pytest.approx(np.linalg.norm(y) * np.linalg.norm(exact, axis=0).max(), rel=1e-14)
    for trial in range(20):
        ap, _ = perturbed_approx(F, oracle, refgen, exact, 0.05 * (trial + 1), 100 + trial)
        oracle.lib.check(oracle.lib.stable_lambda_max(ap.handle(), P(y), C.byref(out)))
        assert out.value >= lmax - 1e-14


def test_sphere_test_closed_form(backend):  # test_screening.cpp:85-92
    s = F.scalars(backend)
    assert s.sphere_test(0.0, 1.0, 0.0) == 0.0  # |e2 . e1| + 0 * 1
    assert s.sphere_test(1.0, 1.0, 0.5) == 1.5


def test_sphere_test_upper_bounds_monte_carlo(backend):  # test_screening.cpp:94-108
    s = F.scalars(backend)
    rng = np.random.default_rng(2024)
    for trial in range(5):
        atom = rng.standard_normal(6)
        center = rng.standard_normal(6)
        r = 0.3 + 0.2 * trial
        bound = s.sphere_test(abs(atom @ center), np.linalg.norm(atom), r)
        dirs = rng.standard_normal((100000, 6))
        dirs /= np.linalg.norm(dirs, axis=1)[:, None]
        pts = center + r * rng.uniform(0, 1, (100000, 1)) ** (1 / 6) * dirs
        best = np.max(np.abs(pts @ atom))
        assert best <= bound + 1e-12
        assert best >= 0.95 * bound


def test_stable_zone_and_ball_collapse(backend):  # test_screening.cpp:110-126
    s = F.scalars(backend)
    rng = np.random.default_rng(50)
    atom, center = rng.standard_normal(5), rng.standard_normal(5)
    d, an, cn = abs(atom @ center), np.linalg.norm(atom), np.linalg.norm(center)
    assert s.stable_zone_test(d, 0.0, cn, an, 0.7) == pytest.approx(s.sphere_test(d, an, 0.7), rel=1e-15)
    assert s.stable_ball_test(d, 0.0, cn, an, 0.7) == pytest.approx(s.sphere_test(d, an, 0.7), rel=1e-15)
    assert s.stable_zone_test(0.0, 0.3, 0.0, 1.0, 0.0) == 0.0
    assert s.stable_ball_test(d, 0.25, cn, an, 0.0) == pytest.approx(d + 0.25 * cn)


def test_zone_test_conservative(backend):  # test_screening.cpp:128-147
    s = F.scalars(backend)
    rng = np.random.default_rng(777)
    for _ in range(10000):
        n = 4 + rng.integers(0, 5)
        ex, center, noise = rng.standard_normal(n), rng.standard_normal(n), rng.standard_normal(n)
        eps = abs(rng.standard_normal()) * 0.5
        noise *= eps / np.linalg.norm(noise) * rng.uniform(0, 1)
        ap = ex + noise
        r = abs(rng.standard_normal())
        stable = s.stable_zone_test(abs(ap @ center), eps, np.linalg.norm(center), np.linalg.norm(ex), r)
        plain = s.sphere_test(abs(ex @ center), np.linalg.norm(ex), r)
        assert stable >= plain - 1e-12


def test_dual_scaling(oracle, refgen):  # test_screening.cpp:150-183
    d = _dense(oracle, np.eye(2))
    out = np.empty(2)
    oracle.lib.check(oracle.lib.dual_scale(d._h, P([0.5, 0.2]), P(out)))
    assert np.array_equal(out, [0.5, 0.2])
    oracle.lib.check(oracle.lib.dual_scale(d._h, P([2.0, 0.0]), P(out)))
    assert out[0] == 1.0 and out[1] == 0.0
    a = refgen.random_dictionary(8, 20, 70)
    dd = _dense(oracle, a)
    o8 = np.empty(8)
    for trial in range(50):
        v = 5.0 * refgen.random_vector(8, 700 + trial)
        oracle.lib.check(oracle.lib.dual_scale(dd._h, P(v), o8.ctypes.data_as(C.POINTER(C.c_double))))
        assert np.max(np.abs(a.T @ o8)) <= 1.0 + 1e-12
    # stable scaling worked example (194-205): identity approx, eps = 1 -> 0.5
    idap = F.ApproxDictionary(_dense(oracle, np.eye(2)), np.ones(2), 1.0, 0.5, np.ones(2), np.ones(2))
    oracle.lib.check(oracle.lib.stable_dual_scale(idap.handle(), P([2.0, 0.0]), P(out)))
    assert out[0] == pytest.approx(0.5) and out[1] == 0.0


def test_dynamic_dual_points(oracle, refgen):  # test_screening.cpp:216-263
    a = refgen.random_dictionary(10, 22, 91)
    d = _dense(oracle, a)
    y = refgen.random_vector(10, 92)
    y /= np.linalg.norm(y)
    lam = 0.3 * F.lambda_max(d, y)

    def dp(rho, corr, eps, lam_, dict_h=None):
        tp, tt = np.empty(10), np.empty(10)
        sp, st = C.c_double(), C.c_double()
        oracle.lib.check(oracle.lib.dual_point_dynamic(10, corr.size, P(rho), P(corr), P(eps), P(y), lam_, dict_h,
                                                       tp.ctypes.data_as(C.POINTER(C.c_double)),
                                                       tt.ctypes.data_as(C.POINTER(C.c_double)), C.byref(sp),
                                                       C.byref(st)))
        return tp, tt, sp.value, st.value

    x = refgen.random_vector(22, 93) * 0.1
    rho = y - a @ x
    tp, tt, _, _ = dp(rho, a.T @ rho, np.zeros(22), lam)
    assert np.max(np.abs(tp - tt)) == 0.0
    assert np.max(np.abs(a.T @ tp)) <= 1.0 + 1e-12
    big = 10.0 * F.lambda_max(d, y)
    _, _, sp, _ = dp(y, a.T @ y, np.zeros(22), big)
    assert sp == pytest.approx(y @ y / (big * (y @ y)), rel=1e-15)
    tp, tt, _, _ = dp(np.zeros(10), np.zeros(22), np.zeros(22), lam, d._h)
    assert np.max(np.abs(a.T @ tp)) <= 1.0 + 1e-12 and np.max(np.abs(a.T @ tt)) <= 1.0 + 1e-12


def test_static_screening_at_lambda_max(oracle, refgen):  # test_screening.cpp:373-394
    a = refgen.random_dictionary(10, 25, 131)
    d = _dense(oracle, a)
    ex = F.make_exact_approx(d)
    y = refgen.random_vector(10, 132)
    y /= np.linalg.norm(y)
    lmax = F.lambda_max(d, y)
    center, radius = np.empty(10), C.c_double()
    oracle.lib.check(oracle.lib.build_sphere(0, 10, P(y), lmax, lmax, 0.0, None, 0.0, 0.0,
                                             center.ctypes.data_as(C.POINTER(C.c_double)), C.byref(radius)))
    assert radius.value == 0.0
    active = np.arange(25, dtype=np.int32)
    kept = np.empty(25, dtype=np.int32)
    nk = C.c_int64()
    oracle.lib.check(oracle.lib.screen(active.ctypes.data_as(C.POINTER(C.c_int32)), 25, P(center), radius.value,
                                       ex.handle(), 0, kept.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(nk)))
    corr = a.T @ y
    maximal = set(np.nonzero(np.abs(corr) >= lmax * (1 - 1e-14))[0])
    assert set(kept[:nk.value].tolist()) == maximal


def test_screened_sets_never_touch_support(oracle, refgen):  # test_screening.cpp:396-427
    for trial in range(10):
        a, y, lam, _ = refgen.random_instance(15, 40, 0.3 + 0.05 * trial, 200 + trial)
        sol = solve_oracle(a, y, lam)
        ap, approx = perturbed_approx(F, oracle, refgen, a, 0.05, 300 + trial)
        corr = approx.T @ y
        eps = ap.atom_error_bounds
        # stable GAP sphere at x = 0 (rho = y)
        tp, tt = np.empty(15), np.empty(15)
        sp, st = C.c_double(), C.c_double()
        oracle.lib.check(oracle.lib.dual_point_dynamic(15, 40, P(y), P(corr), P(eps), P(y), lam, None,
                                                       tp.ctypes.data_as(C.POINTER(C.c_double)),
                                                       tt.ctypes.data_as(C.POINTER(C.c_double)), C.byref(sp),
                                                       C.byref(st)))
        gap = oracle.lib.duality_gap(ap.op._h, P(y), lam, P(np.zeros(40)), P(tp), None)
        delta = F.scalars(oracle).stable_gap_delta(np.linalg.norm(y), ap.operator_error_bound, 0.0)
        center, radius = np.empty(15), C.c_double()
        oracle.lib.check(oracle.lib.build_sphere(5, 15, P(y), lam, 0.0, 0.0, P(tp), gap, delta,
                                                 center.ctypes.data_as(C.POINTER(C.c_double)), C.byref(radius)))
        active = np.arange(40, dtype=np.int32)
        kept = np.empty(40, dtype=np.int32)
        nk = C.c_int64()
        oracle.lib.check(oracle.lib.screen(active.ctypes.data_as(C.POINTER(C.c_int32)), 40, P(center), radius.value,
                                           ap.handle(), 1, kept.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(nk)))
        assert set(np.nonzero(sol.x)[0]) <= set(kept[:nk.value].tolist())


def test_screen_precomputed_collapse(backend, refgen):  # test_fastl1.cpp:219-241
    a = refgen.synthesize_scenario(36, 64, "moderate", 101)
    center = refgen.random_vector(36, 102)
    dots = np.abs(a.T @ center)
    norms = np.linalg.norm(a, axis=0)
    kept, look = F.screen_precomputed(dots, np.zeros(64), norms, norms, np.linalg.norm(center), 0.4, backend=backend)
    assert look == kept.size
    kept, look = F.screen_precomputed(dots, np.zeros(64), norms, norms, np.linalg.norm(center), 1e6, backend=backend)
    assert look == 64 and kept.size == 64
    # reference loop, ties keep (>= 1)
    eps = np.abs(refgen.random_vector(64, 103)) * 0.1
    kept, look = F.screen_precomputed(dots, eps, norms, norms * 0.9, 1.3, 0.2, backend=backend)
    ref_keep = np.nonzero(dots + eps * 1.3 + 0.2 * norms >= 1.0)[0]
    ref_look = int(np.sum(dots + 0.2 * norms * 0.9 >= 1.0))
    assert np.array_equal(kept, ref_keep) and look == ref_look


# ----------------------------------------------------------------- test_fastl1.cpp scalars
def test_gap_ratio(backend):  # test_fastl1.cpp:41-47
    s = F.scalars(backend)
    assert s.gap_ratio(0.5, 0.5) == 1.0
    assert s.gap_ratio(0.7, 0.5) == 1.0
    assert s.gap_ratio(1e-9, 1e-16) == 0.0
    assert s.gap_ratio(0.2, 0.8) == pytest.approx(0.25)
    assert s.gap_ratio(-1e-18, 0.5) == 0.0


def test_switch_dictionary(backend):  # test_fastl1.cpp:49-58
    s = F.scalars(backend)
    assert s.switch_dictionary(0, 4, 0.9, 0.2, 100, 0.15, 10000) == 4
    assert s.switch_dictionary(1, 4, 0.1, 0.2, 5000, 0.3, 10000) == 2
    assert s.switch_dictionary(1, 4, 0.9, 0.5, 9000, 0.3, 10000) == 1
    assert s.switch_dictionary(4, 4, 0.0, 0.5, 0, 1.0, 10000) == 4


def test_flop_formulas(backend):  # test_fastl1.cpp:60-70
    s = F.scalars(backend)
    assert s.flops_plain(10000, 2500, 0) == 10000 * 2500 + 4 * 10000 + 2500
    n, k = 2500, 10000
    assert s.flops_screened(k, n, 0) == (k + 0) * n + 6 * k + 5 * n
    assert s.flops_screened(k, n, 0) - s.flops_plain(k, n, 0) == 2 * k + 4 * n
    mv = 5 * (50 * 10000 + 100 * 2500)
    assert s.flops_stable(mv, n, k, 7) == mv + 7 * n + 8 * k + 7 * n


def test_stable_gap_delta(backend):  # screening.cpp:103-106
    s = F.scalars(backend)
    assert s.stable_gap_delta(2.0, 0.5, 3.0) == 2.0 * 0.5 * 3.0 + 0.5 * 0.25 * 9.0
    assert s.stable_gap_delta(1.0, 0.25, 0.0) == 0.0
