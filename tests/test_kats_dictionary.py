"""Operator KATs ported from test_dictionary.cpp and acceptance.cpp criterion 5/6
(paths relative to /root/reference/proj/tests); the operator products also run
on libfl1cuda.so (-m gpu).
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_1812_06635_b200 import fastl1 as F, synthetic as syn


def test_dense_diagonal_kat(backend):  # test_dictionary.cpp:25-37
    d = F.DenseDictionary(np.diag([1.0, 2.0]), backend=backend)
    assert np.array_equal(d.apply([3.0, 1.0]), [3.0, 2.0])
    assert np.array_equal(d.apply_adjoint([3.0, 2.0]), [3.0, 4.0])
    assert np.array_equal(d.atom_norms2(), [1.0, 2.0])


def test_sukro_identity_kat(backend):  # test_dictionary.cpp:15-24
    s = F.SukroDictionary([(np.eye(2), np.eye(2))], backend=backend)
    assert np.array_equal(s.apply([1.0, 2.0, 3.0, 4.0]), [1.0, 2.0, 3.0, 4.0])
    assert np.array_equal(s.apply_adjoint([1.0, 2.0, 3.0, 4.0]), [1.0, 2.0, 3.0, 4.0])


def test_sukro_matches_dense_expansion(backend, refgen):  # test_dictionary.cpp:39-68
    rng = np.random.default_rng(7)
    shapes = [(2, 2, 2), (4, 4, 2), (3, 5, 3), (8, 16, 4), (16, 16, 1), (5, 12, 6)]
    shapes += [(int(rng.integers(1, 9)), int(rng.integers(1, 17)), int(rng.integers(1, 5))) for _ in range(20)]
    for m, q, t in shapes:
        lefts = [refgen.random_matrix(m, q, 7 + 31 * i) for i in range(t)]
        rights = [refgen.random_matrix(m, q, 7 + 31 * i + 7) for i in range(t)]
        dense = syn.kron_dense(lefts, rights)
        s = F.SukroDictionary(list(zip(lefts, rights)), backend=backend)
        x = rng.standard_normal(q * q)
        r = rng.standard_normal(m * m)
        scale = max(1.0, np.max(np.abs(dense)))
        assert np.max(np.abs(s.apply(x) - dense @ x)) <= 1e-10 * scale * max(1.0, np.abs(x).sum())
        assert np.max(np.abs(s.apply_adjoint(r) - dense.T @ r)) <= 1e-10 * scale * max(1.0, np.abs(r).sum())
        j = int(rng.integers(0, q * q))
        assert np.max(np.abs(s.column(j) - dense[:, j])) <= 1e-12 * scale
        assert s.matvec_flops() == t * (m * q * q + q * m * m)


def test_sukro_column_scale_extension(backend):
    """Column-normalised Kronecker sums (BASELINE config 3): A = Kron(.) diag(d)."""
    rng = np.random.default_rng(3)
    lefts = [rng.standard_normal((4, 6)) for _ in range(3)]
    rights = [rng.standard_normal((4, 6)) for _ in range(3)]
    d = rng.uniform(0.5, 2.0, 36)
    dense = syn.kron_dense(lefts, rights, d)
    s = F.SukroDictionary(list(zip(lefts, rights)), col_scale=d, backend=backend)
    x, r = rng.standard_normal(36), rng.standard_normal(16)
    assert np.allclose(s.apply(x), dense @ x, rtol=1e-12, atol=1e-12)
    assert np.allclose(s.apply_adjoint(r), dense.T @ r, rtol=1e-12, atol=1e-12)
    assert np.allclose(s.atom_norms2(), np.linalg.norm(dense, axis=0), rtol=1e-13)
    assert s.matvec_flops() == 3 * (4 * 36 + 6 * 16)  # the scale is not charged


def test_dimension_errors(backend):  # test_dictionary.cpp:70-76
    d = F.DenseDictionary(np.ones((3, 4)), backend=backend)
    with pytest.raises(F.InvalidArgument):
        d.apply(np.ones(3))
    with pytest.raises(F.InvalidArgument):
        d.apply_adjoint(np.ones(4))
    with pytest.raises(F.InvalidArgument):
        F.DenseDictionary(np.ones((0, 4)), backend=backend)
    with pytest.raises(F.InvalidArgument):
        F.SukroDictionary([(np.ones((2, 3)), np.ones((3, 3)))], backend=backend)
    with pytest.raises(F.InvalidArgument):
        d.column(4)


def test_rank1_kronecker_recovery(refgen):  # test_dictionary.cpp:78-87
    a = np.kron(refgen.random_matrix(4, 5, 1), refgen.random_matrix(4, 5, 2))
    lv = refgen.build_sukro_sequence(a, [1])
    assert lv[0]["eps"].max() <= 1e-10


def test_eps_monotone_and_rc(refgen):  # test_dictionary.cpp:89-122; acceptance.cpp:448-460
    a = refgen.random_dictionary(16, 16, 5)
    lv = refgen.build_sukro_sequence(a, [1, 2, 4])
    for i in range(1, len(lv)):
        assert np.all(lv[i]["eps"] <= lv[i - 1]["eps"] + 1e-15)
    assert lv[0]["rc"] == 0.5  # 16x16, rank 1: 1 * (4*16 + 4*16) / 256
    n, k, m, q = 2500, 10000, 50, 100
    assert [nt * (m * k + q * n) / (n * k) for nt in (5, 10, 15, 20)] == [0.15, 0.30, 0.45, 0.60]


def test_scenario_determinism_and_unit_norms(refgen):  # test_dictionary.cpp:134-169
    a1 = refgen.synthesize_scenario(16, 64, "moderate", 9)
    a2 = refgen.synthesize_scenario(16, 64, "moderate", 9)
    assert np.array_equal(a1, a2)
    assert np.allclose(np.linalg.norm(a1, axis=0), 1.0, atol=1e-12)


def test_lambda_max_and_lipschitz_of_sukro(backend):
    rng = np.random.default_rng(11)
    lefts = [rng.standard_normal((6, 8)) for _ in range(2)]
    rights = [rng.standard_normal((6, 8)) for _ in range(2)]
    dense = syn.kron_dense(lefts, rights)
    s = F.SukroDictionary(list(zip(lefts, rights)), backend=backend)
    y = rng.standard_normal(36)
    assert F.lambda_max(s, y) == pytest.approx(np.max(np.abs(dense.T @ y)), rel=1e-13)
    smax2 = np.linalg.svd(dense, compute_uv=False)[0] ** 2
    L = F.lipschitz_bound(s)
    assert smax2 * (1 - 1e-9) <= L <= 1.05 * smax2 * (1 + 1e-9)
