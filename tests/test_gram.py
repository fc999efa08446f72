"""Gram-backed exact phase (RunOptions::exact_gram; fastl1.cpp:278-394, 584-600,
678-679): the oracle restates it; the CUDA engine runs it on the G matrix built by
fl1_gram_create. Gram and direct products are the same mathematics, so the trajectory
(iterations, preserved sets, ledger, support) is the direct one."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1812_06635_b200 import fastl1 as F, synthetic as syn

from _parity import assert_parity as _assert_parity  # noqa: E402  (shared parity bar)

# Gram vs direct are two different formulas for the same residual norms: the Gram phase forms
# ||y - A x||^2 = ||y||^2 - 2 x.A^T y + x.G x (fastl1.cpp:366-394), which cancels at the
# scale ||y||^2 / 2 >= P: measured <= 19 ulp of P (oracle Gram vs oracle direct), inside the
# shared bar's 64-ulp floor.
GRAM_GAP_ULPS = 64.0


def assert_parity(g, o, a, y, lam, **kw):
    kw.setdefault("gap_ulps", GRAM_GAP_ULPS)
    return _assert_parity(g, o, a, y, lam, **kw)

OPTIONS = [
    dict(solver=F.SOLVER_FISTA, rule=F.RULE_GAP, variant=F.VARIANT_SCREENED),
    dict(solver=F.SOLVER_ISTA, rule=F.RULE_GAP, variant=F.VARIANT_SCREENED),
    dict(solver=F.SOLVER_FISTA, rule=F.RULE_DYNAMIC, variant=F.VARIANT_SCREENED),
    dict(solver=F.SOLVER_FISTA, rule=F.RULE_GAP, variant=F.VARIANT_PLAIN),
]


def _instance(seed=31, n=150, k=600):
    rng = np.random.default_rng(seed)
    a = syn.gaussian_dictionary(rng, n, k)
    y = syn.observe(rng, a @ syn.sparse_signal(rng, k, 8), None, 30.0)
    return a, y, 0.2 * float(np.max(np.abs(a.T @ y)))


def test_gram_matrix(backend):
    a, _, _ = _instance()
    d = F.DenseDictionary(a, backend=backend)
    g = F.gram_matrix(d)
    assert (g.rows(), g.cols()) == (a.shape[1], a.shape[1])
    gm = np.stack([g.column(j) for j in range(0, a.shape[1], 97)], axis=1)
    assert np.allclose(gm, (a.T @ a)[:, ::97], atol=1e-12)


@pytest.mark.parametrize("opt", OPTIONS)
def test_gram_phase_matches_direct(backend, opt):
    a, y, lam = _instance()
    d = F.DenseDictionary(a, backend=backend)
    seq = F.ApproxSequence([F.make_exact_approx(d)])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-7)
    direct = F.run_lasso(seq, y, lam, cfg, F.RunOptions(**opt))
    gram = F.run_lasso(seq, y, lam, cfg, F.RunOptions(**opt, exact_gram=F.gram_matrix(d)))
    assert_parity(gram, direct, a, y, lam)


def test_gram_phase_after_switches(backend):
    """Multi-dictionary run: the SuKro levels use their own operators, the exact phase
    (after the last switch) runs on G."""
    inst = syn.sukro_instance(seed=3, m=16, q=32, nnz=30)
    seq = syn.sukro_sequence(inst, backend)
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-7, gamma_threshold=0.5)
    direct = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions())
    g = F.gram_matrix(seq.exact().op)
    gram = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(exact_gram=g))
    assert direct.switches.size >= 1
    assert_parity(gram, direct, inst.a, inst.y, inst.lam)


@pytest.mark.gpu
def test_gram_gpu_matches_oracle_gram(cuda, oracle):
    a, y, lam = _instance(seed=37, n=400, k=2000)
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-7)
    out = {}
    for tag, b in (("gpu", cuda), ("orc", oracle)):
        d = F.DenseDictionary(a, backend=b)
        seq = F.ApproxSequence([F.make_exact_approx(d)])
        out[tag] = F.run_lasso(seq, y, lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, exact_gram=F.gram_matrix(d)))
    assert out["gpu"].converged
    assert_parity(out["gpu"], out["orc"], a, y, lam)


@pytest.mark.gpu
def test_gram_rejects_wrong_shape(cuda):
    a, y, lam = _instance()
    d = F.DenseDictionary(a, backend=cuda)
    seq = F.ApproxSequence([F.make_exact_approx(d)])
    wrong = F.DenseDictionary(np.eye(7), backend=cuda)
    with pytest.raises(F.InvalidArgument):
        F.run_lasso(seq, y, lam, F.SwitchConfig(), F.RunOptions(exact_gram=wrong))


@pytest.mark.gpu
@pytest.mark.parametrize("prefix", ["0", "1"])
def test_gram_batched(cuda, oracle, monkeypatch, prefix):
    """Batched solves with an exact Gram: the cluster engines run their exact phase on
    G (lockstep or not, the trajectory is the direct one)."""
    monkeypatch.setenv("FL1_BATCH_PREFIX", prefix)
    rng = np.random.default_rng(41)
    n, k, B = 120, 500, 7
    a = syn.gaussian_dictionary(rng, n, k)
    Y = np.empty((n, B), order="F")
    for b in range(B):
        Y[:, b] = syn.observe(rng, a @ syn.sparse_signal(rng, k, 5), None, 30.0)
    lams = 0.25 * np.max(np.abs(a.T @ Y), axis=0)
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-7)
    dg = F.DenseDictionary(a, backend=cuda)
    L = F.lipschitz_bound(dg)
    seq_g = F.ApproxSequence([F.make_exact_approx(dg)])
    opts_g = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], exact_gram=F.gram_matrix(dg))
    res = F.run_lasso_batched(seq_g, Y, lams, cfg, opts_g, concurrency=-2)
    do = F.DenseDictionary(a, backend=oracle)
    seq_o = F.ApproxSequence([F.make_exact_approx(do)])
    opts_o = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], exact_gram=F.gram_matrix(do))
    for b in range(B):
        assert_parity(res[b], F.run_lasso(seq_o, Y[:, b], lams[b], cfg, opts_o), a, Y[:, b], lams[b])
