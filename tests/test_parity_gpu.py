"""GPU parity: libfl1cuda.so against the CPU oracle on the same seeded inputs,
through the C-ABI, at BASELINE.json's full sizes where the oracle finishes in
seconds, and through size-independent properties beyond that.

Parity bar (BASELINE north_star, tests/_parity.py): final objective within 1e-9
relative; final duality gap and every logged gap within GAP_RTOL relative (the
measured bound with margin; see _parity.py for the numerical argument); identical
final support; preserved sets equal at every iteration (trace integer fields);
ledger identical. Achieved discrepancies are recorded (FL1_PARITY_OUT).
"""
from __future__ import annotations

import os
import time

import numpy as np
import pytest

from paper_1812_06635_b200 import fastl1 as F, synthetic as syn

from _refgen import perturbed_approx

pytestmark = pytest.mark.gpu

from _parity import OBJ_RTOL, assert_parity, primal  # noqa: E402,F401  (shared parity bar + recorder)


@pytest.fixture(scope="module")
def oracle16(oracle):
    oracle.lib.set_threads(os.cpu_count() or 1)  # results are identical for any thread count
    return oracle


def run_both(cuda, oracle, build_seq, y, lam, cfg, opts):
    out = {}
    for tag, b in (("gpu", cuda), ("orc", oracle)):
        out[tag] = F.run_lasso(build_seq(b), y, lam, cfg, opts)
    return out["gpu"], out["orc"]


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_dense_configs_full_size(cuda, oracle16, name):
    """BASELINE configs[0], configs[1] at full size: FISTA + GAP every 10, gap <= 1e-6 P."""
    inst = syn.dense_instance(name)
    L = F.lipschitz_bound(F.DenseDictionary(inst.a, backend=cuda))
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L])
    g, o = run_both(cuda, oracle16, lambda b: F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(inst.a, backend=b))]),
                    inst.y, inst.lam, cfg, opts)
    assert g.converged
    assert_parity(g, o, inst.a, inst.y, inst.lam)
    assert g.final_gap <= 1e-6 * primal(inst.a, inst.y, inst.lam, g.x) * (1 + 1e-9)


@pytest.mark.parametrize("solver,rule,pre", [(F.SOLVER_ISTA, F.RULE_GAP, False), (F.SOLVER_FISTA, F.RULE_DYNAMIC, False),
                                             (F.SOLVER_FISTA, F.RULE_DYNAMIC, True)])
def test_c2_full_size_solver_rule_variants(cuda, oracle16, solver, rule, pre):
    """BASELINE configs[1] at full size under the other solver / rule / precompute_aty
    settings of the reference (fastl1.hpp:25-31, 85-96): ISTA with GAP, FISTA with the
    Dynamic Safe rule, and Dynamic with precompute_aty (fastl1.cpp:291-304, 521-548)."""
    inst = syn.dense_instance("c2")
    L = F.lipschitz_bound(F.DenseDictionary(inst.a, backend=cuda))
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6, precompute_aty=pre)
    opts = F.RunOptions(solver=solver, rule=rule, variant=F.VARIANT_SCREENED, full_lipschitz=[L])
    g, o = run_both(cuda, oracle16, lambda b: F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(inst.a, backend=b))]),
                    inst.y, inst.lam, cfg, opts)
    assert_parity(g, o, inst.a, inst.y, inst.lam)


@pytest.mark.parametrize("rule,pre", [(F.RULE_DYNAMIC, False), (F.RULE_DYNAMIC, True)])
def test_kronecker_sum_config_dynamic_rule(cuda, oracle16, rule, pre):
    """BASELINE configs[2] at full size (4096 x 16384, A1 -> A2 -> A4 -> A) with the stable
    Dynamic Safe rule (and precompute_aty: the exact level's A^T y for the dots)."""
    inst = syn.sukro_instance(seed=3)
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6, gamma_threshold=0.5,
                         precompute_aty=pre)
    g, o = run_both(cuda, oracle16, lambda b: _sukro_seq(inst, b), inst.y, inst.lam, cfg, F.RunOptions(rule=rule))
    assert_parity(g, o, inst.a, inst.y, inst.lam)


def test_cold_lipschitz_matches_oracle(cuda, oracle16):
    inst = syn.dense_instance("c1")
    lg = F.lipschitz_bound(F.DenseDictionary(inst.a, backend=cuda))
    lo = F.lipschitz_bound(F.DenseDictionary(inst.a, backend=oracle16))
    assert lg == pytest.approx(lo, rel=1e-12)
    smax2 = np.linalg.svd(inst.a, compute_uv=False)[0] ** 2
    assert smax2 * (1 - 1e-6) <= lg <= 1.05 * smax2 * (1 + 1e-9)


def _sukro_seq(inst, b):
    return syn.sukro_sequence(inst, b)


@pytest.mark.parametrize("size", ["small", "full"])
def test_kronecker_sum_config(cuda, oracle16, size):
    """BASELINE configs[2]: stable screening + switching A1 -> A2 -> A4 -> A (full: 4096 x 16384)."""
    if size == "small":
        inst = syn.sukro_instance(seed=3, m=16, q=32, nnz=30)
    else:
        inst = syn.sukro_instance(seed=3)
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6, gamma_threshold=0.5)
    g, o = run_both(cuda, oracle16, lambda b: _sukro_seq(inst, b), inst.y, inst.lam, cfg, F.RunOptions())
    assert g.converged
    assert g.switches.size >= 1
    assert_parity(g, o, inst.a, inst.y, inst.lam)


OPTION_MATRIX = [
    (s, r, v, pre)
    for s in (F.SOLVER_ISTA, F.SOLVER_FISTA)
    for r in (F.RULE_GAP, F.RULE_DYNAMIC)
    for v in (F.VARIANT_PLAIN, F.VARIANT_SCREENED, F.VARIANT_MULTI_DICT)
    for pre in ((False, True) if r == F.RULE_DYNAMIC else (False,))
]


@pytest.mark.parametrize("solver,rule,variant,pre", OPTION_MATRIX)
def test_option_matrix_small(cuda, oracle16, refgen, solver, rule, variant, pre):
    """Every solver / rule / variant combination on a perturbed-dense 3-level sequence."""
    a, y, lam, _ = refgen.random_instance(60, 180, 0.25, 4242, support=6)

    def build(b):
        c, _ = perturbed_approx(F, b, refgen, a, 0.05, 11, rc=0.3)
        f, _ = perturbed_approx(F, b, refgen, a, 0.01, 12, rc=0.6)
        f.atom_error_bounds = np.minimum(f.atom_error_bounds, c.atom_error_bounds)
        return F.ApproxSequence([c, f, F.make_exact_approx(F.DenseDictionary(a, backend=b))])

    cfg = F.SwitchConfig(screening_interval=3, max_iterations=20000, tolerance=1e-10, precompute_aty=pre,
                         gamma_threshold=0.5)
    g, o = run_both(cuda, oracle16, build, y, lam, cfg, F.RunOptions(solver=solver, rule=rule, variant=variant))
    assert_parity(g, o, a, y, lam)


@pytest.mark.parametrize("n,k", [(7, 13), (33, 1000), (511, 700), (513, 300), (1025, 90), (2049, 40)])
def test_ragged_shapes(cuda, oracle16, refgen, n, k):
    """Odd N (padded leading dimension), N not a multiple of the 2 KiB unit, K < #SMs."""
    a, y, lam, _ = refgen.random_instance(n, k, 0.3, 77 + n, support=min(5, k))
    cfg = F.SwitchConfig(screening_interval=2, max_iterations=5000, tolerance=1e-11)
    g, o = run_both(cuda, oracle16, lambda b: F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=b))]),
                    y, lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED))
    assert_parity(g, o, a, y, lam)


def test_bit_reproducible(cuda):
    inst = syn.dense_instance("c1")
    seq = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(inst.a, backend=cuda))])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    r1 = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED))
    r2 = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED))
    assert np.array_equal(r1.x, r2.x) and r1.final_gap == r2.final_gap
    assert np.array_equal(r1.trace["gap"], r2.trace["gap"])


def test_batched_bit_reproducible(cuda):
    """The lockstep's stream-K products reduce shared tiles in a fixed chunk order and the
    per-signal queue order does not enter the arithmetic: two runs of a batch give the
    same bits for every signal (x, gap trace, iteration counts)."""
    rng = np.random.default_rng(53)
    n, k, B = 256, 1024, 96
    a = syn.gaussian_dictionary(rng, n, k)
    Y = np.empty((n, B), order="F")
    for b in range(B):
        Y[:, b] = syn.observe(rng, a @ syn.sparse_signal(rng, k, 4 + b % 7), None, 30.0)
    lams = 0.25 * np.max(np.abs(a.T @ Y), axis=0)
    d = F.DenseDictionary(a, backend=cuda)
    seq = F.ApproxSequence([F.make_exact_approx(d)])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[F.lipschitz_bound(d)], collect_trace=True)
    r1 = F.run_lasso_batched(seq, Y, lams, cfg, opts, concurrency=0)
    r2 = F.run_lasso_batched(seq, Y, lams, cfg, opts, concurrency=0)
    assert r1[0].kernel_launches == 3
    for x, y in zip(r1, r2):
        assert x.iterations == y.iterations and np.array_equal(x.x, y.x)
        assert np.array_equal(x.trace["gap"], y.trace["gap"])


def test_trace_flush_and_resume(cuda, monkeypatch):
    """A device trace buffer smaller than the run forces kernel exits + resumes; the
    trajectory is unchanged bit for bit (both runs on the full grid: the flush path
    does not take the single-cluster route)."""
    monkeypatch.setenv("FL1_SINGLE_CLUSTER", "0")
    inst = syn.dense_instance("c1")
    seq = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(inst.a, backend=cuda))])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    ref = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED))
    monkeypatch.setenv("FL1_TRACE_CAP", "7")
    r = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED))
    assert r.kernel_launches == (ref.iterations + 6) // 7
    assert np.array_equal(r.x, ref.x)
    for f in ("iter", "active_size", "x_nnz", "gap", "flops_cum"):
        assert np.array_equal(r.trace[f], ref.trace[f]), f


def test_device_resident_entry_point(cuda):
    import torch

    inst = syn.dense_instance("c1")
    seq = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(inst.a, backend=cuda))])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED)
    y_dev = torch.from_numpy(inst.y).cuda()
    r1 = F.run_lasso_device(seq, y_dev.data_ptr(), inst.lam, cfg, opts)
    r2 = F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
    assert np.array_equal(r1.x, r2.x)
    assert r1.h2d_bytes < r2.h2d_bytes


def test_large_path_properties(cuda):
    """BASELINE configs[3] shape (8192 x 65536, 4 GiB), first three lambdas of the warm-started
    path: size-independent checks (certified gap recomputed independently, KKT, nesting)."""
    import torch

    n, k = 8192, 65536
    gen = torch.Generator(device="cuda").manual_seed(4)
    At = torch.randn(k, n, device="cuda", dtype=torch.float64, generator=gen)
    At /= At.norm(dim=1, keepdim=True)
    rng = np.random.default_rng(4)
    x0 = np.zeros(k)
    pos = rng.choice(k, 800, replace=False)
    x0[pos] = rng.standard_normal(800)
    x0t = torch.from_numpy(x0).cuda()
    clean = At.T @ x0t
    sigma = float(clean.norm()) / np.sqrt(n) * 10 ** (-20 / 20)
    y = (clean + sigma * torch.from_numpy(rng.standard_normal(n)).cuda()).cpu().numpy()
    d = F.DenseDictionaryDevice(At.data_ptr(), n, k, backend=cuda)
    lmax = F.lambda_max(d, y)
    corr = (At @ torch.from_numpy(y).cuda()).abs().max().item()
    assert lmax == pytest.approx(corr, rel=1e-12)
    L = F.lipschitz_bound(d)
    seq = F.ApproxSequence([F.make_exact_approx(d)])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    x = None
    yt = torch.from_numpy(y).cuda()
    for ratio in syn.CONFIGS["c4"]["lam_ratios"][:3]:
        lam = ratio * lmax
        r = F.run_lasso(seq, y, lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], x_init=x))
        assert r.converged
        xt = torch.from_numpy(r.x).cuda()
        rho = yt - At.T @ xt
        p = 0.5 * float(rho @ rho) + lam * float(xt.abs().sum())
        c = At @ rho
        s = min(max(float(yt @ rho) / (lam * float(rho @ rho)), -1 / float(c.abs().max())), 1 / float(c.abs().max()))
        dual = 0.5 * float(yt @ yt) - 0.5 * lam * lam * float(((s * rho - yt / lam) ** 2).sum())
        assert p - dual <= 1e-5 * p  # independent fp64 recomputation with the ray at x
        assert np.all(np.diff(r.trace["active_size"]) <= 0)
        nz = np.nonzero(r.x)[0]
        assert set(nz.tolist()) <= set(r.final_active.tolist())
        x = r.x


@pytest.mark.parametrize("concurrency", [1, 4, 16, 0, -1, -4, -16])
def test_batched_many_signal(cuda, oracle16, concurrency):
    """BASELINE configs[4] semantics (independent solves per signal), reduced batch:
    every batched result matches the oracle's own solve of that signal, both for
    concurrent sub-grid launches (concurrency > 0) and for the single launch of
    thread-block clusters (concurrency <= 0: cluster size -concurrency, 0 = default)."""
    rng = np.random.default_rng(5)
    n, k, B = 128, 512, 12
    a = syn.gaussian_dictionary(rng, n, k)
    Y = np.empty((n, B), order="F")
    lams = np.empty(B)
    for b in range(B):
        x0 = syn.sparse_signal(rng, k, 5)
        Y[:, b] = syn.observe(rng, a @ x0, None, 30.0)
        lams[b] = 0.25 * np.max(np.abs(a.T @ Y[:, b]))
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED)
    seq_g = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=cuda))])
    seq_o = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=oracle16))])
    res = F.run_lasso_batched(seq_g, Y, lams, cfg, opts, concurrency=concurrency)
    assert len(res) == B
    for b in range(B):
        o = F.run_lasso(seq_o, Y[:, b], lams[b], cfg, opts)
        assert res[b].converged
        assert_parity(res[b], o, a, Y[:, b], lams[b])


@pytest.mark.parametrize("csize", [1, 2, 8])
def test_batched_clusters_switching_and_trace(cuda, oracle16, csize):
    """Cluster mode with per-signal dictionary switching (stable screening over the
    SuKro levels) and full traces: every signal equals its own oracle solve,
    including the switch events and the per-iteration trace."""
    inst = syn.sukro_instance(seed=3, m=16, q=32, nnz=30)
    rng = np.random.default_rng(11)
    B = 6
    Y = np.empty((inst.a.shape[0], B), order="F")
    lams = np.empty(B)
    for b in range(B):
        Y[:, b] = syn.observe(rng, inst.a @ syn.sparse_signal(rng, inst.a.shape[1], 20 + 3 * b), None, 30.0)
        lams[b] = (0.2 + 0.05 * b) * np.max(np.abs(inst.a.T @ Y[:, b]))
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6, gamma_threshold=0.5)
    opts = F.RunOptions(collect_trace=True)
    res = F.run_lasso_batched(_sukro_seq(inst, cuda), Y, lams, cfg, opts, concurrency=-csize)
    seq_o = _sukro_seq(inst, oracle16)
    n_sw = 0
    for b in range(B):
        o = F.run_lasso(seq_o, Y[:, b], lams[b], cfg, opts)
        assert res[b].converged
        assert_parity(res[b], o, inst.a, Y[:, b], lams[b])
        assert len(res[b].trace) == len(o.trace)
        n_sw += res[b].switches.size
    assert n_sw >= 1


def test_batched_clusters_device_input(cuda):
    """Y resident in HBM (fl1_solve_batched_device) gives the same results as host Y,
    with no signal bytes copied host->device; an empty batch is a no-op."""
    import torch

    rng = np.random.default_rng(7)
    n, k, B = 200, 700, 9
    a = syn.gaussian_dictionary(rng, n, k)
    Y = np.empty((n, B), order="F")
    for b in range(B):
        Y[:, b] = syn.observe(rng, a @ syn.sparse_signal(rng, k, 8), None, 30.0)
    lams = 0.25 * np.max(np.abs(a.T @ Y), axis=0)
    seq = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=cuda))])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED)
    r_host = F.run_lasso_batched(seq, Y, lams, cfg, opts, concurrency=-2)
    y_dev = torch.from_numpy(np.ascontiguousarray(Y.T)).cuda()  # row b = signal b: N x B column-major
    r_dev = F.run_lasso_batched(seq, (n, B), lams, cfg, opts, concurrency=-2, y_dev_ptr=y_dev.data_ptr())
    for b in range(B):
        assert np.array_equal(r_host[b].x, r_dev[b].x)
        assert r_dev[b].h2d_bytes < r_host[b].h2d_bytes
    assert F.run_lasso_batched(seq, Y[:, :0], lams[:0], cfg, opts, concurrency=0) == []


@pytest.mark.parametrize("variant", [F.VARIANT_SCREENED, F.VARIANT_PLAIN])
@pytest.mark.parametrize("solver", [F.SOLVER_FISTA, F.SOLVER_ISTA])
def test_batched_lockstep_prefix(cuda, oracle16, variant, solver):
    """Batched solves with a cached full Lipschitz constant run in the lockstep
    engine (every step: DMMA contractions W = A V for power steps, Corr = A^T R for
    all signals; screening by per-signal masks) and, by the default policy, move to
    the per-signal engine after their first restricted power iteration: every signal
    still equals its own oracle solve, trace and ledger included. Ragged shapes: K
    not a multiple of the atom tile, B not a multiple of 64."""
    rng = np.random.default_rng(17)
    n, k, B = 230, 1000, 70
    a = syn.gaussian_dictionary(rng, n, k)
    Y = np.empty((n, B), order="F")
    for b in range(B):
        Y[:, b] = syn.observe(rng, a @ syn.sparse_signal(rng, k, 6 + b % 7), None, 30.0)
    lams = (0.2 + 0.1 * (np.arange(B) % 3)) * np.max(np.abs(a.T @ Y), axis=0)
    L = F.lipschitz_bound(F.DenseDictionary(a, backend=cuda))
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=3000, rel_tolerance=1e-6)
    opts = F.RunOptions(solver=solver, variant=variant, full_lipschitz=[L], collect_trace=True)
    seq_g = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=cuda))])
    seq_o = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=oracle16))])
    res = F.run_lasso_batched(seq_g, Y, lams, cfg, opts, concurrency=-2)
    assert res[0].kernel_launches == 3  # prefix + cluster engine + trace packing
    for b in range(0, B, 3 if variant == F.VARIANT_PLAIN else 1):
        o = F.run_lasso(seq_o, Y[:, b], lams[b], cfg, opts)
        assert_parity(res[b], o, a, Y[:, b], lams[b])
        assert len(res[b].trace) == len(o.trace)


@pytest.mark.parametrize("narrow", ["0", "1"])
def test_batched_lockstep_narrow_steps(cuda, oracle16, monkeypatch, narrow):
    """Lockstep steps with at most 12 unfinished signals run their products on the CUDA
    cores (FL1_LOCKSTEP_NARROW=1, default) instead of the DMMA tiles: with hand-off policy
    0 every signal stays in the lockstep to the end, so the narrow steps carry whole
    power iterations and FISTA tails; each signal equals its own oracle solve."""
    monkeypatch.setenv("FL1_LOCKSTEP_POLICY", "0")
    monkeypatch.setenv("FL1_LOCKSTEP_NARROW", narrow)
    rng = np.random.default_rng(31)
    n, k, B = 300, 1200, 14
    a = syn.gaussian_dictionary(rng, n, k)
    Y = np.empty((n, B), order="F")
    for b in range(B):
        Y[:, b] = syn.observe(rng, a @ syn.sparse_signal(rng, k, 4 + 2 * b), None, 30.0)
    lams = (0.15 + 0.05 * (np.arange(B) % 4)) * np.max(np.abs(a.T @ Y), axis=0)
    L = F.lipschitz_bound(F.DenseDictionary(a, backend=cuda))
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], collect_trace=True)
    seq_g = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=cuda))])
    seq_o = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=oracle16))])
    res = F.run_lasso_batched(seq_g, Y, lams, cfg, opts, concurrency=0)
    for b in range(B):
        assert_parity(res[b], F.run_lasso(seq_o, Y[:, b], lams[b], cfg, opts), a, Y[:, b], lams[b])


@pytest.mark.parametrize("k", [401, 1200, 4608])
def test_batched_lockstep_atom_counts(cuda, oracle16, monkeypatch, k):
    """An odd atom count leaves the per-signal K-strided rows (the power-iteration vectors
    the lockstep copies in 16-byte pieces) without a 16-byte pitch: such a batch runs on
    the per-signal engines instead (k = 401), an even one in the lockstep (k = 1200); both
    match the per-signal oracle solves. k = 4608 is the largest atom count whose
    per-signal lists fit the lockstep's staging area (prefix_max_atoms)."""
    monkeypatch.setenv("FL1_LOCKSTEP_POLICY", "0")
    rng = np.random.default_rng(47)
    n, B = 200, 24
    a = syn.gaussian_dictionary(rng, n, k)
    Y = np.empty((n, B), order="F")
    for b in range(B):
        Y[:, b] = syn.observe(rng, a @ syn.sparse_signal(rng, k, 3 + b % 5), None, 30.0)
    lams = 0.25 * np.max(np.abs(a.T @ Y), axis=0)
    L = F.lipschitz_bound(F.DenseDictionary(a, backend=cuda))
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], collect_trace=True)
    seq_g = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=cuda))])
    seq_o = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=oracle16))])
    res = F.run_lasso_batched(seq_g, Y, lams, cfg, opts, concurrency=0)
    assert res[0].kernel_launches == (3 if k % 2 == 0 else 2)  # lockstep + engines + trace packing
    for b in range(B):
        assert_parity(res[b], F.run_lasso(seq_o, Y[:, b], lams[b], cfg, opts), a, Y[:, b], lams[b])


@pytest.mark.parametrize("env", [("FL1_LOCKSTEP_TMA", "0"), ("FL1_SK_FANIN", "1"), ("FL1_SK_FANIN", "64"),
                                 ("FL1_LOCKSTEP_WIDTH", "0")])
def test_batched_lockstep_contraction_routes(cuda, oracle16, monkeypatch, env):
    """The lockstep's contraction variants against per-signal oracle solves: the split-K
    cp.async tiles (FL1_LOCKSTEP_TMA=0) and the stream-K TMA ring with every shared tile
    reduced by all its contributors (FL1_SK_FANIN=1) or by its chunk-0 holder alone (64),
    and full-width tiles only. Policy 0 keeps every signal in the lockstep to the end and
    no narrow CUDA-core steps, so wide, medium and one-signal-wide products all occur;
    with 70 signals (two column tiles) and 1200 atoms the tiles span several CTAs."""
    monkeypatch.setenv("FL1_LOCKSTEP_POLICY", "0")
    monkeypatch.setenv("FL1_LOCKSTEP_NARROW", "0")
    monkeypatch.setenv(*env)
    rng = np.random.default_rng(37)
    n, k, B = 300, 1200, 70
    a = syn.gaussian_dictionary(rng, n, k)
    Y = np.empty((n, B), order="F")
    for b in range(B):
        Y[:, b] = syn.observe(rng, a @ syn.sparse_signal(rng, k, 4 + b % 9), None, 30.0)
    lams = (0.15 + 0.05 * (np.arange(B) % 4)) * np.max(np.abs(a.T @ Y), axis=0)
    L = F.lipschitz_bound(F.DenseDictionary(a, backend=cuda))
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], collect_trace=True)
    seq_g = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=cuda))])
    seq_o = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=oracle16))])
    res = F.run_lasso_batched(seq_g, Y, lams, cfg, opts, concurrency=0)
    for b in range(B):
        assert_parity(res[b], F.run_lasso(seq_o, Y[:, b], lams[b], cfg, opts), a, Y[:, b], lams[b])


@pytest.mark.parametrize("policy", ["0", "1", "2", "3"])
def test_batched_prefix_matches_engine_only(cuda, monkeypatch, policy):
    """The lockstep engine changes only the route, not the answer, under every
    hand-off policy (0: never, 1: at the first shrink, 2: after the first power
    iteration, 3: at the first iteration after it with |S| <= FL1_HANDOFF_S): same
    supports, iteration counts and ledgers as the engine-only path."""
    if policy == "3":
        monkeypatch.setenv("FL1_HANDOFF_S", "64")
    monkeypatch.setenv("FL1_LOCKSTEP_POLICY", policy)
    rng = np.random.default_rng(23)
    n, k, B = 128, 512, 20
    a = syn.gaussian_dictionary(rng, n, k)
    Y = np.empty((n, B), order="F")
    for b in range(B):
        Y[:, b] = syn.observe(rng, a @ syn.sparse_signal(rng, k, 5), None, 30.0)
    lams = 0.25 * np.max(np.abs(a.T @ Y), axis=0)
    L = F.lipschitz_bound(F.DenseDictionary(a, backend=cuda))
    seq = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=cuda))])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L])
    r1 = F.run_lasso_batched(seq, Y, lams, cfg, opts, concurrency=0)
    monkeypatch.setenv("FL1_BATCH_PREFIX", "0")
    r2 = F.run_lasso_batched(seq, Y, lams, cfg, opts, concurrency=0)
    for x, y in zip(r1, r2):
        assert x.iterations == y.iterations and x.total_flops == y.total_flops
        assert np.array_equal(x.final_active, y.final_active)
        assert np.max(np.abs(x.x - y.x)) <= 1e-9 * max(1.0, np.max(np.abs(y.x)))


@pytest.mark.parametrize("policy", ["0", "2", "3"])
def test_batched_lockstep_edge_cases(cuda, oracle16, monkeypatch, policy):
    """Lockstep corner cases against per-signal oracle solves: a zero signal (exact
    fit: hand-off to the per-signal engine at iteration 0), lambda >= lambda_max
    (immediate convergence), an iteration cap reached inside the lockstep, a single
    signal, and a dictionary smaller than one contraction tile (K < 128, N < 64)."""
    monkeypatch.setenv("FL1_LOCKSTEP_POLICY", policy)
    rng = np.random.default_rng(29)
    for n, k, B, cap in ((50, 40, 5, 5000), (120, 300, 1, 5000), (120, 300, 6, 7)):
        a = syn.gaussian_dictionary(rng, n, k)
        Y = np.empty((n, B), order="F")
        lams = np.empty(B)
        for b in range(B):
            Y[:, b] = syn.observe(rng, a @ syn.sparse_signal(rng, k, 4), None, 30.0)
            lams[b] = 0.3 * np.max(np.abs(a.T @ Y[:, b]))
        if B >= 5:
            Y[:, 1] = 0.0
            lams[1] = 1.0                                      # exact fit from the start
            lams[2] = 1.5 * np.max(np.abs(a.T @ Y[:, 2]))      # lambda above lambda_max
        L = F.lipschitz_bound(F.DenseDictionary(a, backend=cuda))
        cfg = F.SwitchConfig(screening_interval=10, max_iterations=cap, rel_tolerance=1e-6)
        opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], collect_trace=True)
        seq_g = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=cuda))])
        seq_o = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=oracle16))])
        res = F.run_lasso_batched(seq_g, Y, lams, cfg, opts, concurrency=0)
        for b in range(B):
            o = F.run_lasso(seq_o, Y[:, b], lams[b], cfg, opts)
            assert res[b].converged == o.converged
            assert_parity(res[b], o, a, Y[:, b], lams[b])


def test_batched_beyond_lockstep_shared_memory(cuda, oracle16):
    """A batch whose per-signal index lists (3 x 4 B per signal) would overflow the
    lockstep's shared memory takes the per-signal engines instead (prefix_fits): 6,000
    small signals; every 500th, and every one that does not converge, against its own
    oracle solve. (Signal 581 oscillates to the iteration cap on both sides: after
    screening leaves 2 atoms, the warm-started restricted power iteration converges on
    the lower eigenvalue, so L is underestimated -- the reference's own behaviour.)"""
    rng = np.random.default_rng(43)
    n, k, B = 48, 96, 6000
    a = syn.gaussian_dictionary(rng, n, k)
    X0 = np.zeros((k, B))
    for b in range(B):
        X0[rng.choice(k, 3, replace=False), b] = rng.standard_normal(3)
    Y = np.asfortranarray(a @ X0 + 0.01 * rng.standard_normal((n, B)))
    lams = 0.3 * np.max(np.abs(a.T @ Y), axis=0)
    L = F.lipschitz_bound(F.DenseDictionary(a, backend=cuda))
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L])
    res = F.run_lasso_batched(F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=cuda))]), Y, lams,
                              cfg, opts, concurrency=0)
    assert res[0].kernel_launches == 2  # per-signal engines + trace packing: no lockstep launch
    seq_o = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=oracle16))])
    stuck = [b for b in range(B) if not res[b].converged]
    assert len(stuck) < 10
    for b in stuck:
        o = F.run_lasso(seq_o, Y[:, b], lams[b], cfg, opts)
        assert not o.converged and o.iterations == res[b].iterations
    for b in range(0, B, 500):
        if b not in stuck:
            assert_parity(res[b], F.run_lasso(seq_o, Y[:, b], lams[b], cfg, opts), a, Y[:, b], lams[b])


def test_single_cluster_route_matches_grid(cuda, oracle16, monkeypatch):
    """Small dictionaries solve on one 16-CTA cluster (cheaper barriers); the grid
    route gives the same trajectory and both match the oracle."""
    inst = syn.dense_instance("c1")
    seq = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(inst.a, backend=cuda))])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED)
    cl = F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
    monkeypatch.setenv("FL1_SINGLE_CLUSTER", "0")
    gr = F.run_lasso(seq, inst.y, inst.lam, cfg, opts)
    seq_o = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(inst.a, backend=oracle16))])
    o = F.run_lasso(seq_o, inst.y, inst.lam, cfg, opts)
    assert_parity(cl, o, inst.a, inst.y, inst.lam)
    assert_parity(gr, o, inst.a, inst.y, inst.lam)


def _c4_instance():
    """BASELINE configs[3] instance exactly as bench.make_c4_device builds it (torch CUDA
    generator seed 4): returns (At on the GPU, y, host column-major N x K view)."""
    import bench

    At, y = bench.make_c4_device(4, "cuda")
    return At, y, At.cpu().numpy().T


def test_large_path_all_lambdas_match_oracle(cuda, oracle16):
    """BASELINE configs[3] at full size (8192 x 65536, 4 GiB): the WHOLE 10-lambda
    warm-started path (0.9 -> 0.05 lambda_max, each to gap <= 1e-6 P) against the oracle
    on the same matrix, each side warm-started from its own previous solution as the
    reference path would be (the preserved set restarts at full per lambda):
    identical trajectories (preserved sets and nnz at every iteration, ledger, final set,
    support) and objective / gap within the parity bar at every lambda. lambda_9 has the
    largest preserved sets and the longest run (fastl1.cpp:459-645)."""
    n, k = 8192, 65536
    At, y, a = _c4_instance()
    d = F.DenseDictionaryDevice(At.data_ptr(), n, k, backend=cuda)
    L = F.lipschitz_bound(d)
    lmax = F.lambda_max(d, y)
    seq_g = F.ApproxSequence([F.make_exact_approx(d)])
    seq_o = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=oracle16))])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    xg = xo = None
    ratios = syn.CONFIGS["c4"]["lam_ratios"]
    assert len(ratios) == 10
    path = {"ratios": np.asarray(ratios), "lambda_max": lmax, "L": L, "threads": os.cpu_count() or 1}
    for i, ratio in enumerate(ratios):
        lam = ratio * lmax
        g = F.run_lasso(seq_g, y, lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], x_init=xg))
        t0 = time.perf_counter()
        o = F.run_lasso(seq_o, y, lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L], x_init=xo))
        t_o = time.perf_counter() - t0
        assert g.converged and o.converged
        assert_parity(g, o, a, y, lam, case=f"+[lambda_{i}]")
        assert g.final_gap <= 1e-6 * primal(a, y, lam, g.x) * (1 + 1e-9)
        nz = np.flatnonzero(o.x)
        path.update({f"l{i}/iterations": o.iterations, f"l{i}/active_size": o.trace["active_size"],
                     f"l{i}/x_nnz": o.trace["x_nnz"], f"l{i}/power_bytes": o.profile[7],
                     f"l{i}/oracle_s": t_o, f"l{i}/gpu_ms": g.device_ms, f"l{i}/x_idx": nz.astype(np.int32),
                     f"l{i}/x_val": o.x[nz]})
        xg, xo = g.x, o.x
    out = os.environ.get("FL1_C4_PATH_OUT")
    if out:  # the oracle's own c4 path (bench.py --impl reference replays windows of it)
        np.savez_compressed(out, **path)


def test_batched_full_size_config5_all_signals(cuda, oracle16):
    """BASELINE configs[4] at full size (512 signals on 1024 x 4096) through the default
    batched route (lockstep engine + cluster engines): EVERY signal equals the oracle's own
    per-signal solve (trajectory, ledger, support, objective and gap), the oracle solving
    the signals on a thread pool (one thread per solve, as bench.cpp:283-301)."""
    from concurrent.futures import ThreadPoolExecutor

    import bench

    a, Y, lams = bench.make_c5(5)
    dg = F.DenseDictionary(a, backend=cuda)
    L = F.lipschitz_bound(dg)
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L])
    res = F.run_lasso_batched(F.ApproxSequence([F.make_exact_approx(dg)]), Y, lams, cfg, opts)
    B = Y.shape[1]
    assert len(res) == B and all(r.converged for r in res)
    seq_o = F.ApproxSequence([F.make_exact_approx(F.DenseDictionary(a, backend=oracle16))])
    threads = os.cpu_count() or 1
    oracle16.lib.set_threads(1)
    try:
        with ThreadPoolExecutor(threads) as ex:
            orc = list(ex.map(lambda b: F.run_lasso(seq_o, Y[:, b], lams[b], cfg, opts), range(B)))
    finally:
        oracle16.lib.set_threads(threads)
    for b in range(B):
        assert_parity(res[b], orc[b], a, Y[:, b], lams[b], case=f"+[signal_{b}]")


@pytest.mark.parametrize("n,k", [(7, 13), (500, 2000), (2049, 300)])
def test_device_ingestion_norms(cuda, oracle16, n, k):
    """Dense dictionaries are ingested on the device (one H2D or D2D copy, atom norms by a
    kernel in the restatement's sequential order, dictionary.cpp:59-64): the norms are
    bit-identical to the oracle's for host and device input, and the two handles apply
    identically."""
    import torch

    rng = np.random.default_rng(n + k)
    a = np.asfortranarray(rng.standard_normal((n, k)))
    dh = F.DenseDictionary(a, backend=cuda)
    At = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()
    dd = F.DenseDictionaryDevice(At.data_ptr(), n, k, backend=cuda)
    do = F.DenseDictionary(a, backend=oracle16)
    assert np.array_equal(dh.atom_norms2(), do.atom_norms2())
    assert np.array_equal(dd.atom_norms2(), do.atom_norms2())
    r = rng.standard_normal(n)
    assert np.array_equal(dh.apply_adjoint(r), dd.apply_adjoint(r))


def test_sukro_norms_on_device(cuda, oracle16):
    """SuKro exact atom norms (column-scaled Kronecker sums) expanded on the device match
    the oracle's column-by-column norms."""
    inst = syn.sukro_instance(seed=3, m=16, q=32, nnz=30)
    sg, so = syn.sukro_sequence(inst, cuda), syn.sukro_sequence(inst, oracle16)
    for lg, lo in zip(sg.dicts, so.dicts):
        assert np.allclose(lg.op.atom_norms2(), lo.op.atom_norms2(), rtol=1e-15, atol=0)


def test_random_sweep(cuda, oracle16):
    """Seeded random instances (tests/_fuzz.py): ragged shapes, both single-solve routes, every
    solver / rule / variant / precompute_aty setting, absolute and relative tolerances, iteration
    caps, warm starts, multi-level sequences, and a batched call every fourth case -- each against
    its own oracle solve (integer trajectory, objective and x at the shared bar; gap floor per
    _fuzz.FUZZ_GAP_ULPS)."""
    import _fuzz

    fails = _fuzz.sweep(cuda, oracle16, 80, 20261021, verbose=False)
    assert not fails, fails


def test_random_sweep_sukro(cuda, oracle16):
    """Seeded random sum-of-Kronecker sequences (tests/_fuzz.py draw_sukro_case): ragged factor
    shapes (m 3-22, q up to 40: not multiples of the DMMA tiles), 2-6 terms, 1-3 approximate levels
    before the exact dictionary, every solver / rule / variant, precompute_aty, the Gram-backed exact
    phase and a batched call in a quarter of the cases -- each against its own oracle solve at the
    shared bar (dictionary.cpp:150-164 operators, fastl1.cpp:26-38 switching)."""
    import _fuzz

    fails = _fuzz.sweep_sukro(cuda, oracle16, 40, 20261022, verbose=False)
    assert not fails, fails

