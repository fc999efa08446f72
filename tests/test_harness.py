"""The reference's experiment harness over the CUDA solver (paper_1812_06635_b200/
harness.py): ports of test_bench.cpp plus format / stream / SuKro-construction
parity checks. CPU tests need only the library's host code; -m gpu tests solve."""
from __future__ import annotations

import json
import math
import os
from pathlib import Path

import numpy as np
import pytest

from paper_1812_06635_b200 import fastl1 as F, harness as H

from _refgen import RefGen


def small_config(tmp=None) -> H.ExperimentConfig:  # test_bench.cpp:15-28
    return H.ExperimentConfig(n=36, k=100, scenario="moderate", lambda_ratios=[0.3], tol=1e-6, ranks=[1, 3],
                              trials=2, seed=11, out="" if tmp is None else str(tmp), use_gram=False)


# ---------------------------------------------------------------- host-only
def test_rng_stream_is_the_reference_stream(oracle):
    rg = RefGen(oracle)
    for seed in (0, 11 ^ 0xD1C7, 0x5EEDF00D):
        assert np.array_equal(H.rng_normals(seed, 1000), rg.normals(seed, 1000))


def test_config_validation():  # test_bench.cpp:39-54
    cfg = small_config()
    cfg.validate()
    for field, value in (("bernoulli_p", 0.0), ("lambda_ratios", [1.5]), ("gamma", 1.0), ("trials", 0),
                         ("jobs", 0), ("screen_interval", 0), ("ranks", []), ("tol", 0.0)):
        c = small_config()
        setattr(c, field, value)
        with pytest.raises(F.InvalidArgument):
            c.validate()
    c = small_config()
    c.lambda_ratios, c.lambda_grid = [], 0
    with pytest.raises(F.InvalidArgument):
        c.validate()
    c = small_config()
    c.rc_override = [0.1]
    with pytest.raises(F.InvalidArgument):
        c.validate()


def test_lambda_grid_log_spaced():  # test_bench.cpp:56-67
    cfg = small_config()
    cfg.lambda_ratios, cfg.lambda_grid = [], 5
    g = cfg.resolved_lambda_ratios()
    assert len(g) == 5 and abs(g[0] - 1e-2) < 1e-15 and g[-1] == 1.0
    for i in range(1, len(g)):
        assert abs(g[i] / g[i - 1] - g[1] / g[0]) <= 1e-12 * g[1] / g[0]
    cfg.lambda_grid = 1
    assert cfg.resolved_lambda_ratios() == [0.1]


def test_gamma_defaults():  # test_bench.cpp:69-78
    assert H.default_gamma("hard") == 0.5 and H.default_gamma("moderate") == 0.25 and H.default_gamma("easy") == 0.2
    cfg = small_config()
    cfg.scenario = "easy"
    assert cfg.resolved_gamma() == 0.2
    cfg.gamma = 0.33
    assert cfg.resolved_gamma() == 0.33


def test_config_json(tmp_path):  # test_bench.cpp:272-291
    p = tmp_path / "cfg.json"
    p.write_text('{"n": 36, "k": 100, "scenario": "easy", "lambda_ratio": 0.4, "tol": 1e-5, "ranks": [2, 5], '
                 '"trials": 3, "seed": 9, "solver": "ista", "rule": "dynamic"}')
    cfg = H.load_config_json(str(p))
    assert (cfg.n, cfg.k, cfg.scenario, cfg.lambda_ratios, cfg.trials) == (36, 100, "easy", [0.4], 3)
    assert cfg.solver == F.SOLVER_ISTA and cfg.rule == F.RULE_DYNAMIC and cfg.ranks == [2, 5] and cfg.seed == 9
    cfg.validate()
    p.write_text('{"rule": "gap_safe"}')
    with pytest.raises(F.InvalidArgument):
        H.load_config_json(str(p))
    p.write_text("{not json")
    with pytest.raises(F.InvalidArgument):
        H.load_config_json(str(p))
    with pytest.raises(F.InvalidArgument):
        H.load_config_json(str(tmp_path / "missing.json"))


def test_percentile_oracle():  # test_bench.cpp:221-227
    assert H.percentile([1.0, 2.0, 3.0, 4.0], 0.5) == pytest.approx(2.5)
    assert H.percentile([5.0], 0.25) == 5.0
    assert H.percentile([1.0, 2.0, 3.0, 4.0, 5.0], 0.25) == pytest.approx(2.0)
    assert H.percentile([4.0, 1.0, 3.0, 2.0], 0.0) == 1.0
    assert H.percentile([4.0, 1.0, 3.0, 2.0], 1.0) == 4.0
    assert math.isnan(H.percentile([], 0.5))


def _record(run_id, trial, ratio, variant, rows):
    tr = np.zeros(len(rows), dtype=F.TRACE_DTYPE)
    for i, (it, d, a, gap, gamma, fl, wall, nnz) in enumerate(rows):
        tr[i] = (it, d, a, gap, gamma, fl, wall, nnz, 0)
    return H.RunRecord(run_id=run_id, trial=trial, lambda_ratio=ratio, variant=variant, iterations=len(rows),
                       flops=rows[-1][5], wall_ms=rows[-1][6], converged=True, final_gap=0.0, trace=tr)


def test_csv_formats(tmp_path):
    """Headers, %.17g / %.3f formatting and column order of bench.cpp:336-414."""
    runs = [_record(0, 1, 0.3, F.VARIANT_PLAIN, [(0, 0, 100, 0.5, -1.0, 1234, 0.0123456, 7)]),
            _record(1, 1, 0.3, F.VARIANT_SCREENED, [(0, 1, 90, -1.0, 0.25, 1000, 1.5, 6)]),
            _record(2, 1, 0.3, F.VARIANT_MULTI_DICT, [(0, 2, 80, 1e-7, 0.1, 500, 2.25, 5)])]
    H.write_trace_csv(str(tmp_path / "trace.csv"), runs)
    lines = (tmp_path / "trace.csv").read_text().splitlines()
    assert lines[0] == "run_id,trial,lambda_ratio,variant,iter,dict_index,active_size,gap,gamma,flops_cum,wall_ms,x_nnz"
    assert lines[1] == "0,1,0.29999999999999999,plain,0,0,100,0.5,-1,1234,0.012,7"
    assert lines[2] == "1,1,0.29999999999999999,screened,0,1,90,-1,0.25,1000,1.500,6"
    assert lines[3] == "2,1,0.29999999999999999,fastl1,0,2,80,9.9999999999999995e-08,0.10000000000000001,500,2.250,5"
    row = H.SweepSummaryRow(trial=1, lambda_ratio=0.3, flops_plain=1234, flops_screened=1000, flops_multi=500,
                            time_plain=0.0123456, time_screened=1.5, time_multi=2.25, iters_plain=1, iters_screened=1,
                            iters_multi=1)
    H.write_summary_csv(str(tmp_path / "summary.csv"), [row])
    s = (tmp_path / "summary.csv").read_text().splitlines()
    assert s[0].startswith("trial,lambda_ratio,flops_plain,flops_screened,flops_fastl1,time_plain_ms")
    assert s[0].endswith("time_ratio_screened,time_ratio_fastl1,capped")
    cells = s[1].split(",")
    assert cells[:11] == ["1", "0.29999999999999999", "1234", "1000", "500", "0.012", "1.500", "2.250", "1", "1", "1"]
    assert float(cells[11]) == 1000 / 1234 and float(cells[12]) == 500 / 1234 and cells[-1] == "0"
    H.write_percentiles_csv(str(tmp_path / "pct.csv"), [row, row])
    p = (tmp_path / "pct.csv").read_text().splitlines()
    assert p[0] == "lambda_ratio,metric,p25,median,p75" and len(p) == 5
    assert p[1].startswith("0.29999999999999999,flops_ratio_screened,")


def test_emit_plot_data(tmp_path):  # test_bench.cpp:229-270 (empty trace + sentinel filtering)
    hdr = "run_id,trial,lambda_ratio,variant,iter,dict_index,active_size,gap,gamma,flops_cum,wall_ms,x_nnz\n"
    (tmp_path / "trace.csv").write_text(hdr)
    H.emit_plot_data(str(tmp_path / "trace.csv"), str(tmp_path / "plots"))
    assert (tmp_path / "plots" / "gap_iter.csv").read_text() == "lambda_ratio,trial,variant,iter,gap\n"
    runs = [_record(0, 0, 0.5, F.VARIANT_MULTI_DICT, [(0, 0, 100, -1.0, 0.9, 10, 0.1, 3), (1, 1, 50, 0.25, -1.0, 20, 0.2, 2)])]
    H.write_trace_csv(str(tmp_path / "t2.csv"), runs)
    H.emit_plot_data(str(tmp_path / "t2.csv"), str(tmp_path / "p2"))
    gap = (tmp_path / "p2" / "gap_iter.csv").read_text().splitlines()
    assert gap == ["lambda_ratio,trial,variant,iter,gap", "0.5,0,fastl1,1,0.25"]
    assert len((tmp_path / "p2" / "flops_iter.csv").read_text().splitlines()) == 3
    assert (tmp_path / "p2" / "gap_time.csv").read_text().splitlines()[1] == "0.5,0,fastl1,0.200,0.25"
    (tmp_path / "bad.csv").write_text(hdr + "1,2,3\n")
    with pytest.raises(F.InvalidArgument):
        H.emit_plot_data(str(tmp_path / "bad.csv"), str(tmp_path / "p3"))


def test_dictionary_files_roundtrip(tmp_path):  # dictionary.cpp:76-135
    rng = np.random.default_rng(3)
    a = np.asfortranarray(rng.standard_normal((7, 5)))
    H.save_blob(a, str(tmp_path / "a.blob"))
    raw = (tmp_path / "a.blob").read_bytes()
    assert raw[:8] == (7).to_bytes(4, "little") + (5).to_bytes(4, "little") and len(raw) == 8 + 8 * 35
    assert np.array_equal(H.load_blob(str(tmp_path / "a.blob")), a)
    H.save_csv(a, str(tmp_path / "a.csv"))
    assert np.array_equal(H.load_csv(str(tmp_path / "a.csv")), a)  # %.17g round-trips exactly
    (tmp_path / "r.csv").write_text("1,2\n3\n")
    (tmp_path / "e.csv").write_text("\n\n")
    (tmp_path / "t.blob").write_bytes(raw[:20])
    (tmp_path / "h.blob").write_bytes(b"\x00" * 8)
    for bad, fn in (("r.csv", H.load_csv), ("e.csv", H.load_csv), ("t.blob", H.load_blob), ("h.blob", H.load_blob),
                    ("missing.blob", H.load_blob)):
        with pytest.raises(F.InvalidArgument):
            fn(str(tmp_path / bad))


def test_synthesize_scenario_matches_restatement(oracle):
    rg = RefGen(oracle)
    a = H.synthesize_scenario(36, 100, "moderate", 11)
    b = rg.synthesize_scenario(36, 100, "moderate", 11)
    assert np.array_equal(a, b)
    assert np.allclose(np.linalg.norm(a, axis=0), 1.0, atol=1e-14)
    with pytest.raises(F.InvalidArgument):
        H.synthesize_scenario(35, 100, "moderate", 1)
    with pytest.raises(F.InvalidArgument):
        H.synthesize_scenario(36, 100, "medium", 1)


def test_sukro_construction_argument_errors():
    """build_sukro_sequence's argument checks (dictionary.cpp:19-33, 284-296) raise the
    reference's invalid_argument before any device work."""
    a = np.zeros((36, 100))
    for ranks in ([], [3, 1], [0], [2, 2]):
        with pytest.raises(F.InvalidArgument):
            H.build_sukro_levels(a, ranks)
    with pytest.raises(F.InvalidArgument, match="perfect square"):
        H.build_sukro_levels(np.zeros((35, 100)), [1])
    with pytest.raises(F.InvalidArgument, match="rearranged dimension"):
        H.build_sukro_levels(a, [61])


# ---------------------------------------------------------------- on the GPU
@pytest.mark.gpu
def test_generate_problem(cuda):  # test_bench.cpp:80-99
    cfg = small_config()
    a, b = H.generate_problem(cfg, 0), H.generate_problem(cfg, 0)
    assert np.array_equal(a.y, b.y) and np.array_equal(a.x_true, b.x_true)
    c = H.generate_problem(cfg, 1)
    assert np.max(np.abs(a.y - c.y)) > 0
    assert abs(np.linalg.norm(a.y) - 1.0) <= 1e-12
    assert np.max(np.abs(a.dict @ a.x_true - a.y)) <= 1e-12
    cfg.bernoulli_p = 1e-4
    for trial in range(20):
        assert np.count_nonzero(H.generate_problem(cfg, trial).x_true) >= 1


@pytest.mark.gpu
def test_sweep_summaries_and_deterministic_csvs(cuda, tmp_path):  # test_bench.cpp:120-190
    cfg = small_config(tmp_path / "sweep")
    out = H.run_sweep(cfg)
    assert len(out.runs) == 6 and len(out.summary) == 2 and not out.any_capped
    for r in out.runs:
        assert len(r.trace) and r.flops == int(r.trace["flops_cum"][-1])
    ta = (tmp_path / "sweep" / "trace.csv").read_text()
    sa = (tmp_path / "sweep" / "summary.csv").read_text()
    H.run_sweep(cfg)
    tb = (tmp_path / "sweep" / "trace.csv").read_text()
    sb = (tmp_path / "sweep" / "summary.csv").read_text()

    def strip(csv, cols):
        return [[c for i, c in enumerate(l.split(",")) if i not in cols] for l in csv.splitlines()]

    assert strip(ta, {10}) == strip(tb, {10})
    assert strip(sa, {5, 6, 7, 13, 14}) == strip(sb, {5, 6, 7, 13, 14})
    H.emit_plot_data(str(tmp_path / "sweep" / "trace.csv"), str(tmp_path / "plots"))
    total = sum(len(r.trace) for r in out.runs)
    gap_ok = sum(int(np.count_nonzero(r.trace["gap"] >= 0)) for r in out.runs)
    assert len((tmp_path / "plots" / "flops_iter.csv").read_text().splitlines()) - 1 == total
    assert len((tmp_path / "plots" / "gap_iter.csv").read_text().splitlines()) - 1 == gap_ok


@pytest.mark.gpu
def test_sweep_variants_agree(cuda):  # test_bench.cpp:192-219
    cfg = small_config()
    cfg.tol = 1e-7
    a = H.synthesize_scenario(cfg.n, cfg.k, cfg.scenario, cfg.seed)
    seq = H.sukro_sequence(a, cfg.ranks)
    d = seq.exact().op
    for trial in range(cfg.trials):
        y, _ = H.draw_signal(d, cfg.bernoulli_p, cfg.seed, trial)
        lam = cfg.lambda_ratios[0] * F.lambda_max(d, y)
        sw = F.SwitchConfig(tolerance=cfg.tol, gamma_threshold=cfg.resolved_gamma())
        vals = []
        for v in (F.VARIANT_PLAIN, F.VARIANT_SCREENED, F.VARIANT_MULTI_DICT):
            r = F.run_lasso(seq, y, lam, sw, F.RunOptions(variant=v))
            assert r.converged
            res = y - a @ r.x
            vals.append(0.5 * res @ res + lam * np.abs(r.x).sum())
        assert max(vals) - min(vals) <= 2.0 * cfg.tol


@pytest.mark.gpu
@pytest.mark.parametrize("n,k,scenario,seed,ranks", [(64, 256, "hard", 2, [2, 4]), (64, 256, "moderate", 5, [1, 2, 4]),
                                                     (2500, 10000, "moderate", 7, [5, 10, 15, 20])])
def test_sukro_construction_on_gpu_matches_restatement(cuda, oracle, n, k, scenario, seed, ranks):
    """build_sukro_sequence on the device (fl1_build_sukro_sequence: DMMA range finder,
    Householder QR, Jacobi SVD, streaming residual norms) against the LAPACK restatement
    of dictionary.cpp:253-357: per-level error bounds, approximate norms, RC exactly, and
    the Kronecker sums of the terms. The last case is the paper's 2500 x 10000 SuKro
    setting (RC 0.15 / 0.30 / 0.45 / 0.60, acceptance.cpp:448-460)."""
    rg = RefGen(oracle)
    a = rg.synthesize_scenario(n, k, scenario, seed)
    ours = H.build_sukro_levels(a, ranks, backend=cuda)
    ref = rg.build_sukro_sequence(a, ranks)
    assert len(ours) == len(ref) == len(ranks)
    for o, r in zip(ours, ref):
        assert o.rc == r["rc"]
        assert np.allclose(o.eps, r["eps"], rtol=1e-9, atol=1e-12)
        assert np.allclose(o.approx_norms, r["approx_norms"], rtol=1e-9, atol=1e-12)
        assert o.op_err == pytest.approx(r["op_err"], rel=1e-9)
        if n <= 64:
            ko = sum(np.kron(l, rr) for l, rr in o.terms)
            kr = sum(np.kron(l, rr) for l, rr in r["terms"])
            assert np.allclose(ko, kr, atol=1e-10)
    if n == 2500:
        assert [o.rc for o in ours] == [0.15, 0.30, 0.45, 0.60]


@pytest.mark.gpu
def test_sukro_residual_norms_unstaged_path(oracle, tmp_path):
    """The residual-norm pass reads the factor columns from global memory when they are too
    long to stage in shared memory (forced here with FL1_SUKRO_STAGE=0, in a child process):
    same levels as the LAPACK restatement."""
    import subprocess
    import sys

    code = (
        "import sys, numpy as np; sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests');"
        "from paper_1812_06635_b200 import harness as H, _abi, fastl1 as F;"
        "from _refgen import RefGen;"
        "orc = F.Backend(_abi.Library(sys.argv[1] + '/oracle/_build/libfl1oracle.so', 'orc_', extra=_abi.ORACLE_ONLY));"
        "rg = RefGen(orc); a = rg.synthesize_scenario(64, 256, 'moderate', 5);"
        "ours = H.build_sukro_levels(a, [1, 2, 4]); ref = rg.build_sukro_sequence(a, [1, 2, 4]);"
        "assert all(np.allclose(o.eps, r['eps'], rtol=1e-9, atol=1e-12) and "
        "np.allclose(o.approx_norms, r['approx_norms'], rtol=1e-9, atol=1e-12) for o, r in zip(ours, ref));"
        "print('ok')")
    root = str(Path(__file__).resolve().parents[1])
    env = dict(os.environ, FL1_SUKRO_STAGE="0")
    out = subprocess.run([sys.executable, "-c", code, root], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def _paper_config(tmp):
    """The paper's SuKro experiment shape: N = 2500, K = 10000, SuKro
    ranks 5 / 10 / 15 / 20 (RC 0.15 / 0.30 / 0.45 / 0.60), one trial, one lambda."""
    return H.ExperimentConfig(n=2500, k=10000, scenario="moderate", lambda_ratios=[0.3], tol=1e-5, ranks=[5, 10, 15, 20],
                              trials=1, seed=3, out=str(tmp), use_gram=False, screen_interval=10)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", ["small", "paper"])
def test_sweep_csvs_match_oracle(cuda, oracle, tmp_path, monkeypatch, shape):
    """one ExperimentConfig swept on the CUDA library and on the oracle (the
    same SuKro levels, built once on the device, feed both): trace / summary / percentile
    CSVs are identical in every integer and string column (iterations, dictionary index,
    preserved-set size, ledger, nnz, capped flags, flop ratios) and within the parity bar in
    the floating ones (gap, gamma); only the wall-clock columns differ (bench.cpp:255-421)."""
    import _parity as P

    if shape == "small":
        cfg = small_config(tmp_path / "gpu")
        cfg.lambda_ratios = [0.3, 0.6]
        cfg_o = small_config(tmp_path / "orc")
        cfg_o.lambda_ratios = [0.3, 0.6]
    else:
        cfg, cfg_o = _paper_config(tmp_path / "gpu"), _paper_config(tmp_path / "orc")
        oracle.lib.set_threads(os.cpu_count() or 1)
    a = H.synthesize_scenario(cfg.n, cfg.k, cfg.scenario, cfg.seed)
    levels = H.build_sukro_levels(a, cfg.ranks, backend=cuda)
    drawn = {}
    draw = H.draw_signal

    def draw_once(d, p, seed, trial):  # the signals of the CUDA sweep feed the oracle sweep too
        if trial not in drawn:
            drawn[trial] = draw(d, p, seed, trial)
        return drawn[trial]

    monkeypatch.setattr(H, "draw_signal", draw_once)
    H.run_sweep(cfg, backend=cuda, levels=levels)
    H.run_sweep(cfg_o, backend=oracle, levels=levels)
    walls = {"trace.csv": {10}, "summary.csv": {5, 6, 7, 13, 14}, "percentiles.csv": set()}
    floats = {"trace.csv": {7, 8}, "summary.csv": set(), "percentiles.csv": set()}
    for name in ("trace.csv", "summary.csv", "percentiles.csv"):
        g = [l.split(",") for l in (tmp_path / "gpu" / name).read_text().splitlines()]
        o = [l.split(",") for l in (tmp_path / "orc" / name).read_text().splitlines()]
        assert len(g) == len(o) and g[0] == o[0], name
        for rg_, ro in zip(g[1:], o[1:]):
            if name == "percentiles.csv" and "time" in ro[1]:
                continue  # time-ratio percentiles are wall clock
            for c, (x, y) in enumerate(zip(rg_, ro)):
                if c in walls[name]:
                    continue
                if c in floats[name]:
                    fx, fy = float(x), float(y)
                    assert fx == fy or abs(fx - fy) <= max(P.GAP_RTOL, 1e-6 if c == 8 else 0) * abs(fy) + 1e-14, (name, c, x, y)
                else:
                    assert x == y, (name, c, x, y)


@pytest.mark.gpu
def test_run_single_and_gram_sweep(cuda, tmp_path):
    """run_single (bench.cpp:240-249) equals the matching sweep run; a use_gram sweep
    gives the same iterations and ledgers as a direct one."""
    cfg = small_config(tmp_path / "g")
    cfg.trials = 1
    out_g = H.run_sweep(cfg)
    cfg2 = small_config(tmp_path / "d")
    cfg2.trials, cfg2.use_gram = 1, False
    out_d = H.run_sweep(cfg2)
    for rg, rd in zip(out_g.runs, out_d.runs):
        assert rg.iterations == rd.iterations and rg.flops == rd.flops and rg.converged == rd.converged
    single = H.run_single(cfg2, cfg2.lambda_ratios[0], 0, F.VARIANT_SCREENED)
    assert single.iterations == out_d.runs[1].iterations and single.flops == out_d.runs[1].flops
