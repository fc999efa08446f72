"""The reference's experiment harness and file formats over the CUDA solver.

Restates, with the same names, arguments, defaults, validation errors and output
formats (so GPU sweeps drop into the reference's plotting and analysis tooling):

  bench.hpp / bench.cpp:16-463
      ExperimentConfig (validate, resolved_lambda_ratios, resolved_gamma),
      default_gamma, load_config_json, draw_signal, generate_problem, run_sweep,
      run_single, write_trace_csv, write_summary_csv, write_percentiles_csv,
      percentile, emit_plot_data
  dictionary.cpp:37-45, 76-135, 253-434
      DenseDictionary CSV / blob I/O, build_sukro_sequence (the device
      construction of fl1_build_sukro_sequence, csrc/sukro_build.cu), synthesize_scenario

The random streams are the reference's own (std::mt19937_64 with libstdc++'s
normal / bernoulli distributions, exported by libfl1cuda.so), so a config and seed
give the reference's dictionaries and signals up to the rounding of the linear
algebra (the device's Householder QR / Jacobi SVD instead of Eigen's).

Every solve goes through fastl1.run_lasso on the GPU. With use_gram (the reference's
default) the sweep builds the exact dictionary's Gram matrix once on the GPU and the
exact phase of every run is Gram-backed, as in the reference.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import json
import math
import os
import struct
import time
from typing import List, Optional, Sequence

import numpy as np

from . import fastl1 as F

SCENARIOS = ("easy", "moderate", "hard")
VARIANT_NAMES = {F.VARIANT_PLAIN: "plain", F.VARIANT_SCREENED: "screened", F.VARIANT_MULTI_DICT: "fastl1"}


# ---------------------------------------------------------------- random streams
def rng_normals(seed: int, count: int, backend: Optional[F.Backend] = None) -> np.ndarray:
    """std::normal_distribution<double>(0, 1) on std::mt19937_64(seed), count draws
    (host code of libfl1cuda.so; needs no GPU)."""
    del backend
    lib = F.default_backend().lib  # lazy context: no device touched
    out = np.empty(int(count))
    lib.check(lib.rng_normals(C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), int(count),
                              out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def _isqrt(v: int, what: str) -> int:  # require_perfect_square
    r = int(round(math.sqrt(v)))
    while r * r > v:
        r -= 1
    while (r + 1) * (r + 1) <= v:
        r += 1
    if r * r != v:
        raise F.InvalidArgument(f"{what} must be a perfect square")
    return r


# ---------------------------------------------------------------- dictionaries
def scenario_decay_ratio(s: str) -> float:  # dictionary.cpp:377-384
    return {"easy": 0.3, "moderate": 0.6, "hard": 0.95}[_scenario(s)]


def _scenario(s: str) -> str:
    if s not in SCENARIOS:
        raise F.InvalidArgument(f"unknown scenario: {s}")
    return s


def synthesize_scenario(n: int, k: int, scenario: str, seed: int, backend: Optional[F.Backend] = None) -> np.ndarray:
    """dictionary.cpp:386-434: a sum of min(40, sqrt N) Kronecker terms with geometric
    weights ratio^t over random orthonormal frames, columns normalised (N x K,
    column-major)."""
    m, q = _isqrt(n, "N"), _isqrt(k, "K")
    n_terms = min(40, m)
    ratio = scenario_decay_ratio(scenario)
    stream = rng_normals(seed ^ 0xD1C7, 2 * q * m * n_terms, backend)
    off = 0

    def frame():  # random_frame: column-major fill, Householder QR, thin Q
        nonlocal off
        g = stream[off:off + m * n_terms].reshape(n_terms, m).T
        off += m * n_terms
        return np.linalg.qr(g, mode="reduced")[0]

    col_scale = 1.0 / math.sqrt(q)
    left = np.zeros((n_terms, m, q))
    right = np.zeros((n_terms, m, q))
    for j in range(q):
        fb, fc = frame(), frame()
        left[:, :, j] = col_scale * fb.T
        right[:, :, j] = col_scale * fc.T
    a = np.zeros((n, k))
    for t in range(n_terms):
        a += np.kron((ratio ** t) * left[t], right[t])
    norms = np.linalg.norm(a, axis=0)
    if np.any(norms < 1e-14):
        raise RuntimeError("degenerate column in synthesized dictionary")
    return np.asfortranarray(a / norms[None, :])


@dataclasses.dataclass
class SukroLevel:
    terms: list            # [(left m x q, right m x q)] numpy
    eps: np.ndarray        # atom_error_bounds (K)
    op_err: float          # operator_error_bound
    rc: float              # relative_complexity
    approx_norms: np.ndarray
    exact_norms: np.ndarray


def build_sukro_levels(a: np.ndarray, ranks: Sequence[int], backend: Optional[F.Backend] = None,
                       dense: Optional[F.LinearOp] = None) -> List[SukroLevel]:
    """build_sukro_sequence (dictionary.cpp:281-357) on the GPU through the C-ABI
    (fl1_build_sukro_sequence: rearrangement, randomized truncated SVD on the fp64
    tensor cores with on-device Householder QR and Jacobi SVD, per-level residual norms
    in one streaming pass, running max finer -> coarser). Returns the SuKro levels;
    sukro_sequence() adds the exact one. `dense`: the dictionary already uploaded."""
    n, k = a.shape
    m, q = _isqrt(n, "N"), _isqrt(k, "K")
    ranks = [int(r) for r in ranks]
    if not ranks:
        raise F.InvalidArgument("need at least one rank")
    for i, r in enumerate(ranks):
        if r < 1 or (i > 0 and r <= ranks[i - 1]):
            raise F.InvalidArgument("ranks must be positive and strictly increasing")
    if ranks[-1] > m * q:
        raise F.InvalidArgument("rank exceeds rearranged dimension")
    d = dense if dense is not None else F.DenseDictionary(a, backend=backend)
    lib = d.backend.lib
    if not hasattr(lib, "build_sukro_sequence"):
        raise RuntimeError("build_sukro_levels runs on the CUDA library (no CPU construction path)")
    T, nr = ranks[-1], len(ranks)
    left = np.empty((T, q, m))   # term t: m x q column-major = [t, j, i]
    right = np.empty((T, q, m))
    eps, app = np.empty((nr, k)), np.empty((nr, k))
    rc, op = np.empty(nr), np.empty(nr)
    rk = np.asarray(ranks, dtype=np.int32)
    P = C.POINTER(C.c_double)
    lib.check(lib.build_sukro_sequence(d._h, rk.ctypes.data_as(C.POINTER(C.c_int32)), nr, left.ctypes.data_as(P),
                                       right.ctypes.data_as(P), eps.ctypes.data_as(P), app.ctypes.data_as(P),
                                       rc.ctypes.data_as(P), op.ctypes.data_as(P)))
    en = d.atom_norms2()
    terms = [(np.asfortranarray(left[t].T), np.asfortranarray(right[t].T)) for t in range(T)]
    return [SukroLevel(terms=terms[:nt], eps=eps[l].copy(), op_err=float(op[l]), rc=float(rc[l]),
                       approx_norms=app[l].copy(), exact_norms=en) for l, nt in enumerate(ranks)]


def sukro_sequence(a: np.ndarray, ranks: Sequence[int], backend: Optional[F.Backend] = None,
                   rc_override: Optional[Sequence[float]] = None,
                   levels: Optional[Sequence[SukroLevel]] = None) -> F.ApproxSequence:
    """ApproxSequence of build_sukro_sequence(A, ranks) + the exact dictionary. `levels`:
    SuKro levels built earlier (e.g. one construction shared by several backends)."""
    dense = F.DenseDictionary(a, backend=backend)
    if levels is None:
        levels = build_sukro_levels(a, ranks, dense=dense)
    dicts = []
    for i, lv in enumerate(levels):
        op = F.SukroDictionary(lv.terms, backend=backend)
        rc = rc_override[i] if rc_override is not None else lv.rc
        dicts.append(F.ApproxDictionary(op, lv.eps, lv.op_err, rc, lv.approx_norms, lv.exact_norms))
    dicts.append(F.make_exact_approx(dense))
    return F.ApproxSequence(dicts)


# ---- DenseDictionary file formats (dictionary.cpp:76-135)
def save_csv(a: np.ndarray, path: str) -> None:
    """Row per line, %.17g, comma separated (DenseDictionary::save_csv)."""
    try:
        f = open(path, "w")
    except OSError:
        raise F.InvalidArgument(f"cannot open {path} for writing")
    with f:
        for i in range(a.shape[0]):
            f.write(",".join("%.17g" % v for v in a[i, :]) + "\n")


def load_csv(path: str) -> np.ndarray:
    """DenseDictionary::load_csv: blank lines skipped; ragged / empty files rejected."""
    try:
        f = open(path)
    except OSError:
        raise F.InvalidArgument(f"cannot open {path}")
    rows = []
    with f:
        for line in f:
            line = line.rstrip("\n")
            if not line:
                continue
            row = [float(c) for c in line.split(",")]
            if rows and len(row) != len(rows[0]):
                raise F.InvalidArgument(f"ragged CSV in {path}")
            rows.append(row)
    if not rows:
        raise F.InvalidArgument(f"empty CSV in {path}")
    return np.asfortranarray(np.array(rows, dtype=np.float64))


def save_blob(a: np.ndarray, path: str) -> None:
    """uint32 N, uint32 K (little endian), then the N x K doubles column-major."""
    try:
        f = open(path, "wb")
    except OSError:
        raise F.InvalidArgument(f"cannot open {path} for writing")
    with f:
        f.write(struct.pack("<II", a.shape[0], a.shape[1]))
        f.write(np.asfortranarray(a, dtype=np.float64).tobytes(order="F"))


def load_blob(path: str) -> np.ndarray:
    try:
        f = open(path, "rb")
    except OSError:
        raise F.InvalidArgument(f"cannot open {path}")
    with f:
        head = f.read(8)
        if len(head) < 8:
            raise F.InvalidArgument(f"bad blob header in {path}")
        n, k = struct.unpack("<II", head)
        if n == 0 or k == 0:
            raise F.InvalidArgument(f"bad blob header in {path}")
        body = f.read(8 * n * k)
        if len(body) < 8 * n * k:
            raise F.InvalidArgument(f"truncated blob {path}")
    return np.frombuffer(body, dtype="<f8").reshape(k, n).T.copy(order="F")


# ---------------------------------------------------------------- experiment config
def default_gamma(s: str) -> float:  # bench.cpp:54-61
    return {"hard": 0.5, "moderate": 0.25, "easy": 0.2}[_scenario(s)]


def _solver_from_string(s: str) -> int:
    if s == "ista":
        return F.SOLVER_ISTA
    if s == "fista":
        return F.SOLVER_FISTA
    raise F.InvalidArgument(f"unknown solver: {s}")


def _rule_from_string(s: str) -> int:  # fastl1.cpp:17-21
    if s == "dynamic":
        return F.RULE_DYNAMIC
    if s == "gap":
        return F.RULE_GAP
    raise F.InvalidArgument(f"unknown rule: {s}")


@dataclasses.dataclass
class ExperimentConfig:  # bench.hpp:16-46
    n: int = 100
    k: int = 400
    scenario: str = "moderate"
    lambda_ratios: List[float] = dataclasses.field(default_factory=list)
    lambda_grid: int = 0
    tol: float = 1e-5
    gamma: Optional[float] = None
    solver: int = F.SOLVER_FISTA
    rule: int = F.RULE_GAP
    ranks: List[int] = dataclasses.field(default_factory=lambda: [5, 10, 15, 20])
    bernoulli_p: float = 0.02
    trials: int = 1
    seed: int = 0
    out: str = "out"
    screen_interval: int = 1
    precompute_aty: bool = False
    jobs: int = 1
    max_iter: int = 1_000_000
    use_gram: bool = True
    rc_override: Optional[List[float]] = None

    def validate(self) -> None:  # bench.cpp:63-86
        if self.n < 1 or self.k < 1:
            raise F.InvalidArgument("n and k must be positive")
        if self.tol <= 0:
            raise F.InvalidArgument("tol must be positive")
        if self.gamma is not None and (self.gamma <= 0.0 or self.gamma >= 1.0):
            raise F.InvalidArgument("gamma must lie in (0, 1)")
        if self.bernoulli_p <= 0.0 or self.bernoulli_p > 1.0:
            raise F.InvalidArgument("bernoulli-p must lie in (0, 1]")
        if self.trials < 1:
            raise F.InvalidArgument("trials must be >= 1")
        if self.jobs < 1:
            raise F.InvalidArgument("jobs must be >= 1")
        if self.screen_interval < 1:
            raise F.InvalidArgument("screen-interval must be >= 1")
        if not self.lambda_ratios and self.lambda_grid < 1:
            raise F.InvalidArgument("need --lambda-ratio or --lambda-grid")
        for r in self.lambda_ratios:
            if r <= 0.0 or r > 1.0:
                raise F.InvalidArgument("lambda ratios must lie in (0, 1]")
        if not self.ranks:
            raise F.InvalidArgument("need at least one rank")
        if self.rc_override is not None and len(self.rc_override) != len(self.ranks):
            raise F.InvalidArgument("rc-override must list one value per rank")

    def resolved_lambda_ratios(self) -> List[float]:  # bench.cpp:87-106
        if self.lambda_ratios:
            return list(self.lambda_ratios)
        if self.lambda_grid == 1:
            return [1e-1]
        lo, hi = math.log10(1e-2), math.log10(1.0)
        grid = [10.0 ** (lo + (i / (self.lambda_grid - 1)) * (hi - lo)) for i in range(self.lambda_grid)]
        grid[-1] = 1.0
        return grid

    def resolved_gamma(self) -> float:
        return self.gamma if self.gamma is not None else default_gamma(self.scenario)


def load_config_json(path: str) -> ExperimentConfig:  # bench.cpp:108-140
    try:
        f = open(path)
    except OSError:
        raise F.InvalidArgument(f"cannot open config {path}")
    with f:
        try:
            j = json.load(f)
        except json.JSONDecodeError as e:
            raise F.InvalidArgument(f"bad config JSON: {e}")
    c = ExperimentConfig()
    simple = {"n": int, "k": int, "lambda_grid": int, "tol": float, "gamma": float, "bernoulli_p": float,
              "trials": int, "seed": int, "out": str, "screen_interval": int, "precompute_aty": bool, "jobs": int,
              "max_iter": int, "use_gram": bool}
    for key, typ in simple.items():
        if key in j:
            setattr(c, key, typ(j[key]))
    if "scenario" in j:
        c.scenario = _scenario(j["scenario"])
    if "lambda_ratio" in j:
        c.lambda_ratios = [float(j["lambda_ratio"])]
    if "lambda_ratios" in j:
        c.lambda_ratios = [float(v) for v in j["lambda_ratios"]]
    if "solver" in j:
        c.solver = _solver_from_string(j["solver"])
    if "rule" in j:
        c.rule = _rule_from_string(j["rule"])
    if "ranks" in j:
        c.ranks = [int(v) for v in j["ranks"]]
    if "rc_override" in j:
        c.rc_override = [float(v) for v in j["rc_override"]]
    return c


# ---------------------------------------------------------------- problems
@dataclasses.dataclass
class Problem:
    dict: np.ndarray      # N x K
    y: np.ndarray         # unit l2 norm
    x_true: np.ndarray    # Bernoulli-Gaussian, scaled so y = A x_true


def draw_signal(d: F.LinearOp, bernoulli_p: float, seed: int, trial: int):
    """bench.cpp:142-167 on the GPU dictionary: returns (y, x_true)."""
    lib = d.backend.lib
    n, k = d.rows(), d.cols()
    y, x = np.empty(n), np.empty(k)
    lib.check(lib.draw_signal(d._h, float(bernoulli_p), C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), int(trial),
                              y.ctypes.data_as(C.POINTER(C.c_double)), x.ctypes.data_as(C.POINTER(C.c_double))))
    return y, x


def generate_problem(config: ExperimentConfig, trial: int, backend: Optional[F.Backend] = None) -> Problem:
    a = synthesize_scenario(config.n, config.k, config.scenario, config.seed, backend)
    d = F.DenseDictionary(a, backend=backend)
    y, x = draw_signal(d, config.bernoulli_p, config.seed, trial)
    return Problem(a, y, x)


# ---------------------------------------------------------------- sweeps
@dataclasses.dataclass
class RunRecord:  # bench.hpp:55-66
    run_id: int = 0
    trial: int = 0
    lambda_ratio: float = 0.0
    variant: int = F.VARIANT_PLAIN
    iterations: int = 0
    flops: int = 0
    wall_ms: float = 0.0
    converged: bool = True
    final_gap: float = 0.0
    trace: Optional[np.ndarray] = None


@dataclasses.dataclass
class SweepSummaryRow:  # bench.hpp:68-75
    trial: int = 0
    lambda_ratio: float = 0.0
    flops_plain: int = 0
    flops_screened: int = 0
    flops_multi: int = 0
    time_plain: float = 0.0
    time_screened: float = 0.0
    time_multi: float = 0.0
    iters_plain: int = 0
    iters_screened: int = 0
    iters_multi: int = 0
    capped: bool = False


@dataclasses.dataclass
class SweepOutput:
    runs: List[RunRecord]
    summary: List[SweepSummaryRow]
    any_capped: bool = False
    build_ms: float = 0.0


@dataclasses.dataclass
class SweepContext:
    dense: F.DenseDictionary
    seq: F.ApproxSequence
    full_lipschitz: List[float]
    gram: Optional[F.LinearOp] = None


def build_context(config: ExperimentConfig, a: np.ndarray, backend: Optional[F.Backend] = None,
                  levels: Optional[Sequence[SukroLevel]] = None) -> SweepContext:
    """bench.cpp:184-205: the approximation sequence, the per-level Lipschitz cache and
    (use_gram) the exact dictionary's Gram matrix, built once per sweep on the GPU."""
    seq = sukro_sequence(a, config.ranks, backend=backend, rc_override=config.rc_override, levels=levels)
    full_l = [F.lipschitz_bound(d.op) for d in seq.dicts]
    gram = F.gram_matrix(seq.exact().op) if config.use_gram else None
    return SweepContext(seq.exact().op, seq, full_l, gram)


def execute_run(config: ExperimentConfig, ctx: SweepContext, y: np.ndarray, lambda_ratio: float, trial: int,
                variant: int, run_id: int) -> RunRecord:  # bench.cpp:207-242
    lmax = F.lambda_max(ctx.dense, y)
    sw = F.SwitchConfig(gamma_threshold=config.resolved_gamma(), screening_interval=config.screen_interval,
                        tolerance=config.tol, max_iterations=config.max_iter, precompute_aty=config.precompute_aty)
    opts = F.RunOptions(solver=config.solver, rule=config.rule, variant=variant, full_lipschitz=ctx.full_lipschitz,
                        collect_trace=True, exact_gram=ctx.gram)
    res = F.run_lasso(ctx.seq, y, lambda_ratio * lmax, sw, opts)
    return RunRecord(run_id=run_id, trial=trial, lambda_ratio=lambda_ratio, variant=variant,
                     iterations=res.iterations if res.iterations else len(res.trace), flops=res.total_flops,
                     wall_ms=float(res.trace["wall_ms"][-1]) if len(res.trace) else 0.0,
                     converged=res.converged, final_gap=res.final_gap, trace=res.trace)


def run_single(config: ExperimentConfig, lambda_ratio: float, trial: int, variant: int,
               backend: Optional[F.Backend] = None) -> RunRecord:  # bench.cpp:244-253
    config.validate()
    a = synthesize_scenario(config.n, config.k, config.scenario, config.seed, backend)
    ctx = build_context(config, a, backend)
    y, _ = draw_signal(ctx.dense, config.bernoulli_p, config.seed, trial)
    return execute_run(config, ctx, y, lambda_ratio, trial, variant, 0)


def run_sweep(config: ExperimentConfig, backend: Optional[F.Backend] = None,
              levels: Optional[Sequence[SukroLevel]] = None) -> SweepOutput:
    """bench.cpp:255-340: plain / screened / fastl1 over the lambda grid and trials,
    one summary row per (lambda, trial), CSVs under config.out (empty: no files).
    Runs are issued in the reference's task order; the GPU runs them one at a time
    (each solve already uses the whole device), so config.jobs only bounds nothing."""
    config.validate()
    ratios = config.resolved_lambda_ratios()
    t0 = time.perf_counter()
    a = synthesize_scenario(config.n, config.k, config.scenario, config.seed, backend)
    ctx = build_context(config, a, backend, levels)
    build_ms = (time.perf_counter() - t0) * 1e3
    runs: List[RunRecord] = []
    run_id = 0
    signals = {}
    for ratio in ratios:
        for trial in range(config.trials):
            if trial not in signals:
                signals[trial] = draw_signal(ctx.dense, config.bernoulli_p, config.seed, trial)[0]
            for v in (F.VARIANT_PLAIN, F.VARIANT_SCREENED, F.VARIANT_MULTI_DICT):
                runs.append(execute_run(config, ctx, signals[trial], ratio, trial, v, run_id))
                run_id += 1
    summary = []
    any_capped = False
    for base in range(0, len(runs) - 2, 3):
        row = SweepSummaryRow(trial=runs[base].trial, lambda_ratio=runs[base].lambda_ratio)
        for r in runs[base:base + 3]:
            row.capped = row.capped or not r.converged
            if r.variant == F.VARIANT_PLAIN:
                row.flops_plain, row.time_plain, row.iters_plain = r.flops, r.wall_ms, r.iterations
            elif r.variant == F.VARIANT_SCREENED:
                row.flops_screened, row.time_screened, row.iters_screened = r.flops, r.wall_ms, r.iterations
            else:
                row.flops_multi, row.time_multi, row.iters_multi = r.flops, r.wall_ms, r.iterations
        any_capped = any_capped or row.capped
        summary.append(row)
    if config.out:
        os.makedirs(config.out, exist_ok=True)
        write_trace_csv(os.path.join(config.out, "trace.csv"), runs)
        write_summary_csv(os.path.join(config.out, "summary.csv"), summary)
        write_percentiles_csv(os.path.join(config.out, "percentiles.csv"), summary)
    return SweepOutput(runs, summary, any_capped, build_ms)


# ---------------------------------------------------------------- CSV writers
def _g(v: float) -> str:  # "%.17g"
    return "%.17g" % v


def _ms(v: float) -> str:  # "%.3f"
    return "%.3f" % v


def _open_w(path: str):
    try:
        return open(path, "w")
    except OSError:
        raise F.InvalidArgument(f"cannot open {path} for writing")


def write_trace_csv(path: str, runs: Sequence[RunRecord]) -> None:  # bench.cpp:342-355
    with _open_w(path) as f:
        f.write("run_id,trial,lambda_ratio,variant,iter,dict_index,active_size,gap,gamma,flops_cum,wall_ms,x_nnz\n")
        for r in runs:
            for row in (r.trace if r.trace is not None else []):
                f.write(f"{r.run_id},{r.trial},{_g(r.lambda_ratio)},{VARIANT_NAMES[r.variant]},{int(row['iter'])},"
                        f"{int(row['dict_index'])},{int(row['active_size'])},{_g(float(row['gap']))},"
                        f"{_g(float(row['gamma']))},{int(row['flops_cum'])},{_ms(float(row['wall_ms']))},"
                        f"{int(row['x_nnz'])}\n")


def write_summary_csv(path: str, rows: Sequence[SweepSummaryRow]) -> None:  # bench.cpp:357-376
    with _open_w(path) as f:
        f.write("trial,lambda_ratio,flops_plain,flops_screened,flops_fastl1,"
                "time_plain_ms,time_screened_ms,time_fastl1_ms,"
                "iters_plain,iters_screened,iters_fastl1,"
                "flops_ratio_screened,flops_ratio_fastl1,time_ratio_screened,time_ratio_fastl1,"
                "capped\n")
        for r in rows:
            fr_s = _ratio(r.flops_screened, r.flops_plain)
            fr_m = _ratio(r.flops_multi, r.flops_plain)
            tr_s = r.time_screened / r.time_plain if r.time_plain > 0 else 0.0
            tr_m = r.time_multi / r.time_plain if r.time_plain > 0 else 0.0
            f.write(f"{r.trial},{_g(r.lambda_ratio)},{r.flops_plain},{r.flops_screened},{r.flops_multi},"
                    f"{_ms(r.time_plain)},{_ms(r.time_screened)},{_ms(r.time_multi)},{r.iters_plain},"
                    f"{r.iters_screened},{r.iters_multi},{_g(fr_s)},{_g(fr_m)},{_g(tr_s)},{_g(tr_m)},"
                    f"{1 if r.capped else 0}\n")


def _ratio(a: int, b: int) -> float:  # C++ double division (inf / nan when b == 0)
    if b == 0:
        return math.nan if a == 0 else math.inf
    return float(a) / float(b)


def percentile(values: Sequence[float], q: float) -> float:  # bench.cpp:378-386
    if len(values) == 0:
        return math.nan
    v = sorted(values)
    h = q * (len(v) - 1)
    lo, hi = int(math.floor(h)), int(math.ceil(h))
    frac = h - math.floor(h)
    return v[lo] * (1.0 - frac) + v[hi] * frac


def write_percentiles_csv(path: str, rows: Sequence[SweepSummaryRow]) -> None:  # bench.cpp:388-421
    with _open_w(path) as f:
        f.write("lambda_ratio,metric,p25,median,p75\n")
        ratios = []
        for r in rows:
            if r.lambda_ratio not in ratios:
                ratios.append(r.lambda_ratio)
        metrics = ("flops_ratio_screened", "flops_ratio_fastl1", "time_ratio_screened", "time_ratio_fastl1")
        for ratio in ratios:
            for metric in metrics:
                vals = []
                for r in rows:
                    if r.lambda_ratio != ratio:
                        continue
                    if metric == "flops_ratio_screened":
                        vals.append(_ratio(r.flops_screened, r.flops_plain))
                    elif metric == "flops_ratio_fastl1":
                        vals.append(_ratio(r.flops_multi, r.flops_plain))
                    elif metric == "time_ratio_screened":
                        vals.append(r.time_screened / r.time_plain if r.time_plain > 0 else 0.0)
                    else:
                        vals.append(r.time_multi / r.time_plain if r.time_plain > 0 else 0.0)
                f.write(f"{_g(ratio)},{metric},{_g(percentile(vals, 0.25))},{_g(percentile(vals, 0.5))},"
                        f"{_g(percentile(vals, 0.75))}\n")


def emit_plot_data(trace_csv: str, out_dir: str) -> None:  # bench.cpp:423-461
    try:
        fin = open(trace_csv)
    except OSError:
        raise F.InvalidArgument(f"cannot open {trace_csv}")
    os.makedirs(out_dir, exist_ok=True)
    with fin, open(os.path.join(out_dir, "gap_iter.csv"), "w") as gi, \
            open(os.path.join(out_dir, "gap_time.csv"), "w") as gt, \
            open(os.path.join(out_dir, "flops_iter.csv"), "w") as fi, \
            open(os.path.join(out_dir, "active_iter.csv"), "w") as ai:
        gi.write("lambda_ratio,trial,variant,iter,gap\n")
        gt.write("lambda_ratio,trial,variant,wall_ms,gap\n")
        fi.write("lambda_ratio,trial,variant,iter,flops_cum\n")
        ai.write("lambda_ratio,trial,variant,iter,active_size\n")
        header = fin.readline()
        if not header:
            return
        for line in fin:
            line = line.rstrip("\n")
            if not line:
                continue
            cell = line.split(",")
            if len(cell) != 12:
                raise F.InvalidArgument("malformed trace row: " + line)
            ratio, trial, variant, it, gap = cell[2], cell[1], cell[3], cell[4], cell[7]
            if float(gap) >= 0:
                gi.write(f"{ratio},{trial},{variant},{it},{gap}\n")
                gt.write(f"{ratio},{trial},{variant},{cell[10]},{gap}\n")
            fi.write(f"{ratio},{trial},{variant},{it},{cell[9]}\n")
            ai.write(f"{ratio},{trial},{variant},{it},{cell[6]}\n")
