"""Python mirror of the reference fastl1 API for the hot path.

Names, argument meaning and error behaviour follow
/root/reference/proj/core/include/fastl1/{dictionary,fastl1,solver,screening}.hpp;
every call goes through the C-ABI of libfl1cuda.so (include/fl1cuda.h).
std::invalid_argument surfaces as ``InvalidArgument`` (a ValueError).

    DenseDictionary(entries)              dictionary.hpp:19-48
    SukroDictionary(terms, col_scale)     dictionary.hpp:53-81 (+ column scale extension)
    ApproxDictionary(...)                 dictionary.hpp:111-120
    make_exact_approx(dict)               dictionary.cpp:216-225
    ApproxSequence(dicts)                 dictionary.hpp:128-134 (validate on construction)
    SwitchConfig / RunOptions             fastl1.hpp:25-31, 85-96 (+ rel_tolerance, x_init)
    run_lasso / fastl1_solve              fastl1.hpp:101-111
    lambda_max / lipschitz_bound          screening.cpp:9-11, solver.cpp:108-114

The implementation library is chosen once per object through ``backend``;
the default is the CUDA library, which must have been built
(``__graft_entry__.build()``) — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from pathlib import Path
from typing import Callable, Optional, Sequence

import numpy as np

from . import _abi
from ._abi import InvalidArgument, Library

SOLVER_ISTA, SOLVER_FISTA = 0, 1
RULE_DYNAMIC, RULE_GAP = 0, 1
VARIANT_PLAIN, VARIANT_SCREENED, VARIANT_MULTI_DICT = 0, 1, 2

_SOLVERS = {"ista": SOLVER_ISTA, "fista": SOLVER_FISTA}
_RULES = {"dynamic": RULE_DYNAMIC, "gap": RULE_GAP}
_VARIANTS = {"plain": VARIANT_PLAIN, "screened": VARIANT_SCREENED, "multi_dict": VARIANT_MULTI_DICT}

PKG_DIR = Path(__file__).resolve().parent
CUDA_LIB_PATH = Path(os.environ.get("FL1_LIB", PKG_DIR / "libfl1cuda.so"))  # FL1_LIB: tuning variants


def solver_from_string(s: str) -> int:  # fastl1.cpp:11-15
    if s not in _SOLVERS:
        raise InvalidArgument("unknown solver: " + s)
    return _SOLVERS[s]


def rule_from_string(s: str) -> int:  # fastl1.cpp:17-21
    if s not in _RULES:
        raise InvalidArgument("unknown rule: " + s)
    return _RULES[s]


class Backend:
    """A loaded C-ABI implementation plus one device context."""

    def __init__(self, lib: Library, device: int = 0):
        self.lib = lib
        self.device = device
        self._ctx = None

    @property
    def ctx(self):
        if self._ctx is None:
            h = C.c_void_p()
            self.lib.check(self.lib.ctx_create(self.device, C.byref(h)))
            self._ctx = h
        return self._ctx

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            if self._ctx is not None:
                self.lib.ctx_destroy(self._ctx)
        except Exception:
            pass


_default: Optional[Backend] = None


def cuda_library() -> Library:
    if not CUDA_LIB_PATH.exists():
        raise RuntimeError(
            f"{CUDA_LIB_PATH} is missing: the CUDA extension is not built "
            "(run __graft_entry__.build()); there is no CPU fallback")
    return Library(CUDA_LIB_PATH, "fl1_", extra=_abi.PRODUCT_ONLY)


def default_backend() -> Backend:
    global _default
    if _default is None:
        _default = Backend(cuda_library(), int(os.environ.get("FL1_DEVICE", "0")))
    return _default


def set_default_backend(b: Backend) -> None:
    global _default
    _default = b


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _vec(v, n: Optional[int] = None, what: str = "vector") -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))
    if n is not None and a.size != n:
        raise InvalidArgument(f"{what} has wrong length")
    return a


class LinearOp:
    """Common base of the two operator kinds (dictionary.hpp:86-104)."""

    backend: Backend
    _h: C.c_void_p

    def _lib(self) -> Library:
        return self.backend.lib

    def rows(self) -> int:
        r, c = C.c_int64(), C.c_int64()
        self._lib().check(self._lib().dict_shape(self._h, C.byref(r), C.byref(c)))
        return r.value

    def cols(self) -> int:
        r, c = C.c_int64(), C.c_int64()
        self._lib().check(self._lib().dict_shape(self._h, C.byref(r), C.byref(c)))
        return c.value

    @property
    def shape(self):
        return (self.rows(), self.cols())

    def is_dense(self) -> bool:
        return bool(self._lib().dict_is_dense(self._h))

    def matvec_flops(self) -> int:
        return int(self._lib().dict_matvec_flops(self._h))

    def atom_norms2(self) -> np.ndarray:
        out = np.empty(self.cols())
        self._lib().check(self._lib().dict_atom_norms(self._h, _dptr(out)))
        return out

    def apply(self, x) -> np.ndarray:
        x = _vec(x)
        if x.size != self.cols():
            raise InvalidArgument("matvec: x has wrong length")
        out = np.empty(self.rows())
        self._lib().check(self._lib().dict_apply(self._h, _dptr(x), _dptr(out)))
        return out

    def apply_adjoint(self, r) -> np.ndarray:
        r = _vec(r)
        if r.size != self.rows():
            raise InvalidArgument("adjoint matvec: r has wrong length")
        out = np.empty(self.cols())
        self._lib().check(self._lib().dict_apply_adjoint(self._h, _dptr(r), _dptr(out)))
        return out

    def column(self, j: int) -> np.ndarray:
        out = np.empty(self.rows())
        self._lib().check(self._lib().dict_column(self._h, int(j), _dptr(out)))
        return out

    def __del__(self):  # pragma: no cover
        try:
            self._lib().dict_destroy(self._h)
        except Exception:
            pass


class DenseDictionary(LinearOp):
    """N x K column-major dictionary resident on the backend (dictionary.hpp:19-48)."""

    def __init__(self, entries, backend: Optional[Backend] = None):
        self.backend = backend or default_backend()
        a = np.asfortranarray(np.asarray(entries, dtype=np.float64))
        if a.ndim != 2:
            raise InvalidArgument("dictionary must be a matrix")
        n, k = a.shape
        if n < 1 or k < 1:
            raise InvalidArgument("dictionary must have at least one row and one column")
        self._h = C.c_void_p()
        self._lib().check(self._lib().dict_dense(self.backend.ctx, _dptr(a), n, k, C.byref(self._h)))


class _Handle(LinearOp):
    """A dictionary handle produced by the library (e.g. a Gram matrix)."""

    def __init__(self, h, backend: Backend):
        self.backend = backend
        self._h = h


def gram_matrix(d: LinearOp) -> LinearOp:
    """G = A^T A of a dense dictionary as a dense K x K dictionary, computed by the
    backend (one GPU GEMM; the oracle on the host) -- RunOptions.exact_gram
    (fastl1.hpp:89-91), as the reference harness builds it (bench.cpp:190-197)."""
    h = C.c_void_p()
    d._lib().check(d._lib().gram_create(d._h, C.byref(h)))
    return _Handle(h, d.backend)


class DenseDictionaryDevice(LinearOp):
    """Dense dictionary uploaded from a device pointer (torch tensor data_ptr)."""

    def __init__(self, dev_ptr: int, n: int, k: int, backend: Optional[Backend] = None):
        self.backend = backend or default_backend()
        self._h = C.c_void_p()
        self._lib().check(self._lib().dict_dense_device(self.backend.ctx, C.c_void_p(dev_ptr), n, k, C.byref(self._h)))


class SukroDictionary(LinearOp):
    """sum_t B_t (x) C_t with optional column scale (dictionary.hpp:53-81).

    terms: sequence of (left B_t, right C_t), each m x q.
    """

    def __init__(self, terms: Sequence, col_scale=None, backend: Optional[Backend] = None):
        self.backend = backend or default_backend()
        if len(terms) < 1:
            raise InvalidArgument("SuKro needs at least one term")
        lefts = [np.asfortranarray(np.asarray(t[0], dtype=np.float64)) for t in terms]
        rights = [np.asfortranarray(np.asarray(t[1], dtype=np.float64)) for t in terms]
        m, q = lefts[0].shape
        for b, c in zip(lefts, rights):
            if b.shape != (m, q) or c.shape != (m, q):
                raise InvalidArgument("all SuKro factors must share one shape")
        self._keep = (lefts, rights)
        L = (C.POINTER(C.c_double) * len(terms))(*[_dptr(b) for b in lefts])
        R = (C.POINTER(C.c_double) * len(terms))(*[_dptr(c) for c in rights])
        sc = None
        if col_scale is not None:
            sc = _vec(col_scale, q * q, "col_scale")
            self._keep = (lefts, rights, sc)
        self._h = C.c_void_p()
        self._lib().check(self._lib().dict_sukro(self.backend.ctx, len(terms), m, q, L, R,
                                                 _dptr(sc) if sc is not None else None, C.byref(self._h)))


@dataclasses.dataclass
class ApproxDictionary:
    op: LinearOp
    atom_error_bounds: np.ndarray
    operator_error_bound: float
    relative_complexity: float
    approx_atom_norms2: np.ndarray
    exact_atom_norms2: np.ndarray
    _h: Optional[C.c_void_p] = dataclasses.field(default=None, repr=False)

    def is_exact(self) -> bool:
        return self.operator_error_bound == 0.0

    def handle(self):
        if self._h is None:
            lib = self.op.backend.lib
            k = self.op.cols()
            eps = _vec(self.atom_error_bounds, k, "atom_error_bounds")
            an = _vec(self.approx_atom_norms2, k, "approx_atom_norms2")
            en = _vec(self.exact_atom_norms2, k, "exact_atom_norms2")
            h = C.c_void_p()
            lib.check(lib.approx_create(self.op._h, _dptr(eps), float(self.operator_error_bound),
                                        float(self.relative_complexity), _dptr(an), _dptr(en), C.byref(h)))
            self._h = h
        return self._h


def make_exact_approx(d: LinearOp) -> ApproxDictionary:  # dictionary.cpp:216-225
    if not d.is_dense():
        raise InvalidArgument("make_exact_approx needs a dense dictionary")
    norms = d.atom_norms2()
    return ApproxDictionary(d, np.zeros(d.cols()), 0.0, 1.0, norms.copy(), norms.copy())


class ApproxSequence:
    """Ordered approximations ending with the exact dictionary (validated)."""

    def __init__(self, dicts: Sequence[ApproxDictionary]):
        self.dicts = list(dicts)
        if not self.dicts:
            raise InvalidArgument("empty approximation sequence")
        self.backend = self.dicts[0].op.backend
        lib = self.backend.lib
        arr = (C.c_void_p * len(self.dicts))(*[d.handle().value for d in self.dicts])
        self._h = C.c_void_p()
        lib.check(lib.seq_create(arr, len(self.dicts), C.byref(self._h)))

    def levels(self) -> int:
        return len(self.dicts)

    def exact(self) -> ApproxDictionary:
        return self.dicts[-1]

    def __del__(self):  # pragma: no cover
        try:
            self.backend.lib.seq_destroy(self._h)
        except Exception:
            pass


@dataclasses.dataclass
class SwitchConfig:  # fastl1.hpp:25-31
    gamma_threshold: float = 0.5
    screening_interval: int = 1
    tolerance: float = 1e-6
    max_iterations: int = 1_000_000
    precompute_aty: bool = False
    rel_tolerance: float = 0.0  # extension (0 = reference absolute tolerance)

    def c(self) -> _abi.SwitchConfigC:
        return _abi.SwitchConfigC(self.gamma_threshold, self.screening_interval, self.tolerance,
                                  self.max_iterations, 1 if self.precompute_aty else 0, self.rel_tolerance)


@dataclasses.dataclass
class ScreeningEvent:  # fastl1.hpp:74-83
    iter: int
    dict_index: int
    center: np.ndarray
    radius: float
    theta_prime: np.ndarray
    theta_tilde: np.ndarray
    scale_prime: float
    scale_tilde: float
    active_before: np.ndarray
    kept: np.ndarray


@dataclasses.dataclass
class RunOptions:  # fastl1.hpp:85-96
    solver: int = SOLVER_FISTA
    rule: int = RULE_GAP
    variant: int = VARIANT_MULTI_DICT
    full_lipschitz: Optional[Sequence[float]] = None
    collect_trace: bool = True
    observer: Optional[Callable[[ScreeningEvent], None]] = None
    x_init: Optional[np.ndarray] = None  # extension: warm start
    exact_gram: Optional["LinearOp"] = None  # K x K Gram of the exact dictionary (gram_matrix)


TRACE_DTYPE = np.dtype([("iter", "<u8"), ("dict_index", "<i4"), ("active_size", "<i4"), ("gap", "<f8"),
                        ("gamma", "<f8"), ("flops_cum", "<u8"), ("wall_ms", "<f8"), ("x_nnz", "<i4"),
                        ("pad_", "<i4")])
SWITCH_DTYPE = np.dtype([("iter", "<u8"), ("from", "<i4"), ("to", "<i4"), ("speed", "<i4"), ("pad_", "<i4")])


@dataclasses.dataclass
class SolveResult:  # fastl1.hpp:61-71
    x: np.ndarray
    converged: bool
    final_gap: float
    iterations: int
    total_flops: int
    trace: np.ndarray  # structured array, TRACE_DTYPE
    switches: np.ndarray  # SWITCH_DTYPE
    final_active: np.ndarray
    gap_warning: bool
    device_ms: float = 0.0
    setup_ms: float = 0.0
    kernel_launches: int = 0
    power_iterations: int = 0
    profile: Optional[np.ndarray] = None  # product library only: see fl1_result_profile
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    batch_device_ms: float = 0.0  # batched calls: device time of the whole batch


def _collect_result(lib: Library, h) -> SolveResult:
    info = _abi.ResultInfoC()
    lib.check(lib.result_info_get(h, C.byref(info)))
    x = np.empty(info.k)
    lib.check(lib.result_x(h, _dptr(x)))
    trace = np.zeros(info.n_trace, dtype=TRACE_DTYPE)
    if info.n_trace:
        lib.check(lib.result_trace(h, trace.ctypes.data_as(C.POINTER(_abi.TraceRowC))))
    sws = np.zeros(info.n_switches, dtype=SWITCH_DTYPE)
    if info.n_switches:
        lib.check(lib.result_switches(h, sws.ctypes.data_as(C.POINTER(_abi.SwitchEventC))))
    fa = np.empty(info.n_final_active, dtype=np.int32)
    if info.n_final_active:
        lib.check(lib.result_final_active(h, fa.ctypes.data_as(C.POINTER(C.c_int32))))
    prof = None
    if hasattr(lib, "result_profile"):
        prof = np.zeros(14)
        lib.check(lib.result_profile(h, _dptr(prof)))
    elif hasattr(lib, "result_power_bytes"):  # the oracle reports its power-iteration bytes only
        prof = np.zeros(14)
        pb = C.c_double()
        lib.check(lib.result_power_bytes(h, C.byref(pb)))
        prof[7] = pb.value
    return SolveResult(profile=prof, x=x, converged=bool(info.converged), final_gap=info.final_gap, iterations=int(info.iterations),
                       total_flops=int(info.total_flops), trace=trace, switches=sws, final_active=fa,
                       gap_warning=bool(info.gap_warning), device_ms=info.device_ms, setup_ms=info.setup_ms,
                       kernel_launches=int(info.kernel_launches), power_iterations=int(info.power_iterations),
                       h2d_bytes=int(info.h2d_bytes), d2h_bytes=int(info.d2h_bytes),
                       batch_device_ms=float(info.batch_device_ms))


def _run_options_c(opts: RunOptions, keep: list) -> _abi.RunOptionsC:
    o = _abi.RunOptionsC()
    o.solver = opts.solver
    o.rule = opts.rule
    o.variant = opts.variant
    if opts.full_lipschitz is not None:
        fl = _vec(opts.full_lipschitz)
        keep.append(fl)
        o.full_lipschitz = _dptr(fl)
        o.n_full_lipschitz = fl.size
    o.collect_trace = 1 if opts.collect_trace else 0
    if opts.exact_gram is not None:
        keep.append(opts.exact_gram)
        o.exact_gram = opts.exact_gram._h
    if opts.observer is not None:
        user = opts.observer

        def _cb(ev_p, _u):
            ev = ev_p.contents
            n = ev.n
            user(ScreeningEvent(
                iter=int(ev.iter), dict_index=int(ev.dict_index),
                center=np.ctypeslib.as_array(ev.center, (n,)).copy(), radius=float(ev.radius),
                theta_prime=np.ctypeslib.as_array(ev.theta_prime, (n,)).copy(),
                theta_tilde=np.ctypeslib.as_array(ev.theta_tilde, (n,)).copy(),
                scale_prime=float(ev.scale_prime), scale_tilde=float(ev.scale_tilde),
                active_before=np.ctypeslib.as_array(ev.active_before, (ev.n_active_before,)).copy()
                if ev.n_active_before else np.zeros(0, np.int32),
                kept=np.ctypeslib.as_array(ev.kept, (ev.n_kept,)).copy() if ev.n_kept else np.zeros(0, np.int32)))

        cb = _abi.OBSERVER_FN(_cb)
        keep.append(cb)
        o.observer = cb
    if opts.x_init is not None:
        xi = _vec(opts.x_init)
        keep.append(xi)
        o.x_init = _dptr(xi)
    return o


def run_lasso(seq: ApproxSequence, y, lam: float, cfg: SwitchConfig, opts: RunOptions) -> SolveResult:
    """run_lasso (fastl1.cpp:753-758) through the C-ABI."""
    lib = seq.backend.lib
    yv = _vec(y)
    if yv.size != seq.exact().op.rows():
        raise InvalidArgument("y has wrong length")
    keep: list = []
    o = _run_options_c(opts, keep)
    if opts.x_init is not None and np.asarray(opts.x_init).size != seq.exact().op.cols():
        raise InvalidArgument("x_init has wrong length")
    c = cfg.c()
    h = C.c_void_p()
    lib.check(lib.solve(seq._h, _dptr(yv), float(lam), C.byref(c), C.byref(o), C.byref(h)))
    try:
        return _collect_result(lib, h)
    finally:
        lib.result_free(h)


def run_lasso_device(seq: ApproxSequence, y_dev_ptr: int, lam: float, cfg: SwitchConfig,
                     opts: RunOptions) -> SolveResult:
    """Same as run_lasso with y already resident in HBM (product library only)."""
    lib = seq.backend.lib
    keep: list = []
    o = _run_options_c(opts, keep)
    c = cfg.c()
    h = C.c_void_p()
    lib.check(lib.solve_device(seq._h, C.c_void_p(y_dev_ptr), float(lam), C.byref(c), C.byref(o), C.byref(h)))
    try:
        return _collect_result(lib, h)
    finally:
        lib.result_free(h)


def run_lasso_batched(seq: ApproxSequence, Y, lambdas, cfg: SwitchConfig, opts: RunOptions,
                      concurrency: int = 0, y_dev_ptr: Optional[int] = None) -> list:
    """B independent run_lasso solves (columns of Y, N x B) on the GPU at once
    (BASELINE config 5); product library only. With y_dev_ptr, Y (N x B column-major,
    leading dimension N) is already in HBM and `Y` only gives the shape."""
    lib = seq.backend.lib
    if y_dev_ptr is None:
        Ym = np.asfortranarray(np.asarray(Y, dtype=np.float64))
        if Ym.ndim == 1:
            Ym = Ym.reshape(-1, 1, order="F")
        n, B = Ym.shape
    else:
        n, B = Y
    if n != seq.exact().op.rows():
        raise InvalidArgument("y has wrong length")
    lam = _vec(lambdas, B, "lambdas")
    keep: list = []
    o = _run_options_c(opts, keep)
    c = cfg.c()
    hs = (C.c_void_p * max(B, 1))()
    if y_dev_ptr is None:
        lib.check(lib.solve_batched(seq._h, _dptr(Ym), n, _dptr(lam), B, C.byref(c), C.byref(o), concurrency, hs))
    else:
        lib.check(lib.solve_batched_device(seq._h, C.c_void_p(y_dev_ptr), n, _dptr(lam), B, C.byref(c), C.byref(o),
                                           concurrency, hs))
    try:
        return _collect_results(lib, hs, B)
    finally:
        for b in range(B):
            lib.result_free(hs[b])


def _info_columns(infos) -> dict:
    """Field -> numpy column of a ctypes array of fl1_result_info (no per-struct attribute access)."""
    arr = np.ctypeslib.as_array(infos)
    return {f: arr[f] for f in arr.dtype.names}


def _collect_results(lib: Library, hs, B: int) -> list:
    """All results of a batched call through the bulk accessors (4 library calls)."""
    if B == 0:
        return []
    infos = (_abi.ResultInfoC * B)()
    k = None
    lib.check(lib.results_collect(hs, B, infos, None, None))
    k = infos[0].k
    xs = np.empty((B, k))
    profs = np.zeros((B, 14))
    lib.check(lib.results_collect(hs, B, infos, _dptr(xs), _dptr(profs)))
    cols = {f: v.tolist() for f, v in _info_columns(infos).items()}  # one pass over the structs
    nt, ns, na = cols["n_trace"], cols["n_switches"], cols["n_final_active"]
    traces = np.zeros(max(sum(nt), 1), dtype=TRACE_DTYPE)
    sws = np.zeros(max(sum(ns), 1), dtype=SWITCH_DTYPE)
    fas = np.empty(max(sum(na), 1), dtype=np.int32)
    lib.check(lib.results_tables(hs, B, traces.ctypes.data_as(C.POINTER(_abi.TraceRowC)),
                                 sws.ctypes.data_as(C.POINTER(_abi.SwitchEventC)),
                                 fas.ctypes.data_as(C.POINTER(C.c_int32))))
    out = []
    ot = os_ = oa = 0
    for b in range(B):
        out.append(SolveResult(profile=profs[b], x=xs[b], converged=bool(cols["converged"][b]),
                               final_gap=cols["final_gap"][b], iterations=cols["iterations"][b],
                               total_flops=cols["total_flops"][b], trace=traces[ot:ot + nt[b]],
                               switches=sws[os_:os_ + ns[b]], final_active=fas[oa:oa + na[b]],
                               gap_warning=bool(cols["gap_warning"][b]), device_ms=cols["device_ms"][b],
                               setup_ms=cols["setup_ms"][b], kernel_launches=cols["kernel_launches"][b],
                               power_iterations=cols["power_iterations"][b], h2d_bytes=cols["h2d_bytes"][b],
                               d2h_bytes=cols["d2h_bytes"][b], batch_device_ms=cols["batch_device_ms"][b]))
        ot += nt[b]
        os_ += ns[b]
        oa += na[b]
    return out


def fastl1_solve(seq, y, lam, cfg, solver=SOLVER_FISTA, rule=RULE_GAP) -> SolveResult:  # fastl1.hpp:104-111
    return run_lasso(seq, y, lam, cfg, RunOptions(solver=solver, rule=rule, variant=VARIANT_MULTI_DICT))


def lambda_max(op: LinearOp, y) -> float:  # screening.cpp:9-11
    lib = op.backend.lib
    yv = _vec(y, op.rows(), "y")
    out = C.c_double()
    lib.check(lib.lambda_max(op._h, _dptr(yv), C.byref(out)))
    return out.value


def lipschitz_bound(op: LinearOp) -> float:  # solver.cpp:108-114
    lib = op.backend.lib
    out = C.c_double()
    lib.check(lib.lipschitz_bound(op._h, C.byref(out)))
    return out.value


def screen_precomputed(abs_dots, eps, exact_norms, approx_norms, center_norm, radius, backend=None):
    """screen_precomputed (screening.cpp:136-150) -> (kept positions, lookahead count)."""
    b = backend or default_backend()
    d = _vec(abs_dots)
    n = d.size
    e, en, an = _vec(eps, n), _vec(exact_norms, n), _vec(approx_norms, n)
    kept = np.empty(max(n, 1), dtype=np.int32)
    nk, la = C.c_int64(), C.c_int64()
    b.lib.check(b.lib.screen_precomputed(b.ctx, n, _dptr(d), _dptr(e), _dptr(en), _dptr(an), float(center_norm),
                                         float(radius), kept.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(nk),
                                         C.byref(la)))
    return kept[: nk.value].copy(), int(la.value)


class _Scalars:
    """Scalar formulas of the path, bound to one library."""

    def __init__(self, lib: Library):
        self.lib = lib

    def soft_threshold(self, z, u):
        return self.lib.soft_threshold(z, u)

    def gap_ratio(self, gt, gp):
        return self.lib.gap_ratio(gt, gp)

    def switch_dictionary(self, i, last, gamma, gthr, lookahead, rc, total):
        return self.lib.switch_dictionary(i, last, gamma, gthr, lookahead, rc, total)

    def flops_plain(self, k, n, nnz):
        return int(self.lib.flops_plain(k, n, nnz))

    def flops_screened(self, a, n, nnz):
        return int(self.lib.flops_screened(a, n, nnz))

    def flops_stable(self, mv, n, a, nnz):
        return int(self.lib.flops_stable(mv, n, a, nnz))

    def stable_gap_delta(self, rn, e, x1):
        return self.lib.stable_gap_delta(rn, e, x1)

    def sphere_test(self, d, an, r):
        return self.lib.sphere_test(d, an, r)

    def stable_zone_test(self, d, eps, cn, en, r):
        return self.lib.stable_zone_test(d, eps, cn, en, r)

    def stable_ball_test(self, d, eps, cn, an, r):
        return self.lib.stable_ball_test(d, eps, cn, an, r)


def recompute_flops(trace: np.ndarray, seq: ApproxSequence, variant: int, n: int, k: int):
    """recompute_flops (fastl1.cpp:51-81) -> (total, rows_match)."""
    lib = seq.backend.lib
    tr = np.ascontiguousarray(trace, dtype=TRACE_DTYPE)
    rm = C.c_int32()
    tot = lib.recompute_flops(tr.ctypes.data_as(C.POINTER(_abi.TraceRowC)), tr.size, seq._h, variant, n, k,
                              C.byref(rm))
    return int(tot), bool(rm.value)


def scalars(backend: Optional[Backend] = None) -> _Scalars:
    return _Scalars((backend or default_backend()).lib)
