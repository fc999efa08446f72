"""ctypes binding of the C-ABI in include/fl1cuda.h.

`Library(path, prefix)` binds one shared object. The product is
libfl1cuda.so with prefix ``fl1_``; the test oracle exports the same entry
points with prefix ``orc_`` (oracle/fl1_oracle.h) and is loaded only by the
tests / bench baseline, never by the product path.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

FL1_OK, FL1_EINVAL, FL1_ECUDA, FL1_ENOMEM, FL1_EUNSUPPORTED, FL1_ERUNTIME = range(6)


class SwitchConfigC(C.Structure):
    _fields_ = [
        ("gamma_threshold", C.c_double),
        ("screening_interval", C.c_int32),
        ("tolerance", C.c_double),
        ("max_iterations", C.c_uint64),
        ("precompute_aty", C.c_int32),
        ("rel_tolerance", C.c_double),
    ]


class ScreenEventC(C.Structure):
    _fields_ = [
        ("iter", C.c_uint64),
        ("dict_index", C.c_int32),
        ("n", C.c_int64),
        ("center", C.POINTER(C.c_double)),
        ("radius", C.c_double),
        ("theta_prime", C.POINTER(C.c_double)),
        ("theta_tilde", C.POINTER(C.c_double)),
        ("scale_prime", C.c_double),
        ("scale_tilde", C.c_double),
        ("n_active_before", C.c_int64),
        ("active_before", C.POINTER(C.c_int32)),
        ("n_kept", C.c_int64),
        ("kept", C.POINTER(C.c_int32)),
    ]


OBSERVER_FN = C.CFUNCTYPE(None, C.POINTER(ScreenEventC), C.c_void_p)


class RunOptionsC(C.Structure):
    _fields_ = [
        ("solver", C.c_int32),
        ("rule", C.c_int32),
        ("variant", C.c_int32),
        ("full_lipschitz", C.POINTER(C.c_double)),
        ("n_full_lipschitz", C.c_int32),
        ("collect_trace", C.c_int32),
        ("observer", OBSERVER_FN),
        ("observer_user", C.c_void_p),
        ("x_init", C.POINTER(C.c_double)),
        ("exact_gram", C.c_void_p),
    ]


class TraceRowC(C.Structure):
    _fields_ = [
        ("iter", C.c_uint64),
        ("dict_index", C.c_int32),
        ("active_size", C.c_int32),
        ("gap", C.c_double),
        ("gamma", C.c_double),
        ("flops_cum", C.c_uint64),
        ("wall_ms", C.c_double),
        ("x_nnz", C.c_int32),
        ("pad_", C.c_int32),
    ]


class SwitchEventC(C.Structure):
    _fields_ = [
        ("iter", C.c_uint64),
        ("from_", C.c_int32),
        ("to", C.c_int32),
        ("speed", C.c_int32),
        ("pad_", C.c_int32),
    ]


class ResultInfoC(C.Structure):
    _fields_ = [
        ("k", C.c_int64),
        ("converged", C.c_int32),
        ("gap_warning", C.c_int32),
        ("final_gap", C.c_double),
        ("iterations", C.c_uint64),
        ("total_flops", C.c_uint64),
        ("n_trace", C.c_int64),
        ("n_switches", C.c_int64),
        ("n_final_active", C.c_int64),
        ("device_ms", C.c_double),
        ("setup_ms", C.c_double),
        ("kernel_launches", C.c_int64),
        ("power_iterations", C.c_int64),
        ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64),
        ("batch_device_ms", C.c_double),
    ]


_P = C.c_void_p
_PD = C.POINTER(C.c_double)
_PI32 = C.POINTER(C.c_int32)
_PI64 = C.POINTER(C.c_int64)
_PP = C.POINTER(C.c_void_p)

# name -> (restype, argtypes); identical for both prefixes
SIGNATURES = {
    "last_error": (C.c_char_p, []),
    "version": (C.c_char_p, []),
    "ctx_create": (C.c_int, [C.c_int, _PP]),
    "ctx_destroy": (C.c_int, [_P]),
    "dict_dense": (C.c_int, [_P, _PD, C.c_int64, C.c_int64, _PP]),
    "dict_sukro": (C.c_int, [_P, C.c_int32, C.c_int64, C.c_int64, C.POINTER(_PD), C.POINTER(_PD), _PD, _PP]),
    "dict_destroy": (C.c_int, [_P]),
    "dict_shape": (C.c_int, [_P, _PI64, _PI64]),
    "dict_is_dense": (C.c_int, [_P]),
    "dict_matvec_flops": (C.c_uint64, [_P]),
    "dict_atom_norms": (C.c_int, [_P, _PD]),
    "dict_apply": (C.c_int, [_P, _PD, _PD]),
    "dict_apply_adjoint": (C.c_int, [_P, _PD, _PD]),
    "dict_column": (C.c_int, [_P, C.c_int64, _PD]),
    "approx_create": (C.c_int, [_P, _PD, C.c_double, C.c_double, _PD, _PD, _PP]),
    "approx_exact": (C.c_int, [_P, _PP]),
    "approx_destroy": (C.c_int, [_P]),
    "seq_create": (C.c_int, [_PP, C.c_int32, _PP]),
    "seq_destroy": (C.c_int, [_P]),
    "solve": (C.c_int, [_P, _PD, C.c_double, C.POINTER(SwitchConfigC), C.POINTER(RunOptionsC), _PP]),
    "result_info_get": (C.c_int, [_P, C.POINTER(ResultInfoC)]),
    "result_x": (C.c_int, [_P, _PD]),
    "result_trace": (C.c_int, [_P, C.POINTER(TraceRowC)]),
    "result_switches": (C.c_int, [_P, C.POINTER(SwitchEventC)]),
    "result_final_active": (C.c_int, [_P, _PI32]),
    "result_free": (None, [_P]),
    "lambda_max": (C.c_int, [_P, _PD, _PD]),
    "lipschitz_bound": (C.c_int, [_P, _PD]),
    "screen_precomputed": (C.c_int, [_P, C.c_int64, _PD, _PD, _PD, _PD, C.c_double, C.c_double, _PI32, _PI64, _PI64]),
    "soft_threshold": (C.c_double, [C.c_double, C.c_double]),
    "gap_ratio": (C.c_double, [C.c_double, C.c_double]),
    "switch_dictionary": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int64, C.c_double, C.c_int64]),
    "flops_plain": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64]),
    "flops_screened": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64]),
    "flops_stable": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64]),
    "recompute_flops": (C.c_uint64, [C.POINTER(TraceRowC), C.c_int64, _P, C.c_int32, C.c_int64, C.c_int64, _PI32]),
    "stable_gap_delta": (C.c_double, [C.c_double, C.c_double, C.c_double]),
    "sphere_test": (C.c_double, [C.c_double, C.c_double, C.c_double]),
    "stable_zone_test": (C.c_double, [C.c_double, C.c_double, C.c_double, C.c_double, C.c_double]),
    "stable_ball_test": (C.c_double, [C.c_double, C.c_double, C.c_double, C.c_double, C.c_double]),
    "gram_create": (C.c_int, [_P, _PP]),
}

# product-only entry points
PRODUCT_ONLY = {
    "ctx_info": (C.c_int, [_P, _PI32, _PI64, _PI64]),
    "dict_dense_device": (C.c_int, [_P, C.c_void_p, C.c_int64, C.c_int64, _PP]),
    "result_profile": (C.c_int, [_P, _PD]),
    "solve_batched": (C.c_int, [_P, _PD, C.c_int64, _PD, C.c_int32, C.POINTER(SwitchConfigC), C.POINTER(RunOptionsC),
                                C.c_int32, _PP]),
    "solve_batched_device": (C.c_int, [_P, C.c_void_p, C.c_int64, _PD, C.c_int32, C.POINTER(SwitchConfigC),
                                       C.POINTER(RunOptionsC), C.c_int32, _PP]),
    "solve_device": (C.c_int, [_P, C.c_void_p, C.c_double, C.POINTER(SwitchConfigC), C.POINTER(RunOptionsC), _PP]),
    "rng_normals": (C.c_int, [C.c_uint64, C.c_int64, _PD]),
    "results_collect": (C.c_int, [_PP, C.c_int32, C.POINTER(ResultInfoC), _PD, _PD]),
    "results_tables": (C.c_int, [_PP, C.c_int32, C.POINTER(TraceRowC), C.POINTER(SwitchEventC), _PI32]),
    "draw_signal": (C.c_int, [_P, C.c_double, C.c_uint64, C.c_int32, _PD, _PD]),
    "build_sukro_sequence": (C.c_int, [_P, _PI32, C.c_int32, _PD, _PD, _PD, _PD, _PD, _PD]),
}

# oracle-only entry points (test infrastructure)
ORACLE_ONLY = {
    "set_threads": (None, [C.c_int]),
    "result_power_bytes": (C.c_int, [_P, _PD]),
    "get_threads": (C.c_int, []),
    "dict_to_dense": (C.c_int, [_P, _PD]),
    "ista_step": (C.c_int, [_P, _PD, C.c_double, C.c_double, _PD, _PD, _PD, _PD]),
    "fista_step": (C.c_int, [_P, _PD, C.c_double, C.c_double, _PD, _PD, _PD, _PI32, _PD, _PD, _PD]),
    "primal_value": (C.c_double, [_P, _PD, C.c_double, _PD]),
    "dual_value": (C.c_double, [C.c_int64, _PD, C.c_double, _PD]),
    "duality_gap": (C.c_double, [_P, _PD, C.c_double, _PD, _PD, _PI32]),
    "stable_lambda_max": (C.c_int, [_P, _PD, _PD]),
    "dual_scale": (C.c_int, [_P, _PD, _PD]),
    "stable_dual_scale": (C.c_int, [_P, _PD, _PD]),
    "dual_point_dynamic": (C.c_int, [C.c_int64, C.c_int64, _PD, _PD, _PD, _PD, C.c_double, _P, _PD, _PD, _PD, _PD]),
    "build_sphere": (C.c_int, [C.c_int32, C.c_int64, _PD, C.c_double, C.c_double, C.c_double, _PD, C.c_double, C.c_double, _PD, _PD]),
    "screen": (C.c_int, [_PI32, C.c_int64, _PD, C.c_double, _P, C.c_int32, _PI32, _PI64]),
    "gen_normals": (None, [C.c_uint64, C.c_int64, _PD]),
    "gen_support": (None, [C.c_uint64, C.c_int64, C.c_int32, _PI64, _PD]),
}

ERRORS = {
    FL1_EINVAL: ValueError,
    FL1_ECUDA: RuntimeError,
    FL1_ENOMEM: MemoryError,
    FL1_EUNSUPPORTED: NotImplementedError,
    FL1_ERUNTIME: RuntimeError,
}


class InvalidArgument(ValueError):
    """Image of the reference's std::invalid_argument."""


class Library:
    """One loaded implementation of the C-ABI."""

    def __init__(self, path: str | Path, prefix: str, extra: dict | None = None):
        self.path = str(path)
        self.prefix = prefix
        self.lib = C.CDLL(self.path)
        sigs = dict(SIGNATURES)
        if extra:
            sigs.update(extra)
        for name, (res, args) in sigs.items():
            fn = getattr(self.lib, prefix + name)
            fn.restype = res
            fn.argtypes = args
            setattr(self, name, fn)

    def check(self, status: int) -> None:
        if status == FL1_OK:
            return
        msg = self.last_error().decode(errors="replace")
        if status == FL1_EINVAL:
            raise InvalidArgument(msg)
        raise ERRORS.get(status, RuntimeError)(f"{self.prefix}: {msg}")

    def exports(self) -> list[str]:
        return [self.prefix + n for n in SIGNATURES]
