"""The C-ABI boundary (no GPU needed): libfl1cuda.so loads, exports every symbol
include/fl1cuda.h declares, its host-side scalar formulas match the reference
KATs, and it fails loudly (no CPU fallback) when no device is present.
"""
from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "fl1cuda.h"
LIB = ROOT / "paper_1812_06635_b200" / "libfl1cuda.so"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(fl1_[a-z0-9_]+)\s*\(", text)) - {"fl1_observer_fn"})


@pytest.fixture(scope="module")
def lib():
    if not LIB.exists():
        from paper_1812_06635_b200 import build

        build.build()
    return C.CDLL(str(LIB))


def test_every_declared_symbol_is_exported(lib):
    syms = declared_symbols()
    assert len(syms) > 40
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (fl1_[a-z0-9_]+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        getattr(lib, s)


def test_library_contains_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_oracle_exports_the_same_abi():
    from conftest import _ensure_oracle

    path = _ensure_oracle()
    out = subprocess.run(["nm", "-D", "--defined-only", str(path)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (orc_[a-z0-9_]+)", out))
    from paper_1812_06635_b200 import _abi

    for name in _abi.SIGNATURES:
        assert "orc_" + name in exported, name


def test_host_scalar_formulas_without_a_device():
    from paper_1812_06635_b200 import fastl1 as F

    s = F._Scalars(F.cuda_library())
    assert s.soft_threshold(-2.0, 0.5) == -1.5
    assert s.gap_ratio(0.2, 0.8) == pytest.approx(0.25)
    assert s.switch_dictionary(0, 4, 0.9, 0.2, 100, 0.15, 10000) == 4
    assert s.flops_plain(10000, 2500, 0) == 10000 * 2500 + 4 * 10000 + 2500
    assert s.stable_zone_test(0.5, 0.1, 2.0, 1.0, 0.3) == 0.5 + 0.2 + 0.3


def test_no_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_1812_06635_b200 import fastl1 as F

    lib = F.cuda_library()
    h = C.c_void_p()
    st = lib.ctx_create(0, C.byref(h))
    assert st != 0
    assert lib.last_error()


def test_python_api_mirrors_reference_names():
    from paper_1812_06635_b200 import fastl1 as F

    for name in ("DenseDictionary", "SukroDictionary", "ApproxDictionary", "ApproxSequence", "SwitchConfig",
                 "RunOptions", "SolveResult", "run_lasso", "fastl1_solve", "lambda_max", "lipschitz_bound",
                 "make_exact_approx", "recompute_flops", "screen_precomputed", "solver_from_string",
                 "rule_from_string"):
        assert hasattr(F, name), name
    cfg = F.SwitchConfig()
    assert (cfg.gamma_threshold, cfg.screening_interval, cfg.tolerance, cfg.max_iterations) == (0.5, 1, 1e-6, 1_000_000)
    with pytest.raises(F.InvalidArgument):
        F.solver_from_string("adam")
    assert F.rule_from_string("gap") == F.RULE_GAP
