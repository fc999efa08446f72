"""Shared fixtures. Markers: `gpu` needs a B200 (run on the GPU box)."""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
for _p in (str(ROOT), str(ROOT / "tests")):
    if _p not in sys.path:
        sys.path.insert(0, _p)

ORACLE_LIB = ROOT / "oracle" / "_build" / "libfl1oracle.so"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running test")


def _ensure_oracle():
    if not ORACLE_LIB.exists() or ORACLE_LIB.stat().st_mtime < (ROOT / "oracle" / "fl1_oracle.cpp").stat().st_mtime:
        subprocess.run(["make", "-C", str(ROOT / "oracle")], check=True, capture_output=True)
    return ORACLE_LIB


@pytest.fixture(scope="session")
def oracle():
    """The CPU oracle (test infrastructure) behind the same Python API."""
    from paper_1812_06635_b200 import _abi
    from paper_1812_06635_b200.fastl1 import Backend

    lib = _abi.Library(_ensure_oracle(), "orc_", extra=_abi.ORACLE_ONLY)
    return Backend(lib)


@pytest.fixture(scope="session")
def cuda():
    """The product: libfl1cuda.so on cuda:0. Fails loudly if not built."""
    from paper_1812_06635_b200.fastl1 import default_backend

    return default_backend()


@pytest.fixture(scope="session")
def refgen(oracle):
    from _refgen import RefGen

    return RefGen(oracle)


BACKENDS = ["oracle", pytest.param("cuda", marks=pytest.mark.gpu)]


@pytest.fixture(params=BACKENDS)
def backend(request, oracle):
    """Runs a test on the oracle (CPU suite) and on libfl1cuda.so (-m gpu)."""
    if request.param == "oracle":
        return oracle
    from paper_1812_06635_b200.fastl1 import default_backend

    return default_backend()


def pytest_sessionfinish(session, exitstatus):
    """FL1_PARITY_OUT=path: write the achieved GPU-vs-oracle discrepancies (tests/_parity.py)."""
    import os

    out = os.environ.get("FL1_PARITY_OUT")
    if out:
        import _parity

        _parity.write_records(out)
