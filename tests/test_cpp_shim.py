"""The C++ drop-in header (include/fl1/fastl1.hpp) compiles against the C-ABI
(CPU) and runs the reference's call pattern on the GPU (-m gpu)."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_1812_06635_b200"
SRC = ROOT / "tests" / "cpp" / "shim_test.cpp"


def _compile(out: Path) -> None:
    if not (PKG / "libfl1cuda.so").exists():
        from paper_1812_06635_b200 import build

        build.build()
    cmd = ["/usr/bin/g++", "-std=c++17", "-O2", "-Wall", "-Wextra", f"-I{ROOT / 'include'}", str(SRC), "-o", str(out),
           f"-L{PKG}", "-lfl1cuda", f"-Wl,-rpath,{PKG}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_shim_compiles(tmp_path):
    _compile(tmp_path / "shim_test")


@pytest.mark.gpu
def test_shim_runs_on_gpu(tmp_path):
    exe = tmp_path / "shim_test"
    _compile(exe)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "shim ok" in r.stdout
