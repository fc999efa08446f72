"""Build recipe for libfl1cuda.so (the C-ABI hot path) — nvcc, sm_100a only.

The library is built in-tree (paper_1812_06635_b200/libfl1cuda.so) so it
travels with the repository snapshot to the GPU box. No torch, no JIT cache.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libfl1cuda.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
HOST_CXX = "/usr/bin/g++"  # the image's $CXX wrapper lacks some specs; use the system compiler
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["engine.cu", "batched.cu", "setup.cu", "sukro_build.cu", "api.cpp"]


def _sources_newer(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines: dict | None = None, out: Path | None = None) -> Path:
    """Compile libfl1cuda.so; `defines`/`out` build tuning variants (FL1_THREADS, FL1_UNIT)."""
    lib = out or LIB
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "fl1cuda.h"]
    if not force and not _sources_newer(lib, deps):
        return lib
    objs = []
    build_dir = PKG / "_build" / (lib.stem if out else "main")
    build_dir.mkdir(parents=True, exist_ok=True)
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-ccbin", HOST_CXX, "-lineinfo"]
    common += [f"-D{k}={v}" for k, v in (defines or {}).items()]
    # engine.cu twice: the default engine and the instance with the single-read power steps (_fp entry points)
    for s, extra, tag in [(s, [], "") for s in SOURCES] + [("engine.cu", ["-DFL1_FUSED_VARIANT=1"], "_fp")]:
        obj = build_dir / (s + tag + ".o")
        cmd = [NVCC, *ARCH, *common, *extra, "-Xptxas", "-v", "-c", str(CSRC / s), "-o", str(obj)]
        if s.endswith(".cpp"):
            cmd = [NVCC, *common, "-x", "cu", *ARCH, "-c", str(CSRC / s), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {s}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(str(obj))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-ccbin", HOST_CXX, "-o", str(tmp), *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    tmp.replace(lib)
    return lib


if __name__ == "__main__":
    if "--timeline" in sys.argv:  # instrumented build: per-CTA phase timeline (FL1_TIMELINE_OUT=path)
        print(build(force=True, defines={"FL1_TIMELINE": 1}, out=PKG / "_build" / "libfl1cuda_timeline.so"))
    elif "--variants" in sys.argv:  # tuning sweep: libfl1cuda_t{threads}_u{unit}.so
        for t, u, rg in ((256, 512, 2), (256, 1024, 2), (256, 512, 3)):
            print(build(force=True, defines={"FL1_THREADS": t, "FL1_UNIT": u, "FL1_RING": rg},
                        out=PKG / "_build" / f"libfl1cuda_t{t}_u{u}_r{rg}.so"))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
