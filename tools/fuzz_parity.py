"""Long randomised GPU-vs-oracle parity sweeps: python tools/fuzz_parity.py [cases] [seed] [dense|sukro] (tests/_fuzz.py)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import _fuzz  # noqa: E402

if __name__ == "__main__":
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    kind = sys.argv[3] if len(sys.argv) > 3 else "dense"
    run = _fuzz.sweep_sukro if kind == "sukro" else _fuzz.sweep
    fails = run(_fuzz.F.default_backend(), _fuzz.oracle_backend(), cases, seed)
    for f in fails:
        print(f)
    sys.exit(1 if fails else 0)
