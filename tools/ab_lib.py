"""Run bench.py against another build of libfl1cuda.so (e.g. the round-1 library) for a
same-box A/B: FL1_LIB=<path> python tools/ab_lib.py <bench args>. Entry points the older
build lacks are dropped from the binding table (the bench path does not use them)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1812_06635_b200 import _abi  # noqa: E402

for name in ("build_sukro_sequence",):
    _abi.PRODUCT_ONLY.pop(name, None)
import bench  # noqa: E402

sys.argv = ["bench.py"] + sys.argv[1:]
bench.main()
