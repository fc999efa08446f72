"""Host-side cost of the batched entry point (c5): library call vs result collection vs free."""
import os, sys, time
import ctypes as C
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np
import bench
from paper_1812_06635_b200 import fastl1 as F, _abi

a, Y, lams = bench.make_c5(5)
n, k = a.shape
B = Y.shape[1]
d = F.DenseDictionary(a)
L = F.lipschitz_bound(d)
seq = F.ApproxSequence([F.make_exact_approx(d)])
cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
opts = F.RunOptions(variant=F.VARIANT_SCREENED, full_lipschitz=[L])
lib = seq.backend.lib
Ym = np.asfortranarray(Y)
lam = np.ascontiguousarray(lams)
for rep in range(4):
    keep = []
    o = F._run_options_c(opts, keep)
    c = cfg.c()
    hs = (C.c_void_p * B)()
    t0 = time.perf_counter()
    lib.check(lib.solve_batched(seq._h, F._dptr(Ym), n, F._dptr(lam), B, C.byref(c), C.byref(o), 0, hs))
    t1 = time.perf_counter()
    rs = F._collect_results(lib, hs, B)
    t2 = time.perf_counter()
    for b in range(B):
        lib.result_free(hs[b])
    t3 = time.perf_counter()
    print(f"solve_batched {1e3*(t1-t0):.2f} ms (device {rs[0].batch_device_ms:.2f}, setup {rs[0].setup_ms:.2f}) "
          f"collect {1e3*(t2-t1):.2f} ms free {1e3*(t3-t2):.2f} ms")
