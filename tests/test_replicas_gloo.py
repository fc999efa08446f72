"""N>1 path of bench.py (replicas only) on CPU with gloo, world size 2:
every rank builds the same seeded instance (identical work per replica), times are
max-reduced, iterations summed, and only rank 0 reports."""
from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import time

    import bench
    import numpy as np

    from paper_1812_06635_b200 import fastl1 as F, synthetic as syn

    # every replica solves the same seeded instance (bench.make_problem's seeding, offset 0) on
    # its own device; here the oracle backend stands in for the GPU (CPU test)
    b = bench._oracle_backend(1)
    inst = syn.dense_instance("c1", seed=1, n=60, k=200, nnz=6)
    d = F.DenseDictionary(inst.a, backend=b)
    seq = F.ApproxSequence([F.make_exact_approx(d)])
    cfg = F.SwitchConfig(screening_interval=10, max_iterations=5000, rel_tolerance=1e-6)
    t = time.perf_counter()
    r = F.run_lasso(seq, inst.y, inst.lam, cfg, F.RunOptions(variant=F.VARIANT_SCREENED))
    el = time.perf_counter() - t
    per, e2e, its = bench.reduce_over_ranks(dist, "cpu", el, 2 * el, float(r.iterations))
    # the replica reduction itself on known values: max of times, sum of iterations
    kp, ke, ki = bench.reduce_over_ranks(dist, "cpu", 0.001 * (rank + 1), 0.002 * (rank + 1), 10.0 + rank)
    out[rank] = dict(per=per, e2e=e2e, its=its, el=el, iters=r.iterations, x=np.asarray(r.x).tolist(),
                     conv=r.converged, known=(kp, ke, ki))
    dist.barrier()
    dist.destroy_process_group()


def test_replica_solves_world_size_2():
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn", join=True)
        r0, r1 = dict(out[0]), dict(out[1])
    assert r0["known"] == r1["known"] == (0.002, 0.004, 21.0)
    assert r0["conv"] and r1["conv"]
    assert r0["x"] == r1["x"] and r0["iters"] == r1["iters"]  # identical work on every replica
    assert r0["per"] == r1["per"] == max(r0["el"], r1["el"])  # max over ranks
    assert r0["its"] == r1["its"] == r0["iters"] + r1["iters"]  # summed
