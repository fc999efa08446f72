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
    import bench

    from paper_1812_06635_b200 import synthetic as syn

    inst = syn.dense_instance("c1", seed=1, n=40, k=80, nnz=4)  # bench.make_problem's seeding (offset 0)
    per, e2e, its = bench.reduce_over_ranks(dist, "cpu", 0.001 * (rank + 1), 0.002 * (rank + 1), 10.0 + rank)
    out[rank] = (per, e2e, its, float(inst.y[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_replica_reduction_world_size_2():
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn", join=True)
        r0, r1 = out[0], out[1]
    assert r0[:3] == r1[:3] == (0.002, 0.004, 21.0)
    assert r0[3] == r1[3]  # the same seeded instance on every replica
