"""N>1 host plumbing of the replica layout on CPU (gloo, world size 2)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_17415_b200.replicas import (job_throughput, max_over_ranks,
                                                    share_centroids, world as wd)

        assert wd() == (rank, world)
        cent = np.arange(12, dtype=np.float32).reshape(3, 4) if rank == 0 else None
        got = share_centroids(cent, (3, 4), "cpu")
        ms = max_over_ranks(1.0 + rank, "cpu")
        thr = job_throughput(1000, ms)
        out.put((rank, got.tolist(), ms, thr))
    finally:
        dist.destroy_process_group()


def test_replica_collectives_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.arange(12, dtype=np.float32).reshape(3, 4).tolist()
    for rank, got, ms, thr in res:
        assert got == want                # every replica encodes with rank 0's centroids
        assert ms == 2.0                  # slowest rank's time
        assert thr == pytest.approx(2 * 1000 / 0.002)  # whole-job units over that time


def test_single_process_defaults():
    from paper_2605_17415_b200.replicas import job_throughput, max_over_ranks, world

    assert world() == (0, 1)
    assert max_over_ranks(3.5, "cpu") == 3.5
    assert job_throughput(10, 2.0) == pytest.approx(5000.0)
