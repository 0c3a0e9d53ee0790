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


def test_bench_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` outside torchrun relaunches itself as two ranks over
    127.0.0.1; the reference arm (CPU oracle, rank 0 only) prints one line that
    carries the same n_gpus as the other arm would."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run(
        [sys.executable, str(root / "bench.py"), "--impl", "reference", "--gpus", "2", "--config",
         "c2", "--n", "20000", "--nq", "64", "--steps", "1", "--warmup", "0",
         "--ref-step-seconds", "0.2"],
        capture_output=True, text=True, timeout=300, env=env, cwd=str(root))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                      # rank 1 exits without printing
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
