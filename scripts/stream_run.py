#!/usr/bin/env python
"""BASELINE.json configs[4] (C5): streaming ingest with adaptive refresh, d=96.

Train the coarse partition on the first 1M vectors (GPU k-means, L=4096),
build the index from them, then add 9 shuffled i.i.d. 1M batches. After
batches 3 and 6, refresh the partition (RefreshPolicy defaults, seed 0;
keep_raw=False so the source is the decoded index, refresh.py:164-169). After
every batch: a 10k-query search (k=10, n_p=32) timed with CUDA events, and
recall@10 against the exact top-10 of the cumulative normalised database
(GPU f64 brute force). Writes one JSON file.

  python scripts/stream_run.py [--batches 9] [--batch 1000000] --out profiles/c5_r1.json
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=9)
    ap.add_argument("--batch", type=int, default=1_000_000)
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--refresh-after", default="3,6")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch

    from paper_2605_17415_b200 import _lib
    from paper_2605_17415_b200.evaluation import exact_topk, recall_at_k
    from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex
    from paper_2605_17415_b200.partition import CoarsePartition, train_partition
    from paper_2605_17415_b200.quantizer import design_quantizer
    from paper_2605_17415_b200.refresh import RefreshPolicy, refresh
    from paper_2605_17415_b200.rotation import generate_rotation
    from paper_2605_17415_b200.workloads import make_workload, mixture

    w = make_workload("c5")
    B = args.batch
    total = B * (args.batches + 1)
    dev = torch.device("cuda", 0)
    L = _lib.lib()
    t0 = time.time()
    x_all, means = mixture(total, w.d, w.components, w.sigma, w.base_seed)
    rng = np.random.default_rng(w.base_seed + 5)
    perm = rng.permutation(total)  # shuffled i.i.d. batches
    x_all = x_all[perm]
    queries, _ = mixture(args.nq, w.d, w.components, w.sigma, w.query_seed, means=means)
    gen_s = time.time() - t0

    first = x_all[:B].astype(np.float64)
    first /= np.linalg.norm(first, axis=1)[:, None]
    t0 = time.time()
    cent = train_partition(first, w.n_lists, seed=42, max_iters=w.kmeans_iters,
                           device="cuda").centroids
    km_s = time.time() - t0
    del first
    cfg = IndexConfig(dim=w.d, bits=w.bits, n_lists=w.n_lists)  # keep_raw=False
    idx = IvfTqIndex(cfg, design_quantizer(w.bits, w.d), generate_rotation(w.d, 42),
                     CoarsePartition(w.n_lists, w.d, cent), device=dev)
    pinned = torch.from_numpy(x_all).pin_memory()
    qn = queries.astype(np.float64)
    qn /= np.linalg.norm(qn, axis=1)[:, None]
    Qd = torch.from_numpy(queries).to(dev)
    xn_dev = torch.empty((total, w.d), dtype=torch.float64, device=dev)
    bad = torch.empty(1, dtype=torch.int64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    refresh_at = {int(v) for v in args.refresh_after.split(",") if v}
    n_p = 32
    log = []
    for b in range(args.batches + 1):
        s, e = b * B, (b + 1) * B
        torch.cuda.synchronize()
        e0.record()
        idx.add_batch(pinned[s:e])
        e1.record()
        torch.cuda.synchronize()
        add_s = e0.elapsed_time(e1) / 1000
        xc = pinned[s:e].to(dev)
        _lib.check(L.ivftq_normalize_rows(xc.data_ptr(), _lib.IVFTQ_F32, e - s, w.d,
                                          xn_dev[s:e].data_ptr(), bad.data_ptr(),
                                          _lib.stream_ptr()), "normalize")
        ent = {"batch": b, "n": e, "adds_per_sec": B / add_s}
        if b in refresh_at:
            t1 = time.time()
            rep = refresh(idx, RefreshPolicy(seed=0), kmeans_device="cuda")
            torch.cuda.synchronize()
            ent["refresh"] = {"seconds": time.time() - t1, "sample_size": rep.sample_size,
                              "used_raw": rep.used_raw,
                              "mean_ip_before": rep.mean_assigned_ip_before,
                              "mean_ip_after": rep.mean_assigned_ip_after,
                              "centroid_displacement_mean": rep.centroid_displacement_mean}
        idx.search_batch(Qd, 10, n_p, return_device=True)
        ts = []
        for _ in range(5):
            flush.fill_(1)
            torch.cuda.synchronize()
            e0.record()
            ids, _ = idx.search_batch(Qd, 10, n_p, return_device=True)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1000)
        truth = exact_topk(xn_dev[:e], qn, 10).ids
        ent["qps"] = args.nq / float(np.median(ts))
        ent["recall_at_10"] = recall_at_k(ids.cpu().numpy(), truth, 10)
        log.append(ent)
        print(json.dumps(ent), flush=True)
    rep = {"workload": "c5", "d": w.d, "n_lists": w.n_lists, "bits": w.bits, "batch": B,
           "batches_after_first": args.batches, "nprobe": n_p, "k": 10, "nq": args.nq,
           "keep_raw": False, "refresh_after": sorted(refresh_at),
           "seeds": {"base": w.base_seed, "query": w.query_seed, "shuffle": w.base_seed + 5},
           "timings": {"generate_s": gen_s, "kmeans_s": km_s}, "batches": log}
    print(json.dumps(rep), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main()
