#!/usr/bin/env python
"""Large-config run (BASELINE.json configs[2] C3 = 10M x 96, L=4096; configs[3]
C4 = 10M x 200) on one GPU: train, ingest, search sweep, recall, and parity
against the CPU oracle on bounded samples. Writes one JSON file.

  python scripts/scale_run.py --config c3 [--n N] [--bits B] --out profiles/c3_r1.json

Parity protocol (north_star bars, tests/helpers.py tolerances):
  * codes: a contiguous 100k-row window of the GPU-encoded index is re-encoded
    by the oracle (oracle/ivftq_oracle.encode_batch) from the same input rows;
    bins/signs/list ids/binary16 norms compared, flip fraction reported;
  * search: `--parity-queries` queries searched by the oracle over the
    GPU-encoded fields (bit-identical to the oracle's own encode on the
    checked window) at every n_p of the sweep: ids up to ties, scores within
    1e-4 relative, recall@10 difference.
The oracle is the checker only; every timed number is the GPU path.
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
sys.path.insert(0, str(ROOT / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--bits", type=int, default=None)
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--parity-queries", type=int, default=200)
    ap.add_argument("--parity-rows", type=int, default=100_000)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch

    from paper_2605_17415_b200 import _lib
    from paper_2605_17415_b200.evaluation import exact_topk, recall_at_k
    from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex
    from paper_2605_17415_b200.partition import CoarsePartition, train_partition
    from paper_2605_17415_b200.quantizer import design_quantizer
    from paper_2605_17415_b200.rotation import generate_rotation
    from paper_2605_17415_b200.workloads import make_workload

    over = {}
    if args.n:
        over["n"] = args.n
    if args.bits:
        over["bits"] = args.bits
    w = make_workload(args.config, **over)
    nq = args.nq or w.n_queries
    dev = torch.device("cuda", 0)
    rep = {"workload": w.name, "n": w.n, "d": w.d, "n_lists": w.n_lists, "bits": w.bits,
           "nq": nq, "k": 10, "seeds": {"base": w.base_seed, "query": w.query_seed},
           "kmeans_sample": w.kmeans_sample, "kmeans_iters": w.kmeans_iters}
    T = {}

    t0 = time.time()
    base = w.base()
    queries = w.queries(nq)
    T["generate_s"] = time.time() - t0

    # ---- partition: k-means on a seeded subsample, on the GPU ---------------
    t0 = time.time()
    m = min(w.kmeans_sample or w.n, w.n)
    rng = np.random.default_rng(w.base_seed + 17)
    sub = base[np.sort(rng.choice(w.n, size=m, replace=False))].astype(np.float64)
    sub /= np.linalg.norm(sub, axis=1)[:, None]
    cent = train_partition(sub, w.n_lists, seed=42, max_iters=w.kmeans_iters,
                           device="cuda").centroids
    del sub
    T["kmeans_s"] = time.time() - t0

    q = design_quantizer(w.bits, w.d)
    R = generate_rotation(w.d, 42)
    cfg = IndexConfig(dim=w.d, bits=w.bits, n_lists=w.n_lists)
    idx = IvfTqIndex(cfg, q, R, CoarsePartition(w.n_lists, w.d, cent), device=dev)

    # ---- ingest from pinned host rows -----------------------------------------
    chunk = 1_000_000
    pinned = torch.from_numpy(base).pin_memory()
    # warm-up on a throwaway index: lazy kernel loading and first-use
    # allocations stay out of the timed region
    warm = IvfTqIndex(cfg, q, R, CoarsePartition(w.n_lists, w.d, cent), device=dev)
    warm.add_batch(pinned[:300_000])
    del warm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    e0.record()
    for s in range(0, w.n, chunk):
        idx.add_batch(pinned[s:s + chunk])
    e1.record()
    torch.cuda.synchronize()
    rep["ingest"] = {"adds_per_sec_e2e": w.n / (e0.elapsed_time(e1) / 1000), "chunk": chunk,
                     "wall_s": time.time() - t0}
    sizes = idx._store.sizes
    rep["list_sizes"] = {"min": int(sizes.min()), "mean": float(sizes.mean()),
                         "max": int(sizes.max())}

    # ---- ground truth: f64 brute force on the GPU (reference tie rule) ---------
    t0 = time.time()
    L = _lib.lib()
    xn = torch.empty((w.n, w.d), dtype=torch.float64, device=dev)
    bad = torch.empty(1, dtype=torch.int64, device=dev)
    for s in range(0, w.n, chunk):
        e = min(w.n, s + chunk)
        xc = pinned[s:e].to(dev)
        _lib.check(L.ivftq_normalize_rows(xc.data_ptr(), _lib.IVFTQ_F32, e - s, w.d,
                                          xn[s:e].data_ptr(), bad.data_ptr(),
                                          _lib.stream_ptr()), "normalize")
    qn = queries.astype(np.float64)
    qn /= np.linalg.norm(qn, axis=1)[:, None]
    truth = exact_topk(xn, qn, 10).ids
    del xn
    torch.cuda.empty_cache()
    T["truth_s"] = time.time() - t0

    # ---- search sweep (device-resident queries, L2 flushed, CUDA events) ------
    Qd = torch.from_numpy(queries).to(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    code_b = -(-w.bits * w.d // 8) + -(-w.d // 8) + 2
    sweep = []
    results = {}
    for n_p in w.nprobe:
        idx.search_batch(Qd, 10, n_p, return_device=True)
        ts = []
        for _ in range(args.reps):
            flush.fill_(1)
            torch.cuda.synchronize()
            e0.record()
            ids, sc = idx.search_batch(Qd, 10, n_p, return_device=True)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1000)
        ids_h, sc_h = ids.cpu().numpy(), sc.cpu().numpy()
        results[n_p] = (ids_h, sc_h)
        t = float(np.median(ts))
        ent = {"nprobe": n_p, "qps": nq / t, "ms": t * 1000,
               "recall_at_10": recall_at_k(ids_h, truth, 10)}
        # scan-kernel time and the algorithmic bytes of the per-query code stream
        L.ivftq_set_kernel_timing(1)
        flush.fill_(1)
        idx.search_batch(Qd, 10, n_p, return_device=True)
        torch.cuda.synchronize()
        kms = L.ivftq_last_scan_kernel_ms()
        L.ivftq_set_kernel_timing(0)
        if kms > 0:
            ent["scan_kernel_ms"] = kms
        sweep.append(ent)
        print(json.dumps(ent), flush=True)
    rep["sweep"] = sweep
    rep["bytes_per_vector"] = code_b

    # ---- parity vs the oracle ---------------------------------------------------
    from oracle import ivftq_oracle as orc
    from helpers import compare_topk

    t0 = time.time()
    pr = min(args.parity_rows, w.n)
    off = int(np.random.default_rng(7).integers(0, w.n - pr + 1))
    b_o, s_o, l_o, n_o, _ = orc.encode_batch(base[off:off + pr], cent, R.matrix, q.boundaries,
                                             q.centroids)
    bins, signs = idx.bins, idx.signs
    flips = ((bins[off:off + pr] != b_o) | (signs[off:off + pr] != s_o)).mean()
    codes = {"rows": pr, "offset": off, "flip_fraction": float(flips),
             "list_ids_equal": bool(np.array_equal(idx.list_ids[off:off + pr], l_o)),
             "norms_equal": bool(np.array_equal(idx.norms[off:off + pr].view(np.uint16),
                                                n_o.view(np.uint16)))}
    o = orc.OracleIndex(cent, R.matrix, q.boundaries, q.centroids, q.half_bin_means)
    o.bins, o.signs, o.list_ids, o.norms = bins, signs, idx.list_ids, idx.norms
    pq = min(args.parity_queries, nq)
    srch = []
    for n_p in w.nprobe:
        oi, os_ = o.search_batch(queries[:pq], 10, n_p)
        gi, gs = results[n_p][0][:pq], results[n_p][1][:pq]
        ent = {"nprobe": n_p, "queries": pq}
        try:
            ent["queries_differing"] = int(compare_topk(gi, gs, oi, os_))
            ent["ok"] = True
        except AssertionError as e:  # record, do not hide
            ent["ok"] = False
            ent["error"] = str(e)[:300]
        ent["max_rel_score_diff"] = float(np.max(np.abs(gs - os_) / np.maximum(np.abs(os_),
                                                                                1e-12)))
        ent["recall_gpu"] = recall_at_k(gi, truth[:pq], 10)
        ent["recall_oracle"] = recall_at_k(oi, truth[:pq], 10)
        srch.append(ent)
        print(json.dumps(ent), flush=True)
    rep["parity"] = {"codes": codes, "search": srch}
    T["parity_s"] = time.time() - t0
    rep["timings"] = T
    print(json.dumps(rep), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main()
