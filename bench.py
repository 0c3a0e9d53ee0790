#!/usr/bin/env python
"""Benchmark of the B200 IVF-TQ hot path (search QPS at recall@10, list-scan
roofline, adds/s) on BASELINE.json configs[1] by default.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|pr1|c3] [--nprobe P]

One step = one `search_batch` of the 10k-query batch (k=10) at the headline
nprobe over the resident index. Every timed step is bracketed by CUDA events
on the launching stream; L2 is flushed (a 512 MiB write, larger than the
126 MB L2) before each step, outside the events. N>1 (torchrun): every rank
holds a replica and searches its own query batch (weak scaling, no data-path
collective); the reported time is the max over ranks.

`--impl reference` times the CPU restatement of the reference path
(oracle/ivftq_oracle.py; the reference itself is pure Python and is not on the
GPU box) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "QPS at recall@10 (nprobe sweep); list-scan HBM GB/s vs peak; adds/sec"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--nprobe", type=int, default=None)
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--n", type=int, default=None, help="override database size (testing)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1606.9)), "measured"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampled every 200 ms while the timed region runs."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            if len(r) < 9:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows)}


def code_bytes(bits: int, d: int) -> int:
    """Algorithmic bytes per scanned vector: s(b,d)."""
    return -(-bits * d // 8) + -(-d // 8) + 2


def train_centroids(w, xn_host):
    from paper_2605_17415_b200.partition import train_partition

    n = len(xn_host)
    m = w.kmeans_sample or n
    rng = np.random.default_rng(w.base_seed + 17)
    sub = xn_host[np.sort(rng.choice(n, size=min(m, n), replace=False))] if m < n else xn_host
    return train_partition(sub, w.n_lists, seed=42, max_iters=w.kmeans_iters).centroids


def setup(args, rank):
    from paper_2605_17415_b200.workloads import make_workload

    w = make_workload(args.config)
    if args.n:
        w = make_workload(args.config, n=args.n)
    nq = args.nq or w.n_queries
    base = w.base()
    queries = make_workload(args.config, query_seed=w.query_seed + rank).queries(nq)
    xn = base.astype(np.float64)
    xn /= np.linalg.norm(xn, axis=1)[:, None]
    n_p = args.nprobe or max(w.nprobe)
    return w, base, xn, queries, nq, n_p


def cpu_oracle_index(idx):
    """Oracle index holding the GPU-encoded fields (bit-identical to its own encode)."""
    from oracle import ivftq_oracle as orc

    o = orc.OracleIndex(idx.partition.centroids, idx.rot.matrix, idx.quantizer.boundaries,
                        idx.quantizer.centroids, idx.quantizer.half_bin_means,
                        use_sign=idx.config.use_sign_bit)
    o.bins, o.signs = idx.bins, idx.signs
    o.list_ids, o.norms = idx.list_ids, idx.norms
    return o


def time_cpu_search(o, queries, k, n_p, seconds):
    """Reference protocol (harness.py:281-289): 8-query warm-up, then perf_counter."""
    o.search_batch(queries[:8], k, n_p)
    m = 16
    t0 = time.perf_counter()
    o.search_batch(queries[:m], k, n_p)
    rate = m / (time.perf_counter() - t0)
    m = int(min(len(queries), max(16, rate * seconds)))
    t0 = time.perf_counter()
    o.search_batch(queries[:m], k, n_p)
    dt = time.perf_counter() - t0
    return m / dt, m, dt


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ivftq_oracle as orc
    from paper_2605_17415_b200.quantizer import design_quantizer
    from paper_2605_17415_b200.rotation import generate_rotation

    w, base, xn, queries, nq, n_p = setup(args, 0)
    cent = train_centroids(w, xn)
    q = design_quantizer(w.bits, w.d)
    R = generate_rotation(w.d, 42)
    o = orc.OracleIndex(cent, R.matrix, q.boundaries, q.centroids, q.half_bin_means)
    t0 = time.perf_counter()
    for s in range(0, len(base), 100_000):  # 100k-row add_batch chunks
        o.add_batch(base[s:s + 100_000])
    adds = len(base) / (time.perf_counter() - t0)
    o.search_batch(queries[:8], 10, n_p)
    t0 = time.perf_counter()
    o.search_batch(queries[:16], 10, n_p)
    rate = 16 / (time.perf_counter() - t0)
    per_step = int(min(nq, max(8, rate * 6.0)))
    for i in range(args.warmup):
        o.search_batch(queries[:per_step], 10, n_p)
    times = []
    for i in range(args.steps):
        sl = queries[(i * per_step) % nq:][:per_step]
        t0 = time.perf_counter()
        o.search_batch(sl, 10, n_p)
        times.append(time.perf_counter() - t0)
    qps = per_step * len(times) / sum(times)
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * float(np.mean(times)), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
        "config": {"workload": w.name, "n": len(base), "d": w.d, "n_lists": w.n_lists,
                   "bits": w.bits, "k": 10, "nprobe": n_p, "nq_per_step": per_step},
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": cores, "kind": "port",
                         "sample": f"{per_step} queries per step of the {nq}-query batch; "
                                   f"oracle restatement of the reference (numpy/OpenBLAS, "
                                   f"all {cores} threads)"},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "ingest": {"adds_per_sec": adds, "rows": len(base), "chunk": 100_000},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    from paper_2605_17415_b200 import _lib
    from paper_2605_17415_b200.evaluation import exact_topk, recall_at_k
    from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex
    from paper_2605_17415_b200.partition import CoarsePartition
    from paper_2605_17415_b200.quantizer import design_quantizer
    from paper_2605_17415_b200.rotation import generate_rotation

    from paper_2605_17415_b200.replicas import job_throughput, max_over_ranks, share_centroids

    L = _lib.lib()
    w, base, xn, queries, nq, n_p = setup(args, rank)
    cent = share_centroids(train_centroids(w, xn) if rank == 0 else None, (w.n_lists, w.d), dev)
    cfg = IndexConfig(dim=w.d, bits=w.bits, n_lists=w.n_lists)
    idx = IvfTqIndex(cfg, design_quantizer(w.bits, w.d), generate_rotation(w.d, 42),
                     CoarsePartition(w.n_lists, w.d, cent), device=dev)

    # ---- ingest: adds/s end to end (host f32 rows -> device lists) ----------
    chunk = len(base)  # one add_batch of the whole pinned batch (sub-chunked copy/encode overlap inside)
    pinned = torch.from_numpy(base).pin_memory()
    # warm-up on a throwaway index: first-use allocations and kernel loads stay
    # out of the timed region (the timed run still grows its own store)
    warm = IvfTqIndex(cfg, design_quantizer(w.bits, w.d), generate_rotation(w.d, 42),
                      CoarsePartition(w.n_lists, w.d, cent), device=dev)
    warm.add_batch(pinned[: min(chunk, 600_000)])
    del warm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # three timed ingests of the whole batch into fresh indexes (the last one
    # is the searched index); the median is reported
    ing = []
    for r in range(3):
        if r < 2:
            tgt = IvfTqIndex(cfg, design_quantizer(w.bits, w.d), generate_rotation(w.d, 42),
                             CoarsePartition(w.n_lists, w.d, cent), device=dev)
        else:
            tgt = idx
        torch.cuda.synchronize()
        e0.record()
        for s in range(0, len(base), chunk):
            tgt.add_batch(pinned[s:s + chunk])
        e1.record()
        torch.cuda.synchronize()
        ing.append(e0.elapsed_time(e1) / 1000)
        del tgt
    ingest_s = float(np.median(ing))
    # kernel-only encode throughput on a device-resident chunk
    xd = torch.from_numpy(base[:250_000]).to(dev)
    idx._encode_device(xd)
    torch.cuda.synchronize()
    e0.record()
    idx._encode_device(xd)
    e1.record()
    torch.cuda.synchronize()
    enc_s = e0.elapsed_time(e1) / 1000

    # ---- ground truth (GPU brute force, reference tie rule) ----------------
    qn = queries.astype(np.float64)
    qn /= np.linalg.norm(qn, axis=1)[:, None]
    truth = exact_topk(torch.from_numpy(xn).to(dev), qn, 10).ids
    del xd

    Qd = torch.from_numpy(queries).to(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def step(np_):
        return idx.search_batch(Qd, 10, np_, return_device=True)

    sweep = []
    for p in w.nprobe:
        step(p)
        flush.fill_(1)
        torch.cuda.synchronize()
        e0.record()
        ids, _ = step(p)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1000
        sweep.append({"nprobe": p, "qps": nq / t,
                      "recall_at_10": recall_at_k(ids.cpu().numpy(), truth, 10)})

    # ---- headline: K timed steps (device-resident queries) ------------------
    for _ in range(args.warmup):
        step(n_p)
    clocks = Clocks(local)
    times = []
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        c0 = L.ivftq_launch_count()
        e0.record()
        ids, sc = step(n_p)
        e1.record()
        torch.cuda.synchronize()
        launches += L.ivftq_launch_count() - c0
        times.append(e0.elapsed_time(e1))
    clk = clocks.stop()
    ms_max = max_over_ranks(float(np.mean(times)), dev)
    value = job_throughput(nq, ms_max)
    recall = recall_at_k(ids.cpu().numpy(), truth, 10)

    # ---- e2e through the public API with host buffers -----------------------
    qpin = torch.from_numpy(queries).pin_memory()
    for _ in range(max(args.warmup, 3)):  # also warms the pinned result buffers
        hi, hs = idx.search_batch(qpin, 10, n_p)
    e2e_t = []
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0.record()
        hi, hs = idx.search_batch(qpin, 10, n_p)  # numpy results (D2H inside)
        e1.record()
        torch.cuda.synchronize()
        e2e_t.append(e0.elapsed_time(e1))
    e2e_val = job_throughput(nq, max_over_ranks(float(np.mean(e2e_t)), dev))

    # ---- roofline of the dominant kernel (list scan) ------------------------
    import ctypes as C

    qnd, bad, _ = idx._normalize_queries_device(Qd)
    probe = torch.empty((nq, n_p), dtype=torch.int32, device=dev)
    coarse = torch.empty((nq, n_p), dtype=torch.float64, device=dev)
    pb = L.ivftq_probe_scratch_bytes(nq, w.n_lists, w.d)
    pscr = torch.empty(pb, dtype=torch.uint8, device=dev)
    s = _lib.stream_ptr()
    _lib.check(L.ivftq_probe(qnd.data_ptr(), idx._cent.data_ptr(), nq, w.n_lists, w.d, n_p,
                             probe.data_ptr(), coarse.data_ptr(), pscr.data_ptr(), pb, s))
    qrot = torch.empty((nq, w.d), dtype=torch.float32, device=dev)
    _lib.check(L.ivftq_gemm_nt(qnd.data_ptr(), idx._R.data_ptr(), 1, nq, w.d, w.d,
                               qrot.data_ptr(), 0, s))
    oid = torch.empty((nq, 10), dtype=torch.int64, device=dev)
    osc = torch.empty((nq, 10), dtype=torch.float64, device=dev)
    sb = L.ivftq_scan_scratch_bytes(nq, n_p, 10, w.n_lists)
    sscr = torch.empty(sb, dtype=torch.uint8, device=dev)
    st = idx._store.struct()

    def scan():
        _lib.check(L.ivftq_scan_topk(C.byref(st), probe.data_ptr(), coarse.data_ptr(),
                                     qrot.data_ptr(), idx._levels.data_ptr(), nq, n_p, 10,
                                     oid.data_ptr(), osc.data_ptr(), sscr.data_ptr(), sb, s))

    scan()
    sc_t, k_t = [], []
    L.ivftq_set_kernel_timing(1)
    for _ in range(max(3, args.steps)):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0.record()
        scan()
        e1.record()
        torch.cuda.synchronize()
        sc_t.append(e0.elapsed_time(e1) / 1000)
        k_t.append(L.ivftq_last_scan_kernel_ms() / 1000)
    L.ivftq_set_kernel_timing(0)
    t_scan = float(np.mean(sc_t))       # regroup + scan kernel + per-query merge
    t_kernel = float(np.mean(k_t))      # the tensor-core scan kernel alone
    sizes = idx._store.sizes
    vq = float(sizes[probe.cpu().numpy()].sum())  # sum_q V_q (candidate vectors)
    s_vec = code_bytes(w.bits, w.d)
    alg_bytes = vq * s_vec
    alg_flops = 2.0 * w.d * vq  # one d-dim dot per (query, candidate): SURVEY 8(d)
    hbm, tf, src = peaks()
    achieved_tf = alg_flops / t_kernel / 1e12
    traffic = None
    prof = ROOT / "profiles" / "scan_traffic.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get(w.name)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        o = cpu_oracle_index(idx)
        qps_cpu, m, dt = time_cpu_search(o, queries, 10, n_p, args.cpu_seconds)
        cpu = {"value": qps_cpu, "unit": "queries/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"{m} of {nq} queries at nprobe={n_p} ({dt:.1f} s), oracle "
                         f"restatement over the same encoded index, numpy/OpenBLAS all threads"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32/f64", "data": "synthetic (seeded Gaussian mixture, SURVEY §8d)",
            "config": {"workload": w.name, "n": len(base), "d": w.d, "n_lists": w.n_lists,
                       "bits": w.bits, "sign_bit": True, "nq": nq, "k": 10, "nprobe": n_p,
                       "parallelism": f"replica x{world} (query-sharded)",
                       "l2": "flushed before every timed step (512 MiB write)"},
            "recall_at_10": recall,
            "sweep": sweep,
            # The list-major scan re-uses each list's codes for every query probing
            # it, so it is not HBM-bound: its roofline is the tensor pipe
            # (algorithmic 2*d flops per (query, candidate); executed MMA work is
            # 3x that for the fp16 hi/lo split). effective_gbs is the per-query
            # code stream a query-major scan would read (sum_q V_q * s(b,d)).
            "roofline": {"bound": "tensor", "achieved": achieved_tf, "peak": tf,
                         "unit": "TFLOP/s", "frac": achieved_tf / tf, "traffic": traffic,
                         "kernel": "scan_tc_kernel", "peak_source": src + " bf16 dense",
                         "alg_flops_per_launch": alg_flops, "kernel_ms": t_kernel * 1000,
                         "scan_call_ms": t_scan * 1000, "alg_bytes_per_launch": alg_bytes,
                         "bytes_per_vector": s_vec,
                         "effective_gbs": alg_bytes / t_kernel / 1e9,
                         "effective_frac_of_hbm": alg_bytes / t_kernel / 1e9 / hbm},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "queries/s",
                    "h2d_bytes_per_step": int(queries.nbytes),
                    "d2h_bytes_per_step": int(nq * 10 * 16),
                    "steps_ms": [round(t, 3) for t in e2e_t]},
            "clocks": clk,
            "gpu_launches": int(launches),
            "ingest": {"adds_per_sec_e2e": len(base) / ingest_s,
                       "adds_per_sec_device_encode": 250_000 / enc_s, "rows": len(base),
                       "chunk": chunk, "reps_ms": [round(t * 1000, 2) for t in ing], "stat": "median"},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
