"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (the reference exists only here):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes tests/golden/*.npz. The reference ships no golden files
(SURVEY.md §4, §8c); these pin (1) the oracle restatement and (2) the CUDA
path on the GPU box, where /root/reference does not exist. Inputs are this
repo's seeded mixtures (paper_2605_17415_b200.workloads), so large inputs are
regenerated rather than stored.
"""

from __future__ import annotations

import io
import sys
import warnings
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import ivftq  # noqa: E402  (the reference; build container only)
from ivftq.evaluation import exact_topk  # noqa: E402
from ivftq.index import IndexConfig, IvfTqIndex  # noqa: E402
from ivftq.partition import CoarsePartition, train_partition  # noqa: E402
from ivftq.refresh import RefreshPolicy, _stratified_sample_ids, refresh  # noqa: E402
from ivftq.storage import save_index  # noqa: E402

from paper_2605_17415_b200.workloads import make_workload, mixture  # noqa: E402

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT))
from hashing import row_hash  # noqa: E402


def dump_index(prefix: str, idx: IvfTqIndex) -> dict:
    q = idx.quantizer
    cfg = idx.config
    d = {
        f"{prefix}boundaries": q.boundaries,
        f"{prefix}qcent": q.centroids,
        f"{prefix}half": q.half_bin_means,
        f"{prefix}distortion": np.array([q.distortion, q.distortion_sign]),
        f"{prefix}R": idx.rot.matrix,
        f"{prefix}centroids": idx.partition.centroids,
        f"{prefix}config": np.array([cfg.dim, cfg.bits, cfg.n_lists, cfg.use_sign_bit,
                                     cfg.keep_raw, cfg.flat, cfg.rotation_seed,
                                     cfg.kmeans_seed], dtype=np.int64),
        f"{prefix}list_ids": idx.list_ids.copy(),
        f"{prefix}norms": idx.norms.copy(),
        f"{prefix}ext": idx.external_ids.copy(),
        f"{prefix}bins": idx.bins.copy(),
        f"{prefix}signs": idx.signs.copy(),
        f"{prefix}fingerprint": np.frombuffer(
            idx.compression_fingerprint().encode(), dtype=np.uint8),
    }
    return d


def searches(idx, queries, cases):
    out = {}
    for (k, n_p, rr) in cases:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            ids, sc = idx.search_batch(queries, k, n_p, rr)
        out[f"s_{k}_{n_p}_{rr}_ids"] = ids
        out[f"s_{k}_{n_p}_{rr}_scores"] = sc
    return out


def small_case(name, n, d, comps, bits, n_lists, nq, cases, use_sign=True,
               keep_raw=False, flat=False, kseed=42, seed=0, save=False,
               extra_rows=None):
    x, means = mixture(n, d, comps, 0.3, seed)
    if extra_rows is not None:
        x = np.concatenate([x, extra_rows(x)]).astype(np.float32)
    qx, _ = mixture(nq, d, comps, 0.3, seed + 1, means=means)
    cfg = IndexConfig(dim=d, bits=bits, n_lists=n_lists, use_sign_bit=use_sign,
                      keep_raw=keep_raw, flat=flat, kmeans_seed=kseed)
    idx = IvfTqIndex.build(cfg, x)
    rec = {"x": x, "queries": qx}
    rec.update(dump_index("", idx))
    rec.update(searches(idx, qx, cases))
    xn = x / np.linalg.norm(x.astype(np.float64), axis=1)[:, None]
    rec["truth10"] = exact_topk(xn, qx, 10).ids
    if keep_raw:
        rec["raw"] = idx.raw.copy()
    # probe lists / coarse exactly as index.py:434-438
    qn = qx / np.linalg.norm(qx.astype(np.float64), axis=1)[:, None]
    coarse = qn @ idx.partition.centroids.T.astype(np.float64)
    rec["probe_all"] = np.argsort(-coarse, axis=1, kind="stable")
    rec["coarse"] = coarse
    if save:
        buf = OUT / "_tmp.ivtq"
        save_index(idx, buf)
        rec["ivtq_bytes"] = np.frombuffer(buf.read_bytes(), dtype=np.uint8)
        buf.unlink()
    # a fresh single-vector encode of a centroid (index.py:269-279)
    if not flat:
        code = idx.encode(idx.partition.centroids[min(3, n_lists - 1)].astype(np.float64))
        rec["centroid_code"] = np.frombuffer(code.codes + code.signs, dtype=np.uint8)
        rec["centroid_code_meta"] = np.array([code.list_id,
                                              float(code.residual_norm)])
    np.savez_compressed(OUT / f"{name}.npz", **rec)
    print(name, "ok", idx.count, "vectors")
    return idx


def refresh_case(name, keep_raw, seed):
    x, means = mixture(3000, 32, 24, 0.3, 11)
    qx, _ = mixture(50, 32, 24, 0.3, 12, means=means)
    cfg = IndexConfig(dim=32, bits=4, n_lists=16, keep_raw=keep_raw, kmeans_seed=7)
    idx = IvfTqIndex.build(cfg, x)
    rec = {"x": x, "queries": qx}
    rec.update(dump_index("pre_", idx))
    pol = RefreshPolicy(seed=seed)
    n = idx.count
    sample = min(n, max(100 * 16, n // 10))
    rng = np.random.default_rng(seed)
    rec["sample_ids"] = _stratified_sample_ids(idx, sample, rng)
    rep = refresh(idx, pol)
    rec.update(dump_index("post_", idx))
    rec["report"] = np.array([rep.n_reassigned, rep.sample_size, rep.used_raw,
                              rep.mean_assigned_ip_before, rep.mean_assigned_ip_after,
                              rep.centroid_displacement_mean,
                              rep.centroid_displacement_max])
    rec["post_lists"] = np.concatenate(
        [np.asarray(m, np.int64) for m in idx.partition.lists])
    rec.update(searches(idx, qx, [(10, 8, 0)]))
    np.savez_compressed(OUT / f"{name}.npz", **rec)
    print(name, "ok")


def pr1_case():
    w = make_workload("pr1")
    x = w.base()
    qx = w.queries()
    xn = x.astype(np.float64)
    xn = xn / np.linalg.norm(xn, axis=1)[:, None]
    cfg = IndexConfig(dim=w.d, bits=w.bits, n_lists=w.n_lists)
    part = train_partition(xn, w.n_lists, seed=cfg.kmeans_seed, max_iters=w.kmeans_iters)
    shared = CoarsePartition(n_lists=w.n_lists, dim=w.d, centroids=part.centroids)
    idx = IvfTqIndex(cfg, ivftq.design_quantizer(w.bits, w.d),
                     ivftq.generate_rotation(w.d, cfg.rotation_seed), shared)
    idx.add_batch(x)
    rec = dump_index("", idx)
    for key in ("bins", "signs"):
        del rec[key]
    packed = np.concatenate([ivftq.pack_fields(idx.bins, w.bits),
                             ivftq.pack_fields(idx.signs, 1)], axis=1)
    rec["code_hash"] = row_hash(packed)
    rec["list_ids"] = idx.list_ids.astype(np.int16)
    rec.update(searches(idx, qx, [(10, p, 0) for p in (1, 4, 16, 64)]))
    qn = qx / np.linalg.norm(qx.astype(np.float64), axis=1)[:, None]
    rec["truth10"] = exact_topk(xn, qn, 10).ids
    coarse = qn @ idx.partition.centroids.T.astype(np.float64)
    rec["probe64"] = np.argsort(-coarse, axis=1, kind="stable")[:, :64].astype(np.int16)
    np.savez_compressed(OUT / "pr1.npz", **rec)
    print("pr1 ok")


def quantizer_tables():
    rec = {}
    for b in range(1, 9):
        for d in (16, 32, 96, 128, 200):
            q = ivftq.design_quantizer(b, d)
            rec[f"b{b}_d{d}_bnd"] = q.boundaries
            rec[f"b{b}_d{d}_cent"] = q.centroids
            rec[f"b{b}_d{d}_half"] = q.half_bin_means
            rec[f"b{b}_d{d}_dist"] = np.array([q.distortion, q.distortion_sign])
    for d in (16, 24, 32, 96, 128, 200):
        rec[f"rot_{d}"] = ivftq.generate_rotation(d, 42).matrix
    np.savez_compressed(OUT / "tables.npz", **rec)
    print("tables ok")


def main():
    quantizer_tables()
    # duplicate rows exercise exact score ties (-> lower internal id)
    dup = lambda x: x[:40].copy()  # noqa: E731
    small_case("d32_b4_L16_raw", 2000, 32, 20, 4, 16, 100,
               [(10, 4, 0), (10, 16, 0), (1, 16, 0), (2100, 4, 0), (5, 8, 20),
                (3, 999, 0)], keep_raw=True, extra_rows=dup, save=True)
    small_case("d16_b3_L8", 1200, 16, 10, 3, 8, 100, [(10, 8, 0), (5, 2, 0)], kseed=1)
    small_case("d24_b5_L12_raw", 1500, 24, 12, 5, 12, 40,
               [(8, 6, 0), (8, 6, 10)], keep_raw=True, kseed=2, save=True)
    small_case("d96_b2_nosign_L32", 4000, 96, 40, 2, 32, 64, [(10, 8, 0)],
               use_sign=False, save=True)
    small_case("d200_b3_L16", 3000, 200, 30, 3, 16, 64, [(10, 4, 0), (10, 16, 0)])
    small_case("d64_b8_L8", 1500, 64, 16, 8, 8, 40, [(10, 3, 0)])
    small_case("d40_b1_L4", 800, 40, 8, 1, 4, 40, [(10, 2, 0)])
    small_case("d128_b4_L64", 8000, 128, 64, 4, 64, 200, [(10, 16, 0), (100, 8, 0)])
    small_case("flat_d16_b8", 500, 16, 6, 8, 1, 30, [(5, 1, 0), (600, 1, 0)],
               flat=True, save=True)
    refresh_case("refresh_recon", keep_raw=False, seed=3)
    refresh_case("refresh_raw", keep_raw=True, seed=4)
    pr1_case()


if __name__ == "__main__":
    main()
