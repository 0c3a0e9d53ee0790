"""Partition-only refresh with a device re-encode (refresh.py:24-215 semantics).

Steps (reference order kept so RNG streams match):
  1. source = normalised raw store (keep_raw and allowed) or the device decode
     of every stored code (reconstruct_all);
  2. rng = default_rng(seed); stratified per-list sample over members in
     ascending id order (refresh.py:109-131) -- host, O(n) ids;
  3. spherical k-means on source[sample] (host numpy, or GPU GEMMs);
  4. re-encode ALL vectors on the device against the new centroids (the ingest
     kernel chain), chunked so memory stays bounded (the reference's single
     `_encode_batch` call is row-independent, so chunking is exact);
  5. rebuild the device lists and swap them in; count, external ids, raw
     store, quantizer and rotation are untouched.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .index import IvfTqIndex
from .partition import train_partition
from .store import DeviceStore

__all__ = ["RefreshPolicy", "RefreshReport", "refresh", "reconstruct_all", "reconstruct_vector"]

_CHUNK = 1 << 20


@dataclass(frozen=True)
class RefreshPolicy:
    trigger_every_n: int = 100_000
    sample_size: int | None = None
    use_raw_if_available: bool = True
    seed: int = 0

    def __post_init__(self):
        if self.trigger_every_n < 1:
            raise ValueError("trigger_every_n must be >= 1")


@dataclass(frozen=True)
class RefreshReport:
    refreshed: bool
    duration_seconds: float
    n_reassigned: int
    sample_size: int
    used_raw: bool
    mean_assigned_ip_before: float
    mean_assigned_ip_after: float
    centroid_displacement_mean: float
    centroid_displacement_max: float


def _decode_device(index: IvfTqIndex, first: int, n: int, renormalize: bool) -> torch.Tensor:
    L = _lib.lib()
    d = index.config.dim
    out = torch.empty((max(n, 1), d), dtype=torch.float64, device=index.device)
    sb = L.ivftq_decode_scratch_bytes(n, d)
    scr = torch.empty(sb, dtype=torch.uint8, device=index.device)
    _lib.check(L.ivftq_decode(C.byref(index._store.struct()),
                              index._slot_of.t[first:].data_ptr(),
                              index._list_of.t[first:].data_ptr(), n, index._cent.data_ptr(),
                              index._RT.data_ptr(), index._levels.data_ptr(),
                              int(index.config.flat), int(renormalize), out.data_ptr(),
                              scr.data_ptr(), sb, _lib.stream_ptr()), "decode")
    return out[:n]


def reconstruct_all(index: IvfTqIndex, renormalize: bool = True) -> np.ndarray:
    """x_hat = c_l + ||r|| R^T T[code] per stored vector (refresh.py:63-81)."""
    parts = [_decode_device(index, s, min(_CHUNK, index.count - s), renormalize).cpu().numpy()
             for s in range(0, index.count, _CHUNK)]
    return np.concatenate(parts) if parts else np.zeros((0, index.config.dim))


def reconstruct_vector(index: IvfTqIndex, internal_id: int) -> np.ndarray:
    """Unit-norm reconstruction of one vector (refresh.py:84-106)."""
    if not 0 <= internal_id < index.count:
        raise ValueError(f"unknown internal id {internal_id}")
    return _decode_device(index, internal_id, 1, True).cpu().numpy()[0]


def _stratified_sample_ids(lists, n, n_lists, sample_size, rng):
    picked = []
    for members in lists:
        if len(members) == 0:
            continue
        take = max(1, int(np.ceil(sample_size * len(members) / n)))
        take = min(take, len(members))
        picked.append(rng.choice(np.asarray(members, dtype=np.int64), size=take, replace=False))
    ids = np.concatenate(picked)
    if len(ids) < n_lists:
        rest = np.setdiff1d(np.arange(n, dtype=np.int64), ids)
        extra = n_lists - len(ids)
        ids = np.concatenate([ids, rng.choice(rest, size=min(extra, len(rest)), replace=False)])
    return np.sort(ids)


def _source_rows(index: IvfTqIndex, used_raw: bool, s: int, e: int) -> torch.Tensor:
    """Rows [s, e) of the refresh source, on the device, f64."""
    if used_raw:
        L = _lib.lib()
        raw = index._raw.t[s:e]
        n = e - s
        out = torch.empty((max(n, 1), index.config.dim), dtype=torch.float64, device=index.device)
        bad = torch.empty(1, dtype=torch.int64, device=index.device)
        _lib.check(L.ivftq_normalize_rows(raw.data_ptr(), _lib.IVFTQ_F32, n, index.config.dim,
                                          out.data_ptr(), bad.data_ptr(), _lib.stream_ptr()),
                   "normalize_rows")
        return out[:n]
    return _decode_device(index, s, e - s, True)


def _mean_rowdot(index, src: torch.Tensor, cent: torch.Tensor, lids: torch.Tensor) -> float:
    L = _lib.lib()
    n = src.shape[0]
    out = torch.empty(max(n, 1), dtype=torch.float64, device=index.device)
    _lib.check(L.ivftq_rowdot(src.data_ptr(), cent.data_ptr(), lids.data_ptr(), n,
                              index.config.dim, out.data_ptr(), _lib.stream_ptr()), "rowdot")
    return out[:n]


# sample rows x lists above which "auto" trains on the device: the host path
# materialises an (n, L) f64 score matrix per Lloyd step (2^27 entries = 1 GiB)
_AUTO_DEVICE_WORK = 1 << 27


def refresh(index: IvfTqIndex, policy: RefreshPolicy, kmeans_device: str = "auto",
            centroids: np.ndarray | None = None) -> RefreshReport:
    """Re-cluster the coarse partition and re-encode every vector on the GPU.

    Args:
        kmeans_device: "cpu" (numpy k-means, bit-exact with the reference's
            OpenBLAS path), "cuda" (the hand-written device k-means,
            partition.py:_train_device) or "auto": the device once the sample
            times the list count reaches 2^27 (where the host path's per-step
            (n, L) f64 score matrix passes 1 GiB), the host below that.
        centroids: inject pre-trained (L, d) f32 centroids instead of training
            (isolates the re-encode kernel in parity runs).
    """
    t0 = time.perf_counter()
    n = index.count
    if n == 0:
        return RefreshReport(False, 0.0, 0, 0, False, float("nan"), float("nan"), 0.0, 0.0)
    if index.config.flat:
        raise ValueError("flat-mode indexes have no coarse partition to refresh")
    n_lists = index.partition.n_lists
    sample_size = policy.sample_size
    if sample_size is None:
        sample_size = min(n, max(100 * n_lists, n // 10))
    sample_size = max(sample_size, n_lists)
    used_raw = bool(policy.use_raw_if_available and index._raw is not None)

    rng = np.random.default_rng(policy.seed)
    # per-list members in ascending id order (what partition.lists holds,
    # refresh.py:115-121), as arrays: no Python list of n ints at 10M scale
    lids = index.list_ids
    order = torch.argsort(index._list_of.t[:n], stable=True).cpu().numpy()  # = np.argsort(lids, "stable")
    members = np.split(order, np.cumsum(np.bincount(lids, minlength=n_lists))[:-1])
    sample_ids = _stratified_sample_ids(members, n, n_lists, sample_size, rng)
    dev = index.device
    if centroids is None:
        sid = torch.from_numpy(sample_ids).to(dev)
        rows = []
        for s in range(0, n, _CHUNK):
            e = min(n, s + _CHUNK)
            sel = sid[(sid >= s) & (sid < e)] - s
            if sel.numel():
                rows.append(_source_rows(index, used_raw, s, e)[sel])
        sample = torch.cat(rows)
        del rows
        if kmeans_device == "auto":
            big = len(sample) * n_lists >= _AUTO_DEVICE_WORK
            kmeans_device = "cuda" if big and (index.config.dim + 31) // 32 * 32 <= 256 else "cpu"
        if kmeans_device != "cuda":
            sample = sample.cpu().numpy()
        new_part = train_partition(sample, n_lists, seed=policy.seed, device=kmeans_device,
                                   memberships=False)
        del sample
    else:
        from .partition import CoarsePartition
        new_part = CoarsePartition(n_lists, index.config.dim, np.asarray(centroids, np.float32))
    new_part.lists = [[] for _ in range(n_lists)]
    new_cent = torch.from_numpy(np.ascontiguousarray(new_part.centroids)).to(dev)

    enc = []
    ip_b = torch.zeros((), dtype=torch.float64, device=dev)
    ip_a = torch.zeros((), dtype=torch.float64, device=dev)
    for s in range(0, n, _CHUNK):
        e = min(n, s + _CHUNK)
        src = _source_rows(index, used_raw, s, e)
        ip_b += _mean_rowdot(index, src, index._cent, index._list_of.t[s:e]).sum()
        words, lids, nrm, _ = index._encode_device(src, partition=new_part)
        ip_a += _mean_rowdot(index, src, new_cent, lids).sum()
        enc.append((words, lids, nrm))

    old = index.partition.centroids.astype(np.float64)
    cross = new_part.centroids.astype(np.float64) @ old.T
    disp = np.sqrt(np.maximum(2.0 - 2.0 * cross.max(axis=1), 0.0))

    # swap: fresh device lists holding every vector under the new partition
    st = DeviceStore(index.config.dim, index.config.bits, index.config.use_sign_bit, n_lists, dev)
    L = _lib.lib()
    counts = np.zeros(n_lists, dtype=np.int64)
    cbuf = torch.empty(n_lists, dtype=torch.int32, device=dev)
    for (_, lids, _) in enc:
        _lib.check(L.ivftq_histogram(lids.data_ptr(), lids.shape[0], n_lists, cbuf.data_ptr(),
                                     _lib.stream_ptr()), "histogram")
        counts += cbuf.cpu().numpy()
    st.reserve(counts, index._slot_of.t)
    cursor = torch.empty(n_lists, dtype=torch.int32, device=dev)
    first = 0
    for (words, lids, nrm) in enc:
        m = words.shape[0]
        _lib.check(L.ivftq_append(C.byref(st.struct()), words.data_ptr(), nrm.data_ptr(),
                                  lids.data_ptr(), m, first, cursor.data_ptr(),
                                  index._slot_of.t.data_ptr(), _lib.stream_ptr()), "append")
        st.set_sizes(st.sizes + np.bincount(lids.cpu().numpy(), minlength=n_lists))
        index._list_of.t[first:first + m] = lids
        index._norm_of.t[first:first + m] = nrm
        first += m
    index._store = st
    index._set_partition(new_part)
    index._version += 1
    return RefreshReport(
        refreshed=True, duration_seconds=time.perf_counter() - t0, n_reassigned=n,
        sample_size=int(len(sample_ids)), used_raw=used_raw,
        mean_assigned_ip_before=float(ip_b.item()) / n,
        mean_assigned_ip_after=float(ip_a.item()) / n,
        centroid_displacement_mean=float(disp.mean()),
        centroid_displacement_max=float(disp.max()))
