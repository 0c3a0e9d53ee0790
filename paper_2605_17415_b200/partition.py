"""Coarse partition: spherical k-means (host) + list membership views.

`train_partition` restates partition.py:98-178 (greedy k-means++ seeding,
max-IP Lloyd steps with renormalised means, farthest-point empty repair) with
the same RNG call order, so the same (data, L, seed, max_iters) gives the
reference's centroids bit-for-bit on the host path. With `device="cuda"` the
two O(n*L*d) products per iteration (assignment, k-means++ candidate IPs) run
on the GPU through the library's f64 GEMMs; those differ from OpenBLAS only in
f64 rounding order (documented in DESIGN.md).

Membership: the reference keeps Python lists of member ids per list
(partition.py:34) and appends to them per row (index.py:307-308). Here the
device list store is the source of truth; `CoarsePartition.lists` is a lazy
host view (ascending ids per list, the order refresh sampling relies on,
refresh.py:115-121) produced on access when the partition is attached to an
index.
"""

from __future__ import annotations

from typing import Callable

import numpy as np

__all__ = ["CoarsePartition", "train_partition", "assign"]

_EPS = 1e-12


class CoarsePartition:
    """Unit-norm f32 centroids (L, d) plus per-list member ids."""

    def __init__(self, n_lists: int, dim: int, centroids: np.ndarray, lists=None):
        self.n_lists = int(n_lists)
        self.dim = int(dim)
        self.centroids = np.asarray(centroids, dtype=np.float32)
        self._lists = lists if lists else [[] for _ in range(self.n_lists)]
        self._provider: Callable[[], list] | None = None

    @property
    def lists(self):
        if self._provider is not None:
            return self._provider()
        return self._lists

    @lists.setter
    def lists(self, value):
        self._provider = None
        self._lists = value

    def _attach(self, provider: Callable[[], list] | None):
        self._provider = provider

    @property
    def total_members(self) -> int:
        return sum(len(m) for m in self.lists)

    def assign_batch(self, vectors: np.ndarray):
        """Max-IP assignment on the host (ties -> lowest id), partition.py:45-55."""
        v = np.asarray(vectors, dtype=np.float64)
        ips = v @ self.centroids.T.astype(np.float64)
        ids = np.argmax(ips, axis=1)
        return ids.astype(np.int64), ips[np.arange(len(v)), ids]

    def __eq__(self, other):
        return (isinstance(other, CoarsePartition) and self.n_lists == other.n_lists
                and np.array_equal(self.centroids, other.centroids))

    def __repr__(self):
        return f"CoarsePartition(n_lists={self.n_lists}, dim={self.dim})"


def assign(p: CoarsePartition, v: np.ndarray) -> tuple[int, float]:
    ids, ips = p.assign_batch(np.asarray(v, dtype=np.float64)[None, :])
    return int(ids[0]), float(ips[0])


class _HostOps:
    @staticmethod
    def ip(a, b):
        return a @ b.T

    @staticmethod
    def ipv(a, v):
        return a @ v


def _kmeanspp(data, k, rng, ops):
    n = data.shape[0]
    nc = 2 + int(np.log2(k)) if k > 1 else 1
    chosen = np.empty(k, dtype=np.int64)
    chosen[0] = rng.integers(n)
    d2 = np.maximum(2.0 - 2.0 * ops.ipv(data, data[chosen[0]]), 0.0)
    for j in range(1, k):
        tot = d2.sum()
        if tot <= _EPS:
            keep = np.ones(n, dtype=bool)
            keep[chosen[:j]] = False
            pool = np.flatnonzero(keep)
            chosen[j] = rng.choice(pool) if len(pool) else rng.integers(n)
            d2 = np.minimum(d2, np.maximum(2.0 - 2.0 * ops.ipv(data, data[chosen[j]]), 0.0))
            continue
        cand = rng.choice(n, size=nc, p=d2 / tot)
        cd2 = np.maximum(2.0 - 2.0 * ops.ip(data, data[cand]), 0.0)
        pot = np.minimum(d2[:, None], cd2).sum(axis=0)
        b = int(np.argmin(pot))
        chosen[j] = cand[b]
        d2 = np.minimum(d2, cd2[:, b])
    return data[chosen].copy()


def train_partition(data: np.ndarray, n_lists: int, seed: int, max_iters: int = 25,
                    device: str = "cpu") -> CoarsePartition:
    """Spherical k-means++ / Lloyd on unit rows; f32 centroids + memberships.

    Args:
        device: "cpu" (bit-exact with the reference) or "cuda" (f64 GEMMs on
            the GPU; differs only through f64 summation order).
    """
    data = np.asarray(data, dtype=np.float64)
    n, dim = data.shape
    if n_lists < 1:
        raise ValueError(f"n_lists must be >= 1, got {n_lists}")
    if n < n_lists:
        raise ValueError(f"need at least n_lists={n_lists} rows, got {n}")
    if np.any(np.linalg.norm(data, axis=1) < _EPS):
        raise ValueError("zero-norm row in training data")
    if device == "cuda":
        return _train_device(data, n_lists, seed, max_iters)
    ops = _HostOps()
    rng = np.random.default_rng(seed)
    cent = _kmeanspp(data, n_lists, rng, ops)
    prev = None
    for _ in range(max_iters):
        ips = ops.ip(data, cent)
        a = np.argmax(ips, axis=1)
        if prev is not None and np.array_equal(a, prev):
            break
        prev = a
        cnt = np.bincount(a, minlength=n_lists)
        order = np.argsort(a, kind="stable")
        starts = np.concatenate(([0], np.cumsum(cnt)[:-1]))
        ne = np.flatnonzero(cnt > 0)
        sums = np.zeros((n_lists, dim))
        sums[ne] = np.add.reduceat(data[order], starts[ne], axis=0)
        empty = np.flatnonzero(cnt == 0)
        if len(empty):
            far = np.argsort(ips[np.arange(n), a], kind="stable")
            for slot, pt in zip(empty, far[: len(empty)]):
                sums[slot] = data[pt]
                cnt[slot] = 1
        nn = np.linalg.norm(sums, axis=1)
        bad = nn < _EPS
        if np.any(bad):
            for slot in np.flatnonzero(bad):
                sums[slot] = data[rng.integers(n)]
            nn = np.linalg.norm(sums, axis=1)
        cent = sums / nn[:, None]
    final = np.argmax(ops.ip(data, cent), axis=1)
    order = np.argsort(final, kind="stable")
    counts = np.bincount(final, minlength=n_lists)
    lists = [m.tolist() for m in np.split(order, np.cumsum(counts)[:-1])]
    return CoarsePartition(n_lists=n_lists, dim=dim, centroids=cent.astype(np.float32),
                           lists=lists)


def _train_device(data: np.ndarray, n_lists: int, seed_value: int, max_iters: int,
                  chunk: int = 1 << 16) -> CoarsePartition:
    """The same algorithm and RNG call sequence as the host path, with the data
    resident on the GPU: f64 products through ivftq_gemm_nt, the n-long
    k-means++ potential and Lloyd sums kept on the device (sums by a
    deterministic segmented reduction over rows sorted by list). Only the
    sampling vector p (8n bytes per seeding step) and a few scalars cross to
    the host. Results differ from the host path only through f64 summation
    order; memory is O(n*d + chunk*L), so it trains 1M x 4096 in one pass.
    """
    import torch

    from . import _lib

    L = _lib.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    f64 = torch.float64
    X = torch.from_numpy(np.ascontiguousarray(data, dtype=np.float64)).to(dev)
    n, dim = X.shape
    k = n_lists
    rng = np.random.default_rng(seed_value)

    def gemm(A, B):
        out = torch.empty((A.shape[0], B.shape[0]), dtype=f64, device=dev)
        _lib.check(L.ivftq_gemm_nt(A.data_ptr(), B.data_ptr(), _lib.IVFTQ_F64, A.shape[0],
                                   B.shape[0], dim, out.data_ptr(), _lib.IVFTQ_F64,
                                   _lib.stream_ptr()), "gemm_nt")
        return out

    def argmax_ip(C):
        a = torch.empty(n, dtype=torch.int64, device=dev)
        best = torch.empty(n, dtype=f64, device=dev)
        for s0 in range(0, n, chunk):
            v, i = gemm(X[s0:s0 + chunk], C).max(dim=1)  # first maximal index on ties
            a[s0:s0 + chunk] = i
            best[s0:s0 + chunk] = v
        return a, best

    def dist2(rows):
        return torch.clamp(2.0 - 2.0 * gemm(X, X[torch.as_tensor(rows, device=dev)]), min=0.0)

    # ---- k-means++ seeding (partition.py:_kmeanspp) ----
    # rng.choice(n, size=nc, p=p) draws rng.random(nc) and searches the
    # normalised cdf of p (side="right"); here the host draws the same
    # uniforms and the cdf / search / potential / argmin stay on the device.
    # The fast pass never synchronises; it records each step's potential
    # total, and a degenerate step (total <= eps: fewer distinct points than
    # k) re-runs the seeding with the host-checked branch of the reference.
    nc = 2 + int(np.log2(k)) if k > 1 else 1

    def seed(rng, checked):
        chosen = torch.empty(k, dtype=torch.int64, device=dev)
        tots = torch.empty(k, dtype=f64, device=dev)
        c0 = int(rng.integers(n))
        chosen[0] = c0
        d2 = dist2([c0])[:, 0].contiguous()
        for j in range(1, k):
            tot = d2.sum()
            tots[j] = tot
            if checked and float(tot.item()) <= _EPS:
                keep = np.ones(n, dtype=bool)
                keep[chosen[:j].cpu().numpy()] = False
                pool = np.flatnonzero(keep)
                cj = int(rng.choice(pool)) if len(pool) else int(rng.integers(n))
                chosen[j] = cj
                d2 = torch.minimum(d2, dist2([cj])[:, 0])
                continue
            cdf = torch.cumsum(d2 / tot, 0)
            cdf /= cdf[-1].clone()
            u = torch.from_numpy(rng.random(nc)).to(dev, non_blocking=True)
            cand = torch.clamp(torch.searchsorted(cdf, u, right=True), max=n - 1)
            cd2 = torch.clamp(2.0 - 2.0 * gemm(X, X[cand]), min=0.0)
            pot = torch.minimum(d2[:, None], cd2).sum(dim=0)
            bsel = torch.argmin(pot)  # first minimal index, like np.argmin
            chosen[j] = cand[bsel]
            d2 = torch.minimum(d2, cd2.index_select(1, bsel.reshape(1))[:, 0]).contiguous()
        return chosen, k == 1 or float(tots[1:].min().item()) > _EPS

    chosen, ok = seed(rng, checked=False)
    if not ok:
        rng = np.random.default_rng(seed_value)
        chosen, _ = seed(rng, checked=True)
    cent = X[chosen].clone()

    # ---- Lloyd iterations (partition.py:147-170) ----
    prev = None
    for _ in range(max_iters):
        a, best = argmax_ip(cent)
        if prev is not None and torch.equal(a, prev):
            break
        prev = a
        cnt = torch.bincount(a, minlength=k)
        order = torch.argsort(a, stable=True)
        sums = torch.segment_reduce(X[order], "sum", lengths=cnt, axis=0)
        cnt_h = cnt.cpu().numpy()
        empty = np.flatnonzero(cnt_h == 0)
        if len(empty):
            far = torch.argsort(best, stable=True)[: len(empty)]
            sums[torch.as_tensor(empty, device=dev)] = X[far]
        nn = torch.linalg.vector_norm(sums, dim=1)
        bad = np.flatnonzero((nn < _EPS).cpu().numpy())
        if len(bad):
            for slot in bad:
                sums[int(slot)] = X[int(rng.integers(n))]
            nn = torch.linalg.vector_norm(sums, dim=1)
        cent = sums / nn[:, None]
    final, _ = argmax_ip(cent)
    final = final.cpu().numpy()
    order = np.argsort(final, kind="stable")
    counts = np.bincount(final, minlength=k)
    lists = [m.tolist() for m in np.split(order, np.cumsum(counts)[:-1])]
    return CoarsePartition(n_lists=k, dim=dim, centroids=cent.cpu().numpy().astype(np.float32),
                           lists=lists)
