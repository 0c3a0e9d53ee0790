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


def train_partition(data, n_lists: int, seed: int, max_iters: int = 25,
                    device: str = "cpu", memberships: bool = True) -> CoarsePartition:
    """Spherical k-means++ / Lloyd on unit rows; f32 centroids + memberships.

    Args:
        data: (n, dim) unit rows; a numpy array, or with device="cuda" also a
            CUDA f64 tensor (the refresh sample never leaves the device).
        device: "cpu" (bit-exact with the reference) or "cuda" (the
            hand-written device k-means, `_train_device`).
        memberships: False skips the final assignment and the per-list id
            lists (refresh re-assigns every vector itself, refresh.py:183-203).
    """
    if n_lists < 1:
        raise ValueError(f"n_lists must be >= 1, got {n_lists}")
    if not isinstance(data, np.ndarray) and hasattr(data, "is_cuda"):
        import torch

        if device != "cuda":
            raise ValueError("a device tensor needs device='cuda'")
        if data.shape[0] < n_lists:
            raise ValueError(f"need at least n_lists={n_lists} rows, got {data.shape[0]}")
        if bool((torch.linalg.vector_norm(data, dim=1) < _EPS).any()):
            raise ValueError("zero-norm row in training data")
        return _train_device(data, n_lists, seed, max_iters, memberships)
    data = np.asarray(data, dtype=np.float64)
    n, dim = data.shape
    if n < n_lists:
        raise ValueError(f"need at least n_lists={n_lists} rows, got {n}")
    if np.any(np.linalg.norm(data, axis=1) < _EPS):
        raise ValueError("zero-norm row in training data")
    if device == "cuda":
        return _train_device(data, n_lists, seed, max_iters, memberships)
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


def _train_device(data, n_lists: int, seed_value: int, max_iters: int,
                  memberships: bool = True) -> CoarsePartition:
    """The same algorithm and RNG call sequence as the host path, as hand-written
    kernels over device-resident rows (csrc/kmeans.cu, csrc/coarse_tc.cu):

    * k-means++ seeding (partition.py:83-113): `ivftq_kmeanspp_seed` runs all
      k steps on the device from the host's uniforms (drawn up front: the
      generator yields the same stream as k-1 calls of rng.random(nc));
    * Lloyd assignment (partition.py:149-150): `ivftq_assign_tc64`, the
      tensor-core pass with the exact f64 guard band on the step's f64
      centroids, ties to the lower list;
    * Lloyd update (partition.py:153-170): `ivftq_kmeans_sums` (stable
      counting sort + in-order f64 sums, bit-identical to np.add.reduceat)
      and `ivftq_normalize_rows` (numpy's pairwise norm, then the division).

    One small read-back per Lloyd step (converged / empty list / zero sum).
    Differences from the host path: the seeding's cdf and candidate scores
    and the assignment's exact scores use a fixed f64 summation order that
    is not OpenBLAS's, so a sample or an arg-max can differ where two values
    agree to the last ulps; everything else is bit-identical. The rare
    branches (fewer distinct points than k, empty lists, zero sums) follow
    the reference through torch glue.
    """
    import torch

    from . import _lib

    L = _lib.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    f64 = torch.float64
    if isinstance(data, np.ndarray):
        X = torch.from_numpy(np.ascontiguousarray(data, dtype=np.float64)).to(dev)
    else:
        X = data.to(device=dev, dtype=f64).contiguous()
    n, dim = X.shape
    k = n_lists
    rng = np.random.default_rng(seed_value)
    sp = _lib.stream_ptr

    if not L.ivftq_coarse_tc_supported(dim, k):
        raise ValueError(f"device k-means needs a padded dim <= 256, got dim={dim}")

    def gemm(A, B):
        out = torch.empty((A.shape[0], B.shape[0]), dtype=f64, device=dev)
        _lib.check(L.ivftq_gemm_nt(A.data_ptr(), B.data_ptr(), _lib.IVFTQ_F64, A.shape[0],
                                   B.shape[0], dim, out.data_ptr(), _lib.IVFTQ_F64, sp()), "gemm_nt")
        return out

    # ---- k-means++ seeding ----
    nc = int(L.ivftq_kmeanspp_candidates(k))
    first = int(rng.integers(n))
    uniforms = np.ascontiguousarray(rng.random((max(k - 1, 0), nc)))
    chosen = torch.empty(k, dtype=torch.int64, device=dev)
    tots = torch.empty(k, dtype=f64, device=dev)
    nbytes = int(L.ivftq_kmeanspp_scratch_bytes(n, dim, k))
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    _lib.check(L.ivftq_kmeanspp_seed(X.data_ptr(), n, dim, k, first,
                                     uniforms.ctypes.data if k > 1 else None, chosen.data_ptr(),
                                     tots.data_ptr(), scratch.data_ptr(), nbytes, sp()),
               "kmeanspp_seed")
    del scratch
    if k > 1 and float(tots[1:].min().item()) <= _EPS:
        # fewer distinct points than k: the reference's checked branch
        # (partition.py:91-98), replayed from the seed with host decisions
        rng = np.random.default_rng(seed_value)
        chosen = _seed_checked(X, k, nc, rng, gemm)
    cent = X[chosen].clone()

    # ---- Lloyd iterations ----
    abytes = int(L.ivftq_assign_tc_scratch_bytes(n, k, dim))
    sbytes = int(L.ivftq_kmeans_sums_scratch_bytes(n, k))
    scratch = torch.empty(max(abytes, sbytes), dtype=torch.uint8, device=dev)
    a = torch.empty(n, dtype=torch.int32, device=dev)
    prev = torch.empty(n, dtype=torch.int32, device=dev)
    sums = torch.empty((k, dim), dtype=f64, device=dev)
    cnt = torch.empty(k, dtype=torch.int32, device=dev)
    flags = torch.zeros(2, dtype=torch.int64, device=dev)  # [assignments differ, first zero-norm sum]
    differ = torch.zeros(1, dtype=torch.int32, device=dev)

    def assign_into(out):
        _lib.check(L.ivftq_assign_tc64(X.data_ptr(), cent.data_ptr(), n, k, dim, out.data_ptr(),
                                       scratch.data_ptr(), scratch.numel(), sp()), "assign_tc64")

    have_prev = False
    for _ in range(max_iters):
        assign_into(a)
        if have_prev:
            _lib.check(L.ivftq_lists_differ(a.data_ptr(), prev.data_ptr(), n, differ.data_ptr(), sp()),
                       "lists_differ")
            if int(differ.item()) == 0:
                break
        prev.copy_(a)
        have_prev = True
        _lib.check(L.ivftq_kmeans_sums(X.data_ptr(), a.data_ptr(), n, dim, k, sums.data_ptr(),
                                       cnt.data_ptr(), scratch.data_ptr(), scratch.numel(), sp()),
                   "kmeans_sums")
        new_cent = torch.empty_like(sums)
        _lib.check(L.ivftq_normalize_rows(sums.data_ptr(), _lib.IVFTQ_F64, k, dim,
                                          new_cent.data_ptr(), flags[1:].data_ptr(), sp()),
                   "normalize_rows")
        flags[0] = cnt.amin()
        min_cnt, bad_row = (int(v) for v in flags.cpu())
        if min_cnt == 0 or bad_row < k:
            # rare branches of partition.py:161-170, in the reference's order
            cnt_h = cnt.cpu().numpy()
            empty = np.flatnonzero(cnt_h == 0)
            if len(empty):
                best = torch.empty(n, dtype=f64, device=dev)
                _lib.check(L.ivftq_rowdot64(X.data_ptr(), cent.data_ptr(), a.data_ptr(), n, dim,
                                          best.data_ptr(), sp()), "rowdot")
                far = torch.argsort(best, stable=True)[: len(empty)]
                sums[torch.as_tensor(empty, device=dev)] = X[far]
            nn = torch.linalg.vector_norm(sums, dim=1)
            for slot in np.flatnonzero((nn < _EPS).cpu().numpy()):
                sums[int(slot)] = X[int(rng.integers(n))]
            _lib.check(L.ivftq_normalize_rows(sums.data_ptr(), _lib.IVFTQ_F64, k, dim,
                                              new_cent.data_ptr(), flags[1:].data_ptr(), sp()),
                       "normalize_rows")
        cent = new_cent
    cent32 = cent.cpu().numpy().astype(np.float32)
    if not memberships:
        return CoarsePartition(n_lists=k, dim=dim, centroids=cent32)
    assign_into(a)
    final = a.cpu().numpy().astype(np.int64)
    order = np.argsort(final, kind="stable")
    counts = np.bincount(final, minlength=k)
    lists = [m.tolist() for m in np.split(order, np.cumsum(counts)[:-1])]
    return CoarsePartition(n_lists=k, dim=dim, centroids=cent32, lists=lists)


def _seed_checked(X, k, nc, rng, gemm):
    """partition.py:_kmeanspp with the degenerate branch (total potential <= eps)
    decided on the host each step; only reached when the data hold fewer
    distinct points than k."""
    import torch

    dev = X.device
    n = X.shape[0]

    def dist2(rows):
        return torch.clamp(2.0 - 2.0 * gemm(X, X[torch.as_tensor(rows, device=dev)]), min=0.0)

    chosen = torch.empty(k, dtype=torch.int64, device=dev)
    c0 = int(rng.integers(n))
    chosen[0] = c0
    d2 = dist2([c0])[:, 0].contiguous()
    for j in range(1, k):
        tot = d2.sum()
        if float(tot.item()) <= _EPS:
            keep = np.ones(n, dtype=bool)
            keep[chosen[:j].cpu().numpy()] = False
            pool = np.flatnonzero(keep)
            cj = int(rng.choice(pool)) if len(pool) else int(rng.integers(n))
            chosen[j] = cj
            d2 = torch.minimum(d2, dist2([cj])[:, 0])
            continue
        cdf = torch.cumsum(d2 / tot, 0)
        cdf /= cdf[-1].clone()
        u = torch.from_numpy(rng.random(nc)).to(dev)
        cand = torch.clamp(torch.searchsorted(cdf, u, right=True), max=n - 1)
        cd2 = torch.clamp(2.0 - 2.0 * gemm(X, X[cand]), min=0.0)
        pot = torch.minimum(d2[:, None], cd2).sum(dim=0)
        bsel = torch.argmin(pot)
        chosen[j] = cand[bsel]
        d2 = torch.minimum(d2, cd2.index_select(1, bsel.reshape(1))[:, 0]).contiguous()
    return chosen
