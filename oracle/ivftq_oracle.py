"""CPU oracle for the IVF-TQ search + ingest hot path.

TEST INFRASTRUCTURE ONLY. This module is a numpy restatement of the
reference `ivftq` package's algorithm (pure Python, /root/reference/pkg/src/
ivftq), written for this repo. Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import it, and
only as the checker or the timed CPU baseline -- never as the product path.
The product (`paper_2605_17415_b200`) never imports it.

Parity pinning: every function is checked against golden vectors produced by
running the reference itself in the build container
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`, test file
`tests/test_oracle_golden.py`). The reference ships no golden files of its
own; its inline known-answer tests (packing KAT 0xA3, quantize KATs, tie
rules) are restated in the same test file.

Arithmetic notes (why this matches the reference bit-for-bit where it must):
  * row norms use `np.linalg.norm(axis=1)` exactly like index.py:241,254,265
    (numpy pairwise summation of squares, then a correctly rounded sqrt);
  * GEMMs are float64 numpy matmuls like index.py:436 and partition.py:53;
  * the residual-term GEMM is float32 like index.py:453.
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "EPS",
    "normalize_rows",
    "assign_max_ip",
    "quantize",
    "encode_batch",
    "pack_fields",
    "unpack_fields",
    "OracleIndex",
    "exact_topk",
    "recall_at_k",
    "reconstruct_all",
    "stratified_sample_ids",
    "train_partition",
    "refresh_encode",
]

EPS = 1e-12  # index.py:38, partition.py:17


def normalize_rows(x: np.ndarray, what: str = "input") -> np.ndarray:
    """f64 cast + unit rows; zero rows rejected by first index.

    Follows index.py:238-245 (and 199-210 for build, 380-389 for queries).
    """
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[None, :]
    nrm = np.linalg.norm(x, axis=1)
    bad = np.nonzero(nrm < EPS)[0]
    if bad.size:
        raise ValueError(f"zero-norm {what} row at index {int(bad[0])}")
    return x / nrm[:, None]


def assign_max_ip(xn: np.ndarray, centroids_f32: np.ndarray):
    """Max inner product list per row; ties -> lowest list (partition.py:45-55)."""
    ips = xn @ np.asarray(centroids_f32, dtype=np.float32).astype(np.float64).T
    ids = ips.argmax(axis=1)
    return ids.astype(np.int64), ips[np.arange(len(xn)), ids]


def quantize(v: np.ndarray, boundaries: np.ndarray, qcent: np.ndarray):
    """Lloyd-Max bin + half-bin sign (lloydmax.py:129-144).

    bin = number of finite interior boundaries <= v (a value on a boundary
    goes to the upper bin), clipped to [0, 2^b - 1]; sign = v >= centroid[bin].
    Restated as a branchless count instead of a binary search.
    """
    v = np.asarray(v, dtype=np.float64)
    interior = np.asarray(boundaries, dtype=np.float64)[1:-1]
    bins = np.zeros(v.shape, dtype=np.int64)
    for b in interior:
        bins += v >= b
    bins = np.clip(bins, 0, len(qcent) - 1)
    signs = (v >= np.asarray(qcent)[bins]).astype(np.uint8)
    return bins.astype(np.uint8), signs


def encode_batch(x, centroids_f32, R, boundaries, qcent, flat=False):
    """Canonical encoder (index.py:231-267).

    Returns (bins u8 (n,d), signs u8 (n,d), list_ids i64, norms f16, xn f64).
    """
    xn = normalize_rows(x)
    n, d = xn.shape
    if flat:
        lids = np.zeros(n, dtype=np.int64)
        resid = xn
    else:
        lids, _ = assign_max_ip(xn, centroids_f32)
        resid = xn - np.asarray(centroids_f32, np.float32)[lids].astype(np.float64)
    rn = np.linalg.norm(resid, axis=1)
    stored = rn.astype(np.float16)  # numpy double->half is round-to-nearest-even
    bins = np.zeros((n, d), dtype=np.uint8)
    signs = np.zeros((n, d), dtype=np.uint8)
    live = stored.astype(np.float64) > 0
    if live.any():
        rot = resid[live] @ np.asarray(R, np.float64).T
        unit = rot / np.linalg.norm(rot, axis=1)[:, None]
        bins[live], signs[live] = quantize(unit, boundaries, qcent)
    return bins, signs, lids, stored, xn


def pack_fields(values: np.ndarray, width: int) -> np.ndarray:
    """Coordinate-major LSB-first bit packing (index.py:104-115).

    Field j's bit p lands at stream bit j*width + p; stream bit t is bit
    (t % 8) of byte t // 8.
    """
    if not 1 <= width <= 8:
        raise ValueError(f"width must be in [1, 8], got {width}")
    v = np.ascontiguousarray(values, dtype=np.uint8)
    n, d = v.shape
    shifts = np.arange(width, dtype=np.uint8)
    bits = (v[:, :, None] >> shifts) & 1  # (n, d, width)
    stream = bits.reshape(n, d * width)
    nbytes = -(-d * width // 8)
    pad = np.zeros((n, nbytes * 8), dtype=np.uint8)
    pad[:, : d * width] = stream
    weights = (1 << np.arange(8)).astype(np.uint16)
    return (pad.reshape(n, nbytes, 8) * weights).sum(axis=2).astype(np.uint8)


def unpack_fields(packed: np.ndarray, width: int, count: int) -> np.ndarray:
    """Inverse of pack_fields (index.py:118-127)."""
    if not 1 <= width <= 8:
        raise ValueError(f"width must be in [1, 8], got {width}")
    p = np.ascontiguousarray(packed, dtype=np.uint8)
    n = p.shape[0]
    bits = (p[:, :, None] >> np.arange(8, dtype=np.uint8)) & 1
    stream = bits.reshape(n, -1)[:, : count * width].reshape(n, count, width)
    return (stream.astype(np.uint16) << np.arange(width)).sum(axis=2).astype(np.uint8)


class _Rows:
    """Append-only rows with capacity doubling (index.py:130-159)."""

    def __init__(self, tail, dtype):
        self._buf = np.zeros((16,) + tuple(tail), dtype)
        self._n = 0

    @property
    def data(self) -> np.ndarray:
        return self._buf[: self._n]

    def extend(self, rows) -> None:
        rows = np.asarray(rows, dtype=self._buf.dtype)
        need = self._n + len(rows)
        if need > len(self._buf):
            cap = len(self._buf)
            while cap < need:
                cap *= 2
            nb = np.zeros((cap,) + self._buf.shape[1:], self._buf.dtype)
            nb[: self._n] = self._buf[: self._n]
            self._buf = nb
        self._buf[self._n: need] = rows
        self._n = need

    def replace(self, rows) -> None:
        self._buf = np.asarray(rows, dtype=self._buf.dtype)
        self._n = len(self._buf)


class OracleIndex:
    """Stored fields of an index plus the reference's search semantics.

    The layout is the reference's per-vector one (index.py:177-185): bins and
    signs (n, d) u8, list ids, binary16 residual norms, optional f32 raw store.
    """

    def __init__(self, centroids_f32, R, boundaries, qcent, half_bin_means,
                 use_sign=True, flat=False, keep_raw=False):
        self.centroids = np.asarray(centroids_f32, dtype=np.float32)
        self.R = np.asarray(R, dtype=np.float64)
        self.boundaries = np.asarray(boundaries, dtype=np.float64)
        self.qcent = np.asarray(qcent, dtype=np.float64)
        self.half = np.asarray(half_bin_means, dtype=np.float64)
        self.use_sign = use_sign
        self.flat = flat
        self.n_lists = len(self.centroids)
        d = self.R.shape[0]
        # append-only row stores with doubling growth, like the reference's
        # _Rows (index.py:130-159): add_batch is amortised O(rows added)
        self._rows = {"bins": _Rows((d,), np.uint8), "signs": _Rows((d,), np.uint8),
                      "list_ids": _Rows((), np.int64), "norms": _Rows((), np.float16)}
        if keep_raw:
            self._rows["raw"] = _Rows((d,), np.float32)
        self._w = None

    bins = property(lambda self: self._rows["bins"].data,
                    lambda self, v: self._rows["bins"].replace(v))
    signs = property(lambda self: self._rows["signs"].data,
                     lambda self, v: self._rows["signs"].replace(v))
    list_ids = property(lambda self: self._rows["list_ids"].data,
                        lambda self, v: self._rows["list_ids"].replace(v))
    norms = property(lambda self: self._rows["norms"].data,
                     lambda self, v: self._rows["norms"].replace(v))

    @property
    def raw(self):
        r = self._rows.get("raw")
        return None if r is None else r.data

    @property
    def count(self) -> int:
        return len(self.list_ids)

    def add_batch(self, x):
        """Encode + append (index.py:286-310); returns internal ids."""
        b, s, l, nr, xn = encode_batch(x, self.centroids, self.R, self.boundaries,
                                       self.qcent, self.flat)
        first = self.count
        self._rows["bins"].extend(b)
        self._rows["signs"].extend(s)
        self._rows["list_ids"].extend(l)
        self._rows["norms"].extend(nr)
        if "raw" in self._rows:
            self._rows["raw"].extend(xn.astype(np.float32))
        self._w = None
        return np.arange(first, first + len(l), dtype=np.int64)

    def members(self):
        """Per-list member ids in ascending id order (partition.lists)."""
        order = np.argsort(self.list_ids, kind="stable")
        counts = np.bincount(self.list_ids, minlength=self.n_lists)
        return np.split(order, np.cumsum(counts)[:-1])

    def scoring_rows(self) -> np.ndarray:
        """f32 rows T[bin,sign] * ||r|| (index.py:366-378)."""
        if self._w is None:
            table = (self.half if self.use_sign else self.qcent).astype(np.float32)
            unit = table[self.bins, self.signs] if self.use_sign else table[self.bins]
            self._w = unit * self.norms.astype(np.float32)[:, None]
        return self._w

    def search_batch(self, queries, k, n_p, rerank_depth=0):
        """List-major search with the reference's ordering (index.py:409-483).

        Scores: coarse <q,c_l> (f64) + f64(f32 residual GEMM); per query the
        top-k by (score desc, internal id asc); pad -1 / -inf.
        """
        if k < 1:
            raise ValueError(f"k must be >= 1, got {k}")
        qn = normalize_rows(queries, "query")
        nq = len(qn)
        w = self.scoring_rows()
        qrot = (qn @ self.R.T).astype(np.float32)
        out_i = np.full((nq, k), -1, np.int64)
        out_s = np.full((nq, k), -np.inf, np.float64)
        if self.flat:
            sc = (w @ qrot.T).T.astype(np.float64)
            n = sc.shape[1]
            kk = min(k, n)
            ids = np.arange(n, dtype=np.int64)
            for qi in range(nq):
                top = np.lexsort((ids, -sc[qi]))[:kk]
                out_i[qi, :kk] = top
                out_s[qi, :kk] = sc[qi, top]
            return out_i, out_s
        n_p = min(n_p, self.n_lists)
        coarse = qn @ self.centroids.astype(np.float64).T
        probe = np.argsort(-coarse, axis=1, kind="stable")[:, :n_p]
        groups: dict[int, list[int]] = {}
        for qi in range(nq):
            for l in probe[qi]:
                groups.setdefault(int(l), []).append(qi)
        mem = self.members()
        cand_i = [[] for _ in range(nq)]
        cand_s = [[] for _ in range(nq)]
        for l, qis in groups.items():
            m = mem[l]
            if m.size == 0:
                continue
            blk = w[m] @ qrot[qis].T
            for c, qi in enumerate(qis):
                cand_i[qi].append(m)
                cand_s[qi].append(coarse[qi, l] + blk[:, c].astype(np.float64))
        depth = max(k, rerank_depth) if rerank_depth > 0 else k
        for qi in range(nq):
            if not cand_i[qi]:
                continue
            ids = np.concatenate(cand_i[qi])
            sc = np.concatenate(cand_s[qi])
            pos = np.lexsort((ids, -sc))[:depth]
            sel, est = ids[pos], sc[pos]
            if rerank_depth > 0:
                ex = self.raw[sel].astype(np.float64) @ qn[qi]
                o = np.lexsort((sel, -ex))[:k]
                sel, est = sel[o], ex[o]
            else:
                sel, est = sel[:k], est[:k]
            out_i[qi, : len(sel)] = sel
            out_s[qi, : len(sel)] = est
        return out_i, out_s

    def probes(self, queries, n_p):
        """Probe lists + coarse scores (index.py:434-438)."""
        qn = normalize_rows(queries, "query")
        coarse = qn @ self.centroids.astype(np.float64).T
        probe = np.argsort(-coarse, axis=1, kind="stable")[:, :n_p]
        return probe, np.take_along_axis(coarse, probe, axis=1)


def exact_topk(database, queries, k, chunk=256):
    """Brute-force IP top-k, ties -> lower id (evaluation.py:57-79)."""
    db = np.asarray(database, dtype=np.float64)
    q = np.asarray(queries, dtype=np.float64)
    kk = min(k, len(db))
    out = np.empty((len(q), kk), np.int64)
    for s in range(0, len(q), chunk):
        sc = q[s : s + chunk] @ db.T
        out[s : s + chunk] = np.argsort(-sc, axis=1, kind="stable")[:, :kk]
    return out


def recall_at_k(results, truth, k):
    """Mean |top-k ∩ truth-k| / k (evaluation.py:82-98)."""
    res = np.asarray(results)
    tr = np.asarray(truth)
    hits = [len(np.intersect1d(res[i][:k], tr[i][:k])) / k for i in range(len(res))]
    return float(np.mean(hits))


def reconstruct_all(idx: OracleIndex, renormalize=True):
    """Decode c_l + ||r|| * R^T T[code] (refresh.py:63-81)."""
    table = idx.half if idx.use_sign else idx.qcent
    unit = table[idx.bins, idx.signs] if idx.use_sign else table[idx.bins]
    back = unit @ idx.R
    rec = idx.norms.astype(np.float64)[:, None] * back
    if not idx.flat:
        rec = rec + idx.centroids[idx.list_ids].astype(np.float64)
    if renormalize:
        nr = np.linalg.norm(rec, axis=1)
        rec = rec / np.maximum(nr, 1e-12)[:, None]
    return rec


def stratified_sample_ids(list_members, n, n_lists, sample_size, rng):
    """Proportional per-list sample, floor 1 (refresh.py:109-131)."""
    picked = []
    for m in list_members:
        if len(m) == 0:
            continue
        take = min(max(1, int(np.ceil(sample_size * len(m) / n))), len(m))
        picked.append(rng.choice(np.asarray(m, np.int64), size=take, replace=False))
    ids = np.concatenate(picked)
    if len(ids) < n_lists:
        rest = np.setdiff1d(np.arange(n, dtype=np.int64), ids)
        extra = n_lists - len(ids)
        ids = np.concatenate(
            [ids, rng.choice(rest, size=min(extra, len(rest)), replace=False)])
    return np.sort(ids)


def _kmeanspp(data, k, rng):
    """Greedy k-means++ on the sphere (partition.py:64-95)."""
    n = len(data)
    ncand = 2 + int(np.log2(k)) if k > 1 else 1
    chosen = np.empty(k, np.int64)
    chosen[0] = rng.integers(n)
    d2 = np.maximum(2.0 - 2.0 * (data @ data[chosen[0]]), 0.0)
    for j in range(1, k):
        tot = d2.sum()
        if tot <= EPS:
            mask = np.ones(n, bool)
            mask[chosen[:j]] = False
            pool = np.nonzero(mask)[0]
            chosen[j] = rng.choice(pool) if len(pool) else rng.integers(n)
            d2 = np.minimum(d2, np.maximum(2.0 - 2.0 * (data @ data[chosen[j]]), 0.0))
            continue
        cand = rng.choice(n, size=ncand, p=d2 / tot)
        cd2 = np.maximum(2.0 - 2.0 * (data @ data[cand].T), 0.0)
        pot = np.minimum(d2[:, None], cd2).sum(axis=0)
        b = int(np.argmin(pot))
        chosen[j] = cand[b]
        d2 = np.minimum(d2, cd2[:, b])
    return data[chosen].copy()


def train_partition(data, n_lists, seed, max_iters=25):
    """Spherical k-means; returns f32 centroids (partition.py:98-178)."""
    data = np.asarray(data, dtype=np.float64)
    n, d = data.shape
    if n < n_lists:
        raise ValueError(f"need at least n_lists={n_lists} rows, got {n}")
    rng = np.random.default_rng(seed)
    cent = _kmeanspp(data, n_lists, rng)
    prev = None
    for _ in range(max_iters):
        ips = data @ cent.T
        a = ips.argmax(axis=1)
        if prev is not None and np.array_equal(a, prev):
            break
        prev = a
        cnt = np.bincount(a, minlength=n_lists)
        order = np.argsort(a, kind="stable")
        starts = np.concatenate(([0], np.cumsum(cnt)[:-1]))
        ne = np.nonzero(cnt > 0)[0]
        sums = np.zeros((n_lists, d))
        sums[ne] = np.add.reduceat(data[order], starts[ne], axis=0)
        empty = np.nonzero(cnt == 0)[0]
        if empty.size:
            worst = np.argsort(ips[np.arange(n), a], kind="stable")
            for slot, p in zip(empty, worst[: len(empty)]):
                sums[slot] = data[p]
                cnt[slot] = 1
        nn = np.linalg.norm(sums, axis=1)
        deg = nn < EPS
        if deg.any():
            for slot in np.nonzero(deg)[0]:
                sums[slot] = data[rng.integers(n)]
            nn = np.linalg.norm(sums, axis=1)
        cent = sums / nn[:, None]
    return cent.astype(np.float32)


def refresh_encode(idx: OracleIndex, source: np.ndarray, new_centroids_f32):
    """Re-encode every vector against new centroids and swap (refresh.py:183-203)."""
    b, s, l, nr, _ = encode_batch(source, new_centroids_f32, idx.R, idx.boundaries,
                                  idx.qcent)
    idx.centroids = np.asarray(new_centroids_f32, np.float32)
    idx.bins, idx.signs, idx.list_ids, idx.norms = b, s, l, nr
    idx._w = None
    return idx
