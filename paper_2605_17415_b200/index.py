"""IVF-TQ index with a B200-resident hot path (drop-in for ivftq.index).

Mirrors the reference API (index.py:41-630): `IndexConfig`, `VectorCode`,
`SearchResult`, `IvfTqIndex.build/encode/add/add_batch/search/search_batch`,
the read-only views, `compression_fingerprint`, flat mode, `bit_accounting`
and `bit_flip_ablation`, with the same validation order, error types and
messages. Every numeric stage of ingest and search runs in the CUDA library
(libivftq_b200.so) through its C ABI; this module only validates, moves
buffers and sequences calls. There is no CPU fallback: without a GPU or the
built library the compute methods raise.
"""

from __future__ import annotations

import ctypes as C
import gc
import hashlib
import os
import threading
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .partition import CoarsePartition, train_partition
from .quantizer import ScalarQuantizer, design_quantizer
from .rotation import RotationMatrix, generate_rotation
from .store import DeviceStore

__all__ = [
    "IndexConfig", "VectorCode", "SearchResult", "IvfTqIndex", "build", "search_flat_tq",
    "bit_accounting", "bit_flip_ablation", "pack_fields", "unpack_fields",
]

_EPS = 1e-12


@dataclass(frozen=True)
class IndexConfig:
    """Build-time parameters (index.py:41-75); same defaults and validation."""

    dim: int
    bits: int
    n_lists: int
    use_sign_bit: bool = True
    keep_raw: bool = False
    flat: bool = False
    rotation_seed: int = 42
    kmeans_seed: int = 42

    def __post_init__(self):
        if self.dim < 2:
            raise ValueError(f"dim must be >= 2, got {self.dim}")
        if not 1 <= self.bits <= 8:
            raise ValueError(f"bits must be in [1, 8], got {self.bits}")
        if self.n_lists < 1:
            raise ValueError(f"n_lists must be >= 1, got {self.n_lists}")
        if self.flat and self.n_lists != 1:
            raise ValueError("flat mode requires n_lists == 1")


@dataclass(frozen=True)
class VectorCode:
    """Packed per-vector record (index.py:78-93)."""

    codes: bytes
    signs: bytes
    list_id: int
    residual_norm: np.float16


@dataclass(frozen=True)
class SearchResult:
    ids: np.ndarray
    scores: np.ndarray


def pack_fields(values: np.ndarray, width: int) -> np.ndarray:
    """(n, d) u8 fields -> coordinate-major LSB-first bytes (index.py:104-115)."""
    if not 1 <= width <= 8:
        raise ValueError(f"width must be in [1, 8], got {width}")
    v = np.ascontiguousarray(values, dtype=np.uint8)
    n, d = v.shape
    bits = (v[:, :, None] >> np.arange(width, dtype=np.uint8)) & 1
    return np.packbits(bits.reshape(n, d * width), axis=1, bitorder="little")


def unpack_fields(packed: np.ndarray, width: int, count: int) -> np.ndarray:
    """Inverse of pack_fields (index.py:118-127)."""
    if not 1 <= width <= 8:
        raise ValueError(f"width must be in [1, 8], got {width}")
    p = np.ascontiguousarray(packed, dtype=np.uint8)
    n = p.shape[0]
    bits = np.unpackbits(p, axis=1, count=count * width, bitorder="little")
    bits = bits.reshape(n, count, width).astype(np.uint16)
    return (bits << np.arange(width, dtype=np.uint16)).sum(axis=2).astype(np.uint8)


class _Grow:
    """Grow-only device buffer indexed by internal id."""

    def __init__(self, shape_tail, dtype, device, fill=0):
        self.tail, self.dtype, self.device, self.fill = tuple(shape_tail), dtype, device, fill
        self.t = torch.full((1024, *self.tail), fill, dtype=dtype, device=device)

    def ensure(self, n: int):
        if n <= self.t.shape[0]:
            return
        cap = max(n, 2 * self.t.shape[0])
        g = torch.full((cap, *self.tail), self.fill, dtype=self.dtype, device=self.device)
        g[: self.t.shape[0]] = self.t
        self.t = g


def _to_device_rows(x, dim_expected: int | None, dev, what="input"):
    """Host/torch rows -> (device tensor f32/f64 contiguous, dtype code)."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.dtype not in (torch.float32, torch.float64):
            t = t.double()
        t = t.to(dev, non_blocking=True).contiguous()
    else:
        a = np.asarray(x)
        if a.dtype not in (np.float32, np.float64):
            a = a.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    code = _lib.IVFTQ_F32 if t.dtype == torch.float32 else _lib.IVFTQ_F64
    return t, code


class IvfTqIndex:
    """Trained coarse partition over the fixed compression layer, on one GPU.

    `scan_mode` selects the list-scan kernel: "auto" (tensor-core list-major
    scan for batches, LUT scan otherwise), "tc" or "lut".
    """

    scan_mode = "auto"

    def __init__(self, config: IndexConfig, quantizer: ScalarQuantizer, rot: RotationMatrix,
                 partition: CoarsePartition, device=None):
        self.config = config
        self.quantizer = quantizer
        self.rot = rot
        self.partition = partition
        self._lib = _lib.lib()
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        d = config.dim
        dev = self.device
        self._R = torch.from_numpy(np.array(rot.matrix, np.float64)).to(dev)
        self._RT = torch.from_numpy(np.array(rot.matrix.T, np.float64, order="C")).to(dev)
        self._bnd = torch.from_numpy(np.array(quantizer.boundaries, np.float64)).to(dev)
        self._qcent = torch.from_numpy(np.array(quantizer.centroids, np.float64)).to(dev)
        self._levels = torch.from_numpy(np.array(quantizer.levels(config.use_sign_bit), order="C")).to(dev)
        self._store = DeviceStore(d, config.bits, config.use_sign_bit, partition.n_lists, dev)
        self._slot_of = _Grow((), torch.int64, dev, -1)
        self._list_of = _Grow((), torch.int32, dev, 0)
        self._norm_of = _Grow((), torch.int16, dev, 0)
        self._raw = _Grow((d,), torch.float32, dev) if config.keep_raw else None
        self._ext = None  # external ids; None while every one equals its internal id
        self._count = 0
        self._version = 0
        self._host_cache: dict = {}
        self._set_partition(partition)

    # ------------------------------------------------------------------
    # construction

    @classmethod
    def build(cls, config: IndexConfig, training_data: np.ndarray,
              kmeans_device: str = "cpu") -> "IvfTqIndex":
        """Normalise, train the partition, fix the compression layer, add all rows
        (index.py:190-226)."""
        data = np.asarray(training_data, dtype=np.float64)
        if data.ndim != 2 or data.shape[1] != config.dim:
            raise ValueError(f"training data must be (n, {config.dim})")
        norms = np.linalg.norm(data, axis=1)
        bad = np.flatnonzero(norms < _EPS)
        if len(bad):
            raise ValueError(f"zero-norm training row at index {bad[0]}")
        if data.shape[0] < config.n_lists:
            raise ValueError(f"need at least n_lists={config.n_lists} rows, got {data.shape[0]}")
        normalized = data / norms[:, None]
        quantizer = design_quantizer(config.bits, config.dim)
        rot = generate_rotation(config.dim, config.rotation_seed)
        if config.flat:
            ph = np.zeros((1, config.dim), dtype=np.float32)
            ph[0, 0] = 1.0
            partition = CoarsePartition(n_lists=1, dim=config.dim, centroids=ph)
        else:
            partition = train_partition(normalized, config.n_lists, seed=config.kmeans_seed,
                                        device=kmeans_device)
            partition.lists = [[] for _ in range(config.n_lists)]
        index = cls(config, quantizer, rot, partition)
        index.add_batch(normalized)
        return index

    def _set_partition(self, partition: CoarsePartition):
        self.partition = partition
        self._cent = torch.from_numpy(np.ascontiguousarray(partition.centroids, np.float32)).to(
            self.device)
        partition._attach(self._members_view)

    # ------------------------------------------------------------------
    # encoding

    def _encode_device(self, x, partition: CoarsePartition | None = None, what="input",
                       defer_check=False):
        """Run the fused device encoder; returns device (words, lids, norms16, xn).
        With defer_check the zero-row flag (first bad row index, n if none) is
        returned as a device scalar as a fifth element instead of being read
        here, so a caller pipelining several batches syncs once."""
        cfg = self.config
        cent = self._cent if partition is None else torch.from_numpy(
            np.ascontiguousarray(partition.centroids, np.float32)).to(self.device)
        if isinstance(x, torch.Tensor):
            shape = tuple(x.shape)
        else:
            x = np.asarray(x)
            if x.dtype not in (np.float32, np.float64):
                x = x.astype(np.float64)
            shape = x.shape
        if len(shape) != 2 or shape[1] != cfg.dim:
            raise ValueError(f"expected (n, {cfg.dim}) input, got {shape}")
        xt, code = _to_device_rows(x, cfg.dim, self.device)
        n, d = shape
        W = self._store.words_per_vec
        dev = self.device
        xn = torch.empty((n, d), dtype=torch.float64, device=dev)
        bad = torch.empty(1, dtype=torch.int64, device=dev)
        lids = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        nrm = torch.empty(max(n, 1), dtype=torch.int16, device=dev)
        words = torch.empty((max(n, 1), W), dtype=torch.int32, device=dev)
        sb = self._lib.ivftq_encode_scratch_bytes(n, d, self.partition.n_lists)
        scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
        _lib.check(self._lib.ivftq_encode(
            xt.data_ptr(), code, n, d, cfg.bits, int(cfg.use_sign_bit), int(cfg.flat),
            cent.data_ptr(), cent.shape[0], self._R.data_ptr(), self._bnd.data_ptr(),
            self._qcent.data_ptr(), xn.data_ptr(), bad.data_ptr(), lids.data_ptr(),
            nrm.data_ptr(), words.data_ptr(), scratch.data_ptr(), sb, _lib.stream_ptr()),
            "encode")
        if defer_check:
            return words[:n], lids[:n], nrm[:n], xn, bad
        b = int(bad.item())
        if b < n:
            raise ValueError(f"zero-norm {what} row at index {b}")
        return words[:n], lids[:n], nrm[:n], xn

    def _unpack_words(self, words: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """Host unpack of device code words (n, W) -> bins, signs (n, d) u8."""
        s = self._store
        d = self.config.dim
        w = words.view(np.uint32)
        n = w.shape[0]
        f = np.arange(d)
        word_idx, fld = f // s.fields_per_word, f % s.fields_per_word
        vals = (w[:, word_idx] >> (s.field_bits * fld).astype(np.uint32)) & ((1 << s.field_bits) - 1)
        return (vals >> 1).astype(np.uint8), (vals & 1).astype(np.uint8)

    def _encode_batch(self, x: np.ndarray, partition: CoarsePartition | None = None):
        """Host-visible encode (index.py:231-267): (bins, signs, list_ids, f16 norms, xn)."""
        words, lids, nrm, xn = self._encode_device(x, partition)
        bins, signs = self._unpack_words(words.cpu().numpy())
        return (bins, signs, lids.cpu().numpy().astype(np.int64),
                nrm.cpu().numpy().view(np.float16), xn.cpu().numpy())

    def encode(self, x: np.ndarray) -> VectorCode:
        """Encode one vector to its packed record without adding it (index.py:269-279)."""
        bins, signs, lids, stored, _ = self._encode_batch(np.asarray(x, dtype=np.float64)[None, :])
        return VectorCode(codes=pack_fields(bins, self.config.bits).tobytes(),
                          signs=pack_fields(signs, 1).tobytes(), list_id=int(lids[0]),
                          residual_norm=stored[0])

    def add(self, x: np.ndarray, external_id: int | None = None) -> int:
        ext = None if external_id is None else np.asarray([external_id], dtype=np.int64)
        return int(self.add_batch(np.asarray(x, dtype=np.float64)[None, :], ext)[0])

    _QUERY_CHUNK = 1 << 16  # queries per search call (scratch bound)
    _PIPE_ROWS = 1 << 17  # host->device sub-chunk of a large host batch (measured best at C2)

    def _encode_host_pipelined(self, x: torch.Tensor):
        """Encode a large host (ideally pinned) batch in sub-chunks, copying
        sub-chunk j+1 on a side stream while sub-chunk j encodes. Nothing is
        appended here, so a bad row anywhere still leaves the index untouched."""
        dev = self.device
        n, d = x.shape
        sub = self._PIPE_ROWS
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = torch.cuda.Stream(device=dev)
        cs = self._copy_stream
        cur = torch.cuda.current_stream(dev)
        bufs = [torch.empty((sub, d), dtype=x.dtype, device=dev) for _ in range(2)]
        copied = [torch.cuda.Event() for _ in range(2)]
        freed = [torch.cuda.Event() for _ in range(2)]
        spans = [(s, min(n, s + sub)) for s in range(0, n, sub)]

        def issue(j):
            s, e = spans[j]
            b = j % 2
            with torch.cuda.stream(cs):
                if j >= 2:
                    cs.wait_event(freed[b])
                bufs[b][: e - s].copy_(x[s:e], non_blocking=True)
                copied[b].record(cs)

        issue(0)
        if len(spans) > 1:
            issue(1)
        parts = []
        flags = []
        keep_xn = self._raw is not None
        for j, (s, e) in enumerate(spans):
            b = j % 2
            cur.wait_event(copied[b])
            words, lids, nrm, xn, bad = self._encode_device(bufs[b][: e - s], defer_check=True)
            freed[b].record(cur)
            if j + 2 < len(spans):
                issue(j + 2)
            parts.append((words, lids, nrm, xn if keep_xn else None))
            flags.append(bad)
        # one sync for the whole batch: the first zero row, with its batch-wide index
        bad = torch.cat(flags).cpu().numpy()
        for (s, e), bi in zip(spans, bad):
            if bi < e - s:
                raise ValueError(f"zero-norm input row at index {s + int(bi)}")
        words = torch.cat([p[0] for p in parts])
        lids = torch.cat([p[1] for p in parts])
        nrm = torch.cat([p[2] for p in parts])
        xn = torch.cat([p[3] for p in parts]) if keep_xn else None
        return words, lids, nrm, xn

    def add_batch(self, x, external_ids: np.ndarray | None = None) -> np.ndarray:
        """Encode and append rows; returns internal ids (index.py:286-310)."""
        if (isinstance(x, np.ndarray) and x.ndim == 2 and x.dtype in (np.float32, np.float64)
                and x.shape[0] > 2 * self._PIPE_ROWS):
            x = torch.from_numpy(np.ascontiguousarray(x))  # host batch: bounded sub-chunks
        if (isinstance(x, torch.Tensor) and x.device.type == "cpu" and x.dim() == 2
                and x.shape[1] == self.config.dim and x.shape[0] > 2 * self._PIPE_ROWS
                and x.dtype in (torch.float32, torch.float64)):
            words, lids, nrm, xn = self._encode_host_pipelined(x)
        else:
            words, lids, nrm, xn = self._encode_device(x)
        n = words.shape[0]
        if external_ids is not None:
            external_ids = np.asarray(external_ids, dtype=np.int64)
            if len(external_ids) != n:
                raise ValueError("external_ids length mismatch")
        self._append_encoded(words, lids, nrm, xn)
        first = self._count - n
        # external ids default to the internal ones (index.py:299-303); while
        # every id so far is a default, none is stored (_ext is None)
        if external_ids is not None and self._ext is None:
            self._ext = np.arange(max(self._count, 1024), dtype=np.int64)
        if self._ext is not None:
            if len(self._ext) < self._count:
                g = np.zeros(max(self._count, 2 * len(self._ext)), dtype=np.int64)
                g[:first] = self._ext[:first]
                self._ext = g
            self._ext[first:self._count] = (np.arange(first, self._count, dtype=np.int64)
                                            if external_ids is None else external_ids)
        return np.arange(first, first + n, dtype=np.int64)

    def _append_encoded(self, words, lids, nrm, xn):
        n = words.shape[0]
        if n == 0:
            self._version += 1
            return
        L = self.partition.n_lists
        dev = self.device
        counts = torch.empty(L, dtype=torch.int32, device=dev)
        _lib.check(self._lib.ivftq_histogram(lids.data_ptr(), n, L, counts.data_ptr(),
                                             _lib.stream_ptr()), "histogram")
        inc = counts.cpu().numpy().astype(np.int64)
        first = self._count
        for g in (self._slot_of, self._list_of, self._norm_of):
            g.ensure(first + n)
        st = self._store
        st.reserve(inc, self._slot_of.t)
        cursor = torch.empty(L, dtype=torch.int32, device=dev)
        _lib.check(self._lib.ivftq_append(C.byref(st.struct()), words.data_ptr(), nrm.data_ptr(),
                                          lids.data_ptr(), n, first, cursor.data_ptr(),
                                          self._slot_of.t.data_ptr(), _lib.stream_ptr()), "append")
        st.set_sizes(st.sizes + inc)
        self._list_of.t[first:first + n] = lids
        self._norm_of.t[first:first + n] = nrm
        if self._raw is not None:
            self._raw.ensure(first + n)
            self._raw.t[first:first + n] = xn.to(torch.float32)
        self._count += n
        self._version += 1

    # ------------------------------------------------------------------
    # read-only views (index.py:315-346); materialised lazily per state

    def _cached(self, key, fn):
        ent = self._host_cache.get(key)
        if ent is not None and ent[0] == self._version:
            return ent[1]
        val = fn()
        self._host_cache[key] = (self._version, val)
        return val

    @property
    def count(self) -> int:
        return self._count

    def _export(self):
        n = self._count
        d = self.config.dim
        bins = torch.empty((max(n, 1), d), dtype=torch.uint8, device=self.device)
        signs = torch.empty((max(n, 1), d), dtype=torch.uint8, device=self.device)
        if n:
            _lib.check(self._lib.ivftq_export_codes(
                C.byref(self._store.struct()), self._slot_of.t.data_ptr(), 0, n,
                bins.data_ptr(), signs.data_ptr(), _lib.stream_ptr()), "export_codes")
        return bins[:n].cpu().numpy(), signs[:n].cpu().numpy()

    @property
    def bins(self) -> np.ndarray:
        return self._cached("codes", self._export)[0]

    @property
    def signs(self) -> np.ndarray:
        return self._cached("codes", self._export)[1]

    @property
    def list_ids(self) -> np.ndarray:
        return self._cached("lids", lambda: self._list_of.t[: self._count].cpu().numpy().astype(
            np.int64))

    @property
    def norms(self) -> np.ndarray:
        return self._cached("norms", lambda: self._norm_of.t[: self._count].cpu().numpy().view(
            np.float16))

    @property
    def external_ids(self) -> np.ndarray:
        if self._ext is None:
            return np.arange(self._count, dtype=np.int64)
        return self._ext[: self._count]

    @property
    def raw(self) -> np.ndarray | None:
        if self._raw is None:
            return None
        return self._cached("raw", lambda: self._raw.t[: self._count].cpu().numpy())

    def _members_view(self):
        def make():
            lids = self.list_ids
            order = np.argsort(lids, kind="stable")
            counts = np.bincount(lids, minlength=self.partition.n_lists)
            return [m.tolist() for m in np.split(order, np.cumsum(counts)[:-1])]
        return self._cached("members", make)

    @property
    def state_tag(self) -> str:
        return f"n={self.count}/v={self._version}"

    def compression_fingerprint(self) -> str:
        """SHA-256 over quantizer tables and rotation (index.py:348-361)."""
        h = hashlib.sha256()
        for a in (self.quantizer.boundaries, self.quantizer.centroids,
                  self.quantizer.half_bin_means, self.rot.matrix):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()

    # ------------------------------------------------------------------
    # search

    def _normalize_queries_device(self, q):
        cfg = self.config
        if isinstance(q, torch.Tensor):
            shape = tuple(q.shape)
        else:
            q = np.asarray(q)
            shape = q.shape
        if len(shape) == 1:
            q = q[None, :]
            shape = (1, shape[0])
        if shape[1] != cfg.dim:
            raise ValueError(f"query dim {shape[1]} != index dim {cfg.dim}")
        qt, code = _to_device_rows(q, cfg.dim, self.device)
        nq = shape[0]
        qn = torch.empty((nq, cfg.dim), dtype=torch.float64, device=self.device)
        bad = torch.empty(1, dtype=torch.int64, device=self.device)
        _lib.check(self._lib.ivftq_normalize_rows(qt.data_ptr(), code, nq, cfg.dim, qn.data_ptr(),
                                                  bad.data_ptr(), _lib.stream_ptr()),
                   "normalize_rows")
        return qn, bad, nq

    def search(self, q: np.ndarray, k: int, n_p: int, rerank_depth: int = 0) -> SearchResult:
        ids, scores = self.search_batch(np.asarray(q, dtype=np.float64)[None, :], k, n_p,
                                        rerank_depth)
        return SearchResult(ids=ids[0], scores=scores[0])

    def search_batch(self, queries, k: int, n_p: int, rerank_depth: int = 0,
                     return_device: bool = False):
        """Probe n_p lists per query and return the top-k (index.py:409-478).

        Returns (ids int64 (nq, k), scores float64 (nq, k)), score-descending
        with ties to the lower internal id, padded with -1 / -inf.
        """
        if k < 1:
            raise ValueError(f"k must be >= 1, got {k}")
        if self.config.flat:
            return self._search_flat_batch(queries, k, return_device)
        if n_p < 1:
            raise ValueError(f"n_p must be >= 1, got {n_p}")
        if n_p > self.config.n_lists:
            warnings.warn(f"n_p={n_p} exceeds n_lists={self.config.n_lists}; clamping",
                          stacklevel=2)
            n_p = self.config.n_lists
        if rerank_depth > 0 and self._raw is None:
            raise ValueError("rerank requires an index built with keep_raw=True")
        nq_all = (queries.shape[0] if isinstance(queries, torch.Tensor) and queries.dim() == 2
                  else np.shape(queries)[0] if np.ndim(queries) == 2 else 1)
        if nq_all > self._QUERY_CHUNK:
            # bound the per-call scratch (probe scores, pairs, candidate buffers
            # grow with nq): search in chunks, results in order
            parts = [self.search_batch(queries[s:s + self._QUERY_CHUNK], k, n_p, rerank_depth,
                                       return_device=True)
                     for s in range(0, nq_all, self._QUERY_CHUNK)]
            ids = torch.cat([p[0] for p in parts])
            scores = torch.cat([p[1] for p in parts])
            if return_device:
                return ids, scores
            return ids.cpu().numpy(), scores.cpu().numpy()
        depth = max(k, rerank_depth) if rerank_depth > 0 else k
        if self._graph_eligible(queries):
            if isinstance(queries, np.ndarray):
                queries = torch.from_numpy(np.ascontiguousarray(queries))
            try:
                ids, scores, bad = self._search_graphed(queries, k, n_p, depth, rerank_depth)
            except (RuntimeError, _lib.IvftqError) as err:  # capture refused: run eagerly
                if "captur" not in str(err):
                    raise
                warnings.warn(f"CUDA graph capture failed ({err}); searching without graphs",
                              stacklevel=2)
                self.use_graphs = False
                torch.cuda.synchronize(self.device)
            else:
                nq = queries.shape[0]
                if return_device:  # the graph's outputs are overwritten by its next replay
                    ids, scores = ids.clone(), scores.clone()
                return self._finish(ids, scores, bad, nq, return_device)
        ids, scores, bad, nq = self._search_core(queries, k, n_p, depth, rerank_depth)
        return self._finish(ids, scores, bad, nq, return_device)

    # Repeated searches of one shape replay a CUDA graph of the whole device
    # sequence (normalize, probe, rotate, regroup, seed, scan, merge): one
    # launch instead of ~30, no host work between kernels. Graphs are keyed by
    # (rows, dtype, k, n_p, depth, rerank) and dropped whenever the index
    # changes (they hold its buffer pointers).
    use_graphs = os.environ.get("IVFTQ_NO_GRAPH", "") != "1"
    _MAX_GRAPHS = 8

    def _graph_eligible(self, queries) -> bool:
        if isinstance(queries, np.ndarray) and queries.dtype in (np.float32, np.float64):
            queries = torch.from_numpy(queries)  # a view; copied into the graph input
        return (self.use_graphs and isinstance(queries, torch.Tensor) and queries.dim() == 2
                and queries.dtype in (torch.float32, torch.float64)
                and queries.shape[1] == self.config.dim
                and 1 <= queries.shape[0] <= self._QUERY_CHUNK)

    def _search_graphed(self, queries, k, n_p, depth, rerank_depth):
        # Graphs are per host thread: a replay overwrites its static input and
        # output buffers, so concurrent readers of one index
        # must never share one.
        tls = self._thread_state()
        if getattr(tls, "graph_version", None) != self._version:
            tls.graphs = {}
            tls.graph_version = self._version
        graphs = tls.graphs
        key = (tuple(queries.shape), queries.dtype, k, n_p, depth, rerank_depth, self.scan_mode,
               self._lib.ivftq_get_kernel_timing())
        ent = graphs.pop(key, None)
        if ent is not None:
            graphs[key] = ent  # most recently used last
            ent[1].copy_(queries, non_blocking=True)
        else:
            while len(graphs) >= self._MAX_GRAPHS:  # bound the graphs' memory pools
                graphs.pop(next(iter(graphs)))
            static_in = torch.empty(queries.shape, dtype=queries.dtype, device=self.device)
            static_in.copy_(queries)
            # warm-up outside capture: library lazy state, allocator pools
            self._search_core(static_in, k, n_p, depth, rerank_depth)
            torch.cuda.synchronize(self.device)
            g = torch.cuda.CUDAGraph()
            c0 = self._lib.ivftq_launch_count()
            # no garbage collection inside the capture: a collected pinned
            # buffer would record a CUDA event on the capturing stream
            gc_on = gc.isenabled()
            gc.disable()
            try:
                # a per-thread capture stream: torch's default capture stream
                # is shared by every thread
                if getattr(tls, "capture_stream", None) is None:
                    tls.capture_stream = torch.cuda.Stream(device=self.device)
                with torch.cuda.graph(g, stream=tls.capture_stream,
                                      capture_error_mode="thread_local"):
                    out = self._search_core(static_in, k, n_p, depth, rerank_depth)[:3]
            finally:
                if gc_on:
                    gc.enable()
            ent = (g, static_in, out, self._lib.ivftq_launch_count() - c0)
            graphs[key] = ent
        g, _, out, n_launch = ent
        g.replay()
        self._lib.ivftq_note_graph_launches(n_launch)
        return out

    def _thread_state(self):
        """Per-host-thread search state (side stream, graph cache)."""
        tls = self.__dict__.get("_tls")
        if tls is None:
            tls = self.__dict__.setdefault("_tls", threading.local())
        return tls

    def _search_core(self, queries, k, n_p, depth, rerank_depth):
        """The device sequence of one search (no host synchronisation)."""
        qn, bad, nq = self._normalize_queries_device(queries)
        dev = self.device
        d = self.config.dim
        # the query rotation depends only on qn: it runs on a side stream
        # while the probe kernels run on the current one
        qrot = torch.empty((max(nq, 1), d), dtype=torch.float32, device=dev)
        cur = torch.cuda.current_stream(dev)
        tls = self._thread_state()
        if getattr(tls, "side_stream", None) is None:
            tls.side_stream = torch.cuda.Stream(device=dev)
        side = tls.side_stream
        forked, rotated = torch.cuda.Event(), torch.cuda.Event()
        forked.record(cur)
        side.wait_event(forked)
        with torch.cuda.stream(side):
            self._rotate(qn, nq, qrot)
            rotated.record(side)
        probe, coarse = self._probe(qn, nq, n_p)
        cur.wait_event(rotated)
        ids, scores = self._scan(qn, nq, probe, coarse, n_p, depth, qrot)
        if rerank_depth > 0:
            ids, scores = self._rerank(qn, nq, ids, depth, k)
        return ids, scores, bad, nq

    def _probe(self, qn, nq, n_p):
        """Top-n_p lists per query and their f64 coarse scores (index.py:434-438)."""
        L = self.partition.n_lists
        d = self.config.dim
        probe = torch.empty((max(nq, 1), n_p), dtype=torch.int32, device=self.device)
        coarse = torch.empty((max(nq, 1), n_p), dtype=torch.float64, device=self.device)
        pb = self._lib.ivftq_probe_scratch_bytes(nq, L, d)
        pscr = torch.empty(pb, dtype=torch.uint8, device=self.device)
        _lib.check(self._lib.ivftq_probe_prepared(
            qn.data_ptr(), self._cent.data_ptr(), self._coarse_prep().data_ptr(), nq, L, d, n_p,
            probe.data_ptr(), coarse.data_ptr(), pscr.data_ptr(), pb, _lib.stream_ptr()),
            "probe")
        return probe, coarse

    def _coarse_prep(self):
        """Tensor-core operand images of the current centroids (made once per
        centroid set; the probe then skips its three preparation kernels)."""
        cent = self._cent
        if getattr(self, "_cprep_for", None) is not cent:
            L, d = cent.shape
            buf = torch.empty(self._lib.ivftq_coarse_prep_bytes(L, d), dtype=torch.uint8,
                              device=self.device)
            _lib.check(self._lib.ivftq_coarse_prepare(cent.data_ptr(), L, d, buf.data_ptr(),
                                                      _lib.stream_ptr()), "coarse_prepare")
            self._cprep, self._cprep_for = buf, cent
        return self._cprep

    def _rotate(self, qn, nq, qrot):
        """Pi q (rotation.py:35-40, index.py:439): f64 product, f32 result."""
        d = self.config.dim
        _lib.check(self._lib.ivftq_gemm_nt(qn.data_ptr(), self._R.data_ptr(), _lib.IVFTQ_F64, nq,
                                           d, d, qrot.data_ptr(), _lib.IVFTQ_F32,
                                           _lib.stream_ptr()), "rotate")

    def _scan(self, qn, nq, probe, coarse, n_p, depth, qrot=None):
        dev = self.device
        d = self.config.dim
        s = _lib.stream_ptr()
        if qrot is None:
            qrot = torch.empty((max(nq, 1), d), dtype=torch.float32, device=dev)
            self._rotate(qn, nq, qrot)
        ids = torch.empty((max(nq, 1), depth), dtype=torch.int64, device=dev)
        scores = torch.empty((max(nq, 1), depth), dtype=torch.float64, device=dev)
        sb = self._lib.ivftq_scan_scratch_bytes(nq, n_p, depth, self.partition.n_lists)
        scr = torch.empty(sb, dtype=torch.uint8, device=dev)
        fn = {"auto": self._lib.ivftq_scan_topk, "lut": self._lib.ivftq_scan_topk_lut,
              "tc": self._lib.ivftq_scan_topk_tc}[self.scan_mode]
        _lib.check(fn(C.byref(self._store.struct()), probe.data_ptr(), coarse.data_ptr(),
                      qrot.data_ptr(), self._levels.data_ptr(), nq, n_p, depth, ids.data_ptr(),
                      scores.data_ptr(), scr.data_ptr(), sb, s), "scan_topk")
        return ids, scores

    def _rerank(self, qn, nq, cand, depth, k):
        dev = self.device
        ids = torch.empty((max(nq, 1), k), dtype=torch.int64, device=dev)
        scores = torch.empty((max(nq, 1), k), dtype=torch.float64, device=dev)
        _lib.check(self._lib.ivftq_rerank(self._raw.t.data_ptr(), qn.data_ptr(), cand.data_ptr(),
                                          nq, depth, self.config.dim, k, ids.data_ptr(),
                                          scores.data_ptr(), _lib.stream_ptr()), "rerank")
        return ids, scores

    def _finish(self, ids, scores, bad, nq, return_device):
        if return_device:
            if int(bad.item()) < nq:
                raise ValueError("zero-norm query")
            return ids[:nq], scores[:nq]
        # one synchronisation: results and the bad-row flag land in pinned
        # host buffers (torch's caching host allocator) with async copies
        ih = torch.empty((nq, ids.shape[1]), dtype=ids.dtype, pin_memory=True)
        sh = torch.empty((nq, scores.shape[1]), dtype=scores.dtype, pin_memory=True)
        bh = torch.empty(1, dtype=bad.dtype, pin_memory=True)
        ih.copy_(ids[:nq], non_blocking=True)
        sh.copy_(scores[:nq], non_blocking=True)
        bh.copy_(bad, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        if int(bh[0]) < nq:
            raise ValueError("zero-norm query")
        return ih.numpy(), sh.numpy()

    def _search_flat_batch(self, queries, k, return_device=False):
        """Exhaustive flat scan, score = <Pi q, rho_hat> (index.py:485-500)."""
        qn, bad, nq = self._normalize_queries_device(queries)
        dev = self.device
        probe = torch.zeros((max(nq, 1), 1), dtype=torch.int32, device=dev)
        coarse = torch.zeros((max(nq, 1), 1), dtype=torch.float64, device=dev)
        ids, scores = self._scan(qn, nq, probe, coarse, 1, k)
        return self._finish(ids, scores, bad, nq, return_device)

    # ------------------------------------------------------------------
    # diagnostics

    def bit_accounting(self) -> dict:
        """Logical per-vector bit budget (index.py:505-534)."""
        cfg = self.config
        code_bits = cfg.bits * cfg.dim
        sign_bits = cfg.dim if cfg.use_sign_bit else 0
        list_bits = int(np.ceil(np.log2(cfg.n_lists))) if cfg.n_lists > 1 else 0
        exact = code_bits + sign_bits + list_bits + 16
        return {
            "bits_per_vec": exact,
            "bits_per_vec_32bit_overhead": code_bits + sign_bits + 32,
            "breakdown": {"code_bits": code_bits, "sign_bits": sign_bits,
                          "list_id_bits": list_bits, "norm_bits": 16},
            "fixed_overhead_bits": {"centroid_table": cfg.n_lists * cfg.dim * 32,
                                    "rotation_matrix": cfg.dim * cfg.dim * 64},
            "count": self.count,
            "total_logical_bytes": int(np.ceil(exact * self.count / 8)),
        }

    def bit_flip_ablation(self, bit_position: str, fraction: float, queries: np.ndarray,
                          k: int, n_p: int, seed: int = 0,
                          truth: np.ndarray | None = None) -> dict:
        """Recall drop when one stored bit position is flipped in a seeded fraction
        of (vector, coordinate) slots; codes are restored (index.py:536-601)."""
        from .evaluation import exact_topk, recall_at_k

        if not 0 <= fraction <= 1:
            raise ValueError(f"fraction must be in [0, 1], got {fraction}")
        if bit_position not in ("msb_primary", "lsb_primary", "sign"):
            raise ValueError(f"unknown bit_position {bit_position!r}")
        if bit_position == "sign" and not self.config.use_sign_bit:
            raise ValueError("sign-bit ablation requires use_sign_bit=True")
        if truth is None:
            if self.raw is None:
                raise ValueError("need truth or an index built with keep_raw=True")
            truth = exact_topk(self.raw, queries, k).ids

        def run() -> float:
            ids, _ = self.search_batch(queries, k, n_p)
            return recall_at_k(ids, truth, k)

        base = run()
        rng = np.random.default_rng(seed)
        mask = rng.random((self.count, self.config.dim)) < fraction
        which = 1 if bit_position == "sign" else 0
        flip = 1 << (self.config.bits - 1) if bit_position == "msb_primary" else 1
        m = torch.from_numpy(mask.astype(np.uint8)).to(self.device)

        def apply():
            _lib.check(self._lib.ivftq_xor_codes(C.byref(self._store.struct()),
                                                 self._slot_of.t.data_ptr(), self.count,
                                                 m.data_ptr(), which, flip, _lib.stream_ptr()),
                       "xor_codes")
            self._version += 1

        try:
            apply()
            corrupted = run()
        finally:
            apply()  # XOR again restores the codes bit-for-bit
        return {"bit_position": bit_position, "fraction": fraction, "recall_base": base,
                "recall_corrupted": corrupted, "recall_drop": base - corrupted}


def build(config: IndexConfig, training_data: np.ndarray) -> IvfTqIndex:
    return IvfTqIndex.build(config, training_data)


def search_flat_tq(index: IvfTqIndex, q: np.ndarray, k: int) -> SearchResult:
    if not index.config.flat:
        raise ValueError("index was not built in flat mode")
    return index.search(q, k, n_p=1)


def bit_accounting(index: IvfTqIndex) -> dict:
    return index.bit_accounting()


def bit_flip_ablation(index: IvfTqIndex, bit_position: str, fraction: float,
                      queries: np.ndarray, k: int, n_p: int, seed: int = 0,
                      truth: np.ndarray | None = None) -> dict:
    return index.bit_flip_ablation(bit_position, fraction, queries, k, n_p, seed, truth)
