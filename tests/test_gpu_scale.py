"""GPU parity at the BASELINE configs' shapes (driver-run, `-m gpu`).

The golden fixtures pin the small shapes; these tests take the CUDA path to
the shapes the bench measures, with the CPU oracle (oracle/ivftq_oracle.py)
as the checker on bounded samples:

  * C3 shape: d=96, L=4096, 1M rows, n_p=32, 10k-query batch (the tensor-core
    list-major scan with ~78 queries per list, as at C3);
  * C4 shape: d=200, log-normal base norms, shifted (out-of-distribution)
    queries, b in {2, 3, 4}, n_p=64 (64-vector scan tiles);
  * a mini C5 stream: batches appended, a refresh after batches 2 and 4 that
    injects the oracle's refreshed centroids (SURVEY §7 "Refresh centroid
    parity"), codes and searches compared after every batch;
  * concurrent readers: two host threads search one index on two streams.

Bars are north_star's (tests/helpers.py): codes bit-exact up to <= 1e-4 flips,
list ids and binary16 norms identical, ids identical up to ties within 1e-4
relative, recall within 0.1 pp.
"""

import threading

import numpy as np
import pytest

from helpers import compare_topk

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _index(d, bits, cent, R=None, keep_raw=False):
    from paper_2605_17415_b200 import (CoarsePartition, IndexConfig, IvfTqIndex,
                                       design_quantizer, generate_rotation)

    L = len(cent)
    q = design_quantizer(bits, d)
    R = R if R is not None else generate_rotation(d, 42)
    cfg = IndexConfig(dim=d, bits=bits, n_lists=L, keep_raw=keep_raw)
    return IvfTqIndex(cfg, q, R, CoarsePartition(L, d, cent)), q, R


def _sample_centroids(x, L, seed):
    """L distinct unit data rows as f32 centroids (a valid coarse partition)."""
    rng = np.random.default_rng(seed)
    c = x[rng.choice(len(x), L, replace=False)].astype(np.float64)
    return (c / np.linalg.norm(c, axis=1)[:, None]).astype(np.float32)


def _code_window(idx, x, cent, R, q, off, m):
    from oracle import ivftq_oracle as orc

    b, s, l, n, _ = orc.encode_batch(x[off:off + m], cent, R.matrix, q.boundaries, q.centroids)
    flips = ((idx.bins[off:off + m] != b) | (idx.signs[off:off + m] != s)).mean()
    assert flips <= 1e-4, flips
    np.testing.assert_array_equal(idx.list_ids[off:off + m], l)
    np.testing.assert_array_equal(idx.norms[off:off + m].view(np.uint16), n.view(np.uint16))


def _search_parity(idx, cent, R, q, queries, n_p, sample, truth=None):
    """GPU batch search vs the oracle over the GPU-encoded fields (bit-exact to
    the oracle's own encode on the checked windows) on a query sample."""
    from oracle import ivftq_oracle as orc
    from paper_2605_17415_b200.evaluation import recall_at_k

    gi, gs = idx.search_batch(queries, 10, n_p)  # the whole batch: list reuse as in the bench
    o = orc.OracleIndex(cent, R.matrix, q.boundaries, q.centroids, q.half_bin_means)
    o.bins, o.signs, o.list_ids, o.norms = idx.bins, idx.signs, idx.list_ids, idx.norms
    oi, os_ = o.search_batch(queries[sample], 10, n_p)
    compare_topk(gi[sample], gs[sample], oi, os_)
    if truth is not None:
        r_g = recall_at_k(gi[sample], truth[sample], 10)
        r_o = recall_at_k(oi, truth[sample], 10)
        assert abs(r_g - r_o) <= 0.001, (r_g, r_o)
    return gi, gs


def test_c3_shape_parity():
    """d=96, L=4096, 1M rows, 10k queries at n_p=32 (configs[2] shape)."""
    import torch

    from paper_2605_17415_b200.evaluation import exact_topk
    from paper_2605_17415_b200.workloads import mixture

    n, d, L = 1_000_000, 96, 4096
    x, means = mixture(n, d, 4096, 0.3, 31, threads=8)
    qx, _ = mixture(10_000, d, 4096, 0.3, 32, means=means)
    cent = _sample_centroids(x, L, 33)
    idx, q, R = _index(d, 4, cent)
    idx.add_batch(x[:400_000])
    idx.add_batch(x[400_000:])
    _code_window(idx, x, cent, R, q, 500_000, 200_000)
    xn = torch.from_numpy(x).cuda().double()
    xn /= xn.norm(dim=1, keepdim=True)
    qn = qx.astype(np.float64) / np.linalg.norm(qx, axis=1)[:, None]
    truth = exact_topk(xn, qn, 10).ids
    del xn
    sample = np.sort(np.random.default_rng(3).choice(10_000, 600, replace=False))
    _search_parity(idx, cent, R, q, qx, 32, sample, truth)
    # n_p=16 and 64 on a smaller sample: the scan's item mix changes with n_p
    for n_p in (16, 64):
        _search_parity(idx, cent, R, q, qx, n_p, sample[:200])


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_c4_shape_parity(bits):
    """d=200, log-normal norms, shifted queries (configs[3] shape), n_p=64."""
    from paper_2605_17415_b200.workloads import make_workload

    w = make_workload("c4", n=300_000, bits=bits, n_queries=3000)
    x = w.base()
    qx = w.queries()
    cent = _sample_centroids(x, 1024, 41)
    idx, q, R = _index(w.d, bits, cent)
    idx.add_batch(x)
    _code_window(idx, x, cent, R, q, 100_000, 60_000)
    sample = np.sort(np.random.default_rng(4).choice(3000, 250, replace=False))
    _search_parity(idx, cent, R, q, qx, 64, sample)


def test_c5_mini_stream_injected_refresh():
    """configs[4] protocol at reduced size: d=96, L=256; 6 batches of 40k;
    refresh after batches 2 and 4 with the oracle's refreshed centroids
    injected (refresh.py:134-215 composed from the oracle's pieces); codes and
    search parity after every batch against the oracle's own index."""
    from oracle import ivftq_oracle as orc
    from paper_2605_17415_b200.refresh import RefreshPolicy, refresh
    from paper_2605_17415_b200.workloads import mixture

    d, L, nb = 96, 256, 40_000
    x, means = mixture(7 * nb, d, 512, 0.3, 51)
    qx, _ = mixture(400, d, 512, 0.3, 52, means=means)
    perm = np.random.default_rng(53).permutation(6 * nb)
    train = orc.normalize_rows(x[:nb])
    cent = orc.train_partition(train, L, seed=42, max_iters=10)
    idx, q, R = _index(d, 4, cent)
    o = orc.OracleIndex(cent, R.matrix, q.boundaries, q.centroids, q.half_bin_means)
    stream = x[nb:][perm]
    for b in range(6):
        rows = stream[b * nb:(b + 1) * nb]
        idx.add_batch(rows)
        o.add_batch(rows)
        if b in (2, 4):
            # the oracle's refresh: stratified sample (ascending-id lists,
            # refresh.py:109-131), k-means on decoded rows, full re-encode
            rng = np.random.default_rng(7 + b)
            n = o.count
            sample_size = min(n, max(100 * L, n // 10))
            ids = orc.stratified_sample_ids(o.members(), n, L, sample_size, rng)
            src = orc.reconstruct_all(o)
            new_c = orc.train_partition(src[ids], L, seed=7 + b, max_iters=25)
            orc.refresh_encode(o, src, new_c)
            rep = refresh(idx, RefreshPolicy(seed=7 + b), centroids=new_c)
            assert rep.refreshed and rep.n_reassigned == n
        np.testing.assert_array_equal(idx.list_ids, o.list_ids)
        np.testing.assert_array_equal(idx.norms.view(np.uint16), o.norms.view(np.uint16))
        assert ((idx.bins != o.bins) | (idx.signs != o.signs)).mean() <= 1e-4
        gi, gs = idx.search_batch(qx, 10, 16)
        oi, os_ = o.search_batch(qx, 10, 16)
        compare_topk(gi, gs, oi, os_)


def test_concurrent_readers_two_streams(golden):
    """Two host threads search one index on their own streams (graphs and the
    library's side streams are per thread): results equal the serial ones."""
    import torch

    from helpers import index_from_golden

    g = golden("d128_b4_L64")
    idx = index_from_golden(g)
    idx.add_batch(g["x"])
    rng = np.random.default_rng(9)
    qs = [g["x"][rng.integers(0, len(g["x"]), 300)] + 0.05 * rng.standard_normal((300, 128))
          for _ in range(2)]
    ref = [idx.search_batch(qq, 10, 8) for qq in qs]
    errors = []

    def worker(t):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for r in range(15):
                    ids, sc = idx.search_batch(qs[t], 10, 8)
                    np.testing.assert_array_equal(ids, ref[t][0])
                    np.testing.assert_array_equal(sc, ref[t][1])
                    di, ds = idx.search_batch(torch.from_numpy(qs[t]).cuda(), 10, 8,
                                              return_device=True)
                    np.testing.assert_array_equal(di.cpu().numpy(), ref[t][0])
        except Exception as e:  # surfaced in the main thread
            errors.append(e)

    th = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors[0]


def test_seeded_bounds_exact_near_ties_d200(monkeypatch):
    """d=200 near-ties at the pruning bound: results with the seeded global
    bounds equal the unseeded scan (the seed margin is derived from d)."""
    from paper_2605_17415_b200.workloads import mixture

    d, L = 200, 16
    base, means = mixture(400, d, 20, 0.3, 61)
    rng = np.random.default_rng(62)
    # 40 near-copies of each row: their codes mostly coincide, scores tie or
    # differ in the last bits
    x = np.repeat(base, 40, axis=0) + 1e-7 * rng.standard_normal((16_000, d)).astype(np.float32)
    qx = base[rng.integers(0, 400, 200)] + 0.02 * rng.standard_normal((200, d))
    cent = _sample_centroids(x, L, 63)
    idx, _, _ = _index(d, 4, cent)
    idx.add_batch(x)
    idx.use_graphs = False
    a = idx.search_batch(qx, 10, 4)
    monkeypatch.setenv("IVFTQ_NO_SEED", "1")
    b = idx.search_batch(qx, 10, 4)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])
