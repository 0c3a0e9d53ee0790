"""The behavioural scenarios of the reference's own index tests, restated
against this package on seeded mixture data (the reference's files themselves
run unmodified through scripts/run_reference_tests.py; these are the
driver-run counterparts). Each test names the reference test it follows
(/root/reference/pkg/tests/test_index.py, test_refresh.py, test_storage.py).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rows(n, d, seed):
    from paper_2605_17415_b200.workloads import mixture

    x, _ = mixture(n, d, 24, 0.35, seed, mean_seed=1234)
    return x.astype(np.float64)


@pytest.fixture(scope="module")
def built():
    from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex

    data = _rows(2000, 32, seed=0)
    return IvfTqIndex.build(IndexConfig(dim=32, bits=4, n_lists=16, keep_raw=True), data), data


def test_self_retrieval_with_full_probe(built):
    """test_index.py:74-78: nearly every stored vector is its own nearest neighbour."""
    index, data = built
    ids, _ = index.search_batch(data[:500], 1, n_p=16)
    assert np.mean(ids[:, 0] == np.arange(500)) >= 0.99


def test_reconstruction_error_within_rate_envelope(built):
    """test_index.py:107-119: |x_hat - x~| <= |r| (sqrt(D_b) + margin) for nearly all vectors."""
    from paper_2605_17415_b200.refresh import reconstruct_all

    index, data = built
    xn = data / np.linalg.norm(data, axis=1)[:, None]
    err = np.linalg.norm(reconstruct_all(index, renormalize=False)[: len(data)] - xn, axis=1)
    bound = index.norms[: len(data)].astype(np.float64) * (np.sqrt(index.quantizer.distortion_sign) + 0.15)
    assert np.mean(err <= bound) >= 0.99


def test_add_then_search_finds_new_vector(built):
    """test_index.py:121-129: an added vector gets the next id and is found with rerank."""
    index, _ = built
    before = index.count
    v = np.random.default_rng(5).standard_normal(32)
    assert index.add(v) == before
    ids, _ = index.search_batch(v[None, :], 1, n_p=16, rerank_depth=4)
    assert ids[0, 0] == before


def test_interleaved_adds_match_batch_build():
    """test_index.py:142-169: equal content + the same partition -> identical results,
    whatever the add order and the searches in between."""
    from paper_2605_17415_b200 import CoarsePartition
    from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex

    data, queries = _rows(1200, 16, seed=3), _rows(100, 16, seed=4)
    cfg = IndexConfig(dim=16, bits=3, n_lists=8)
    batch = IvfTqIndex.build(cfg, data)
    shared = CoarsePartition(n_lists=8, dim=16, centroids=batch.partition.centroids.copy())
    inc = IvfTqIndex(cfg, batch.quantizer, batch.rot, shared)
    inc.add_batch(data[:600])
    inc.search_batch(queries, 5, n_p=8)
    for row in data[600:900]:
        inc.add(row)
    inc.add_batch(data[900:])
    a = batch.search_batch(queries, 10, n_p=8)
    b = inc.search_batch(queries, 10, n_p=8)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_exact_self_query_with_rerank(built):
    """test_index.py:173-177: reranked self query scores 1."""
    index, data = built
    res = index.search(data[42], 1, n_p=16, rerank_depth=20)
    assert res.ids[0] == 42 and abs(res.scores[0] - 1.0) < 1e-4


def test_scores_sorted_ids_distinct_and_candidate_superset(built):
    """test_index.py:179-194: non-increasing scores, distinct ids, and a deeper probe
    only ever adds candidates."""
    index, data = built
    res = index.search(data[0], 10, n_p=4)
    assert np.all(np.diff(res.scores) <= 0) and len(set(res.ids.tolist())) == len(res.ids)
    q = np.random.default_rng(8).standard_normal(32)
    shallow, _ = index.search_batch(q[None], 2000, n_p=4)
    deep, _ = index.search_batch(q[None], 2000, n_p=8)
    assert set(shallow[0][shallow[0] >= 0].tolist()) <= set(deep[0][deep[0] >= 0].tolist())


def test_score_decomposition_exact_without_quantization(built):
    """test_index.py:222-237: with the true unit residual and the stored norm, the
    asymmetric score is the exact inner product up to binary16 rounding of the norm."""
    index, data = built
    q = np.random.default_rng(9).standard_normal(32)
    qn = q / np.linalg.norm(q)
    for i in (3, 100, 999):
        x = data[i] / np.linalg.norm(data[i])
        cent = index.partition.centroids[int(index.list_ids[i])].astype(np.float64)
        r = x - cent
        rho = index.rot.apply(r / np.linalg.norm(r))
        est = qn @ cent + float(index.norms[i]) * (index.rot.apply(qn) @ rho)
        assert abs(est - qn @ x) <= np.linalg.norm(r) * 2 ** -10 + 1e-9


def test_save_load_round_trip_searches_identically(built, tmp_path):
    """test_storage.py:22-44: a saved and reloaded index returns the same results."""
    from paper_2605_17415_b200.storage import load_index, save_index

    index, data = built
    path = tmp_path / "index.ivtq"
    save_index(index, path)
    again = load_index(path)
    a = index.search_batch(data[:50], 5, n_p=8)
    b = again.search_batch(data[:50], 5, n_p=8)
    assert again.count == index.count
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_refresh_keeps_compression_layer_and_recall():
    """test_refresh.py:124-129 and 96-110: refresh never touches the quantizer or the
    rotation, and recall after it stays within a point of before."""
    from paper_2605_17415_b200.evaluation import exact_topk, recall_at_k
    from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex
    from paper_2605_17415_b200.refresh import RefreshPolicy, refresh

    data, queries = _rows(6000, 48, seed=20), _rows(200, 48, seed=21)
    index = IvfTqIndex.build(IndexConfig(dim=48, bits=4, n_lists=24, keep_raw=True, kmeans_seed=5), data)
    truth = exact_topk(data / np.linalg.norm(data, axis=1)[:, None], queries, 10)
    before = recall_at_k(index.search_batch(queries, 10, n_p=8)[0], truth, 10)
    fp, quantizer, rot = index.compression_fingerprint(), index.quantizer, index.rot
    report = refresh(index, RefreshPolicy(seed=3))
    assert report.refreshed
    assert index.quantizer is quantizer and index.rot is rot
    assert index.compression_fingerprint() == fp
    after = recall_at_k(index.search_batch(queries, 10, n_p=8)[0], truth, 10)
    assert after >= before - 0.01
