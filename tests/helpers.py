"""Shared test helpers: build indexes from golden fixtures, compare results."""

import numpy as np

SCORE_RTOL = 1e-4  # north_star: estimated scores within 1e-4 relative
# absolute floor for scores near 0: the reference's own f32 residual GEMM
# (index.py:453) carries ~d * 2^-24 absolute error, so a relative bound is
# meaningless for |score| << 1e-2.
SCORE_ATOL = 1e-6


def parts_from_golden(g, prefix=""):
    from paper_2605_17415_b200.partition import CoarsePartition
    from paper_2605_17415_b200.quantizer import ScalarQuantizer
    from paper_2605_17415_b200.rotation import RotationMatrix
    from paper_2605_17415_b200.index import IndexConfig

    c = g[prefix + "config"]
    cfg = IndexConfig(dim=int(c[0]), bits=int(c[1]), n_lists=int(c[2]), use_sign_bit=bool(c[3]),
                      keep_raw=bool(c[4]), flat=bool(c[5]), rotation_seed=int(c[6]),
                      kmeans_seed=int(c[7]))
    dist = g[prefix + "distortion"]
    q = ScalarQuantizer(bits=cfg.bits, dim=cfg.dim, boundaries=g[prefix + "boundaries"].copy(),
                        centroids=g[prefix + "qcent"].copy(),
                        half_bin_means=g[prefix + "half"].copy(), distortion=float(dist[0]),
                        distortion_sign=float(dist[1]))
    rot = RotationMatrix(dim=cfg.dim, matrix=g[prefix + "R"].copy(), seed=cfg.rotation_seed)
    part = CoarsePartition(cfg.n_lists, cfg.dim, g[prefix + "centroids"].copy())
    return cfg, q, rot, part


def index_from_golden(g, prefix=""):
    from paper_2605_17415_b200.index import IvfTqIndex

    cfg, q, rot, part = parts_from_golden(g, prefix)
    return IvfTqIndex(cfg, q, rot, part)


def compare_topk(ids, scores, ref_ids, ref_scores, rtol=SCORE_RTOL, atol=SCORE_ATOL):
    """Assert top-k parity up to ties within rtol; return #queries that differ."""
    ids = np.asarray(ids)
    ref_ids = np.asarray(ref_ids)
    assert ids.shape == ref_ids.shape
    fin = np.isfinite(ref_scores)
    np.testing.assert_array_equal(np.isfinite(scores), fin)
    np.testing.assert_array_equal(ids[~fin], -1)
    np.testing.assert_allclose(scores[fin], ref_scores[fin], rtol=rtol, atol=atol)
    ndiff = 0
    for q in range(len(ids)):
        if np.array_equal(ids[q], ref_ids[q]):
            continue
        ndiff += 1
        k = int(fin[q].sum())
        for i in range(k):
            if ids[q, i] == ref_ids[q, i]:
                continue
            # a swap is only allowed between candidates tied within rtol
            assert abs(scores[q, i] - ref_scores[q, i]) <= rtol * abs(ref_scores[q, i]) + atol
            if ids[q, i] not in ref_ids[q, :k]:
                kth = ref_scores[q, k - 1]
                assert abs(scores[q, i] - kth) <= rtol * abs(kth) + atol, (q, i)
    return ndiff
