"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle on the same seeded inputs.

Bars (north_star): codes bit-exact (a fraction <= 1e-4 of boundary flips is
tolerated and reported), list ids and binary16 norms identical, probe lists
identical, scores within 1e-4 relative, top-k ids identical up to ties within
that tolerance, recall@10 within 0.1 pp.
"""

import warnings

import numpy as np
import pytest

from helpers import SCORE_RTOL, compare_topk, index_from_golden, parts_from_golden

pytestmark = pytest.mark.gpu

SMALL = ["d32_b4_L16_raw", "d16_b3_L8", "d24_b5_L12_raw", "d96_b2_nosign_L32",
         "d200_b3_L16", "d64_b8_L8", "d40_b1_L4", "d128_b4_L64", "flat_d16_b8"]


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _search_keys(g):
    out = []
    for k in g:
        if k.startswith("s_") and k.endswith("_ids"):
            _, kk, p, rr, _ = k.split("_")
            out.append((int(kk), int(p), int(rr)))
    return out


def test_device_normalize_bit_exact():
    import torch

    from paper_2605_17415_b200 import _lib

    L = _lib.lib()
    for d in (2, 7, 16, 96, 128, 129, 200, 300):
        rng = np.random.default_rng(d)
        x = rng.standard_normal((777, d)) * np.exp(rng.uniform(-3, 3, (777, 1)))
        x[5] = 0.0
        x[9] = 0.0
        xt = torch.from_numpy(x).cuda()
        out = torch.empty_like(xt)
        bad = torch.empty(1, dtype=torch.int64, device="cuda")
        _lib.check(L.ivftq_normalize_rows(xt.data_ptr(), 1, 777, d, out.data_ptr(),
                                          bad.data_ptr(), _lib.stream_ptr()))
        assert int(bad.item()) == 5
        ref = x / np.linalg.norm(x, axis=1)[:, None]
        got = out.cpu().numpy()
        ok = np.ones(777, bool)
        ok[[5, 9]] = False
        np.testing.assert_array_equal(got[ok], ref[ok])


@pytest.mark.parametrize("name", SMALL)
def test_encode_matches_reference(golden, name):
    g = golden(name)
    idx = index_from_golden(g)
    ids = idx.add_batch(g["x"])
    np.testing.assert_array_equal(ids, np.arange(len(g["x"])))
    np.testing.assert_array_equal(idx.list_ids, g["list_ids"])
    np.testing.assert_array_equal(idx.norms.view(np.uint16), g["norms"].view(np.uint16))
    flips = (idx.bins != g["bins"]) | (idx.signs != g["signs"])
    assert flips.mean() <= 1e-4, flips.mean()
    np.testing.assert_array_equal(idx.bins, g["bins"])
    np.testing.assert_array_equal(idx.signs, g["signs"])
    if g["config"][4]:
        np.testing.assert_array_equal(idx.raw, g["raw"])
    assert idx.compression_fingerprint() == g["fingerprint"].tobytes().decode()


def _tc_ok(idx, depth):
    from paper_2605_17415_b200 import _lib

    return bool(_lib.lib().ivftq_scan_tc_supported(idx.config.dim, idx.config.bits, depth))


def _set_mode(idx, mode, monkeypatch):
    """lut, or the tensor-core scan with its kernel forced: tc_vq (vectors x
    queries, scan_vq.cu) or tc_qm (queries x vectors, scan_tc.cu)."""
    if mode.startswith("tc"):
        monkeypatch.setenv("IVFTQ_SCAN_VQ", "1" if mode == "tc_vq" else "0")
        idx.scan_mode = "tc"
    else:
        idx.scan_mode = mode


@pytest.mark.parametrize("mode", ["lut", "tc_vq", "tc_qm"])
@pytest.mark.parametrize("name", SMALL)
def test_search_matches_reference(golden, name, mode, monkeypatch):
    g = golden(name)
    idx = index_from_golden(g)
    _set_mode(idx, mode, monkeypatch)
    idx.add_batch(g["x"])
    ran = 0
    for (k, n_p, rr) in _search_keys(g):
        depth = max(k, rr) if rr else k
        if mode != "lut" and not _tc_ok(idx, depth):
            continue
        ran += 1
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            ids, sc = idx.search_batch(g["queries"], k, n_p, rr)
        assert ids.dtype == np.int64 and sc.dtype == np.float64
        compare_topk(ids, sc, g[f"s_{k}_{n_p}_{rr}_ids"], g[f"s_{k}_{n_p}_{rr}_scores"])
    if mode != "lut" and not ran:
        pytest.skip("no tensor-core-eligible case (bits or depth)")


def test_probes_identical(golden):
    import torch

    from paper_2605_17415_b200 import _lib

    g = golden("d128_b4_L64")
    idx = index_from_golden(g)
    qn, bad, nq = idx._normalize_queries_device(g["queries"])
    L = _lib.lib()
    probe = torch.empty((nq, 64), dtype=torch.int32, device="cuda")
    coarse = torch.empty((nq, 64), dtype=torch.float64, device="cuda")
    sb = L.ivftq_probe_scratch_bytes(nq, 64, 128)
    scr = torch.empty(sb, dtype=torch.uint8, device="cuda")
    _lib.check(L.ivftq_probe(qn.data_ptr(), idx._cent.data_ptr(), nq, 64, 128, 64,
                             probe.data_ptr(), coarse.data_ptr(), scr.data_ptr(), sb,
                             _lib.stream_ptr()))
    np.testing.assert_array_equal(probe.cpu().numpy(), g["probe_all"][:, :64])
    ref = np.take_along_axis(g["coarse"], g["probe_all"][:, :64], 1)
    np.testing.assert_allclose(coarse.cpu().numpy(), ref, rtol=0, atol=1e-15)


@pytest.mark.parametrize("mode", ["lut", "tc_vq", "tc_qm"])
@pytest.mark.parametrize("seed,d,bits,L,sign", [(1, 48, 4, 24, True), (2, 100, 3, 40, True),
                                                  (3, 64, 2, 16, False), (4, 130, 4, 8, True),
                                                  (5, 33, 6, 12, True), (6, 20, 7, 6, False),
                                                  (7, 200, 4, 32, True), (8, 96, 4, 64, True)])
def test_random_configs_against_oracle(seed, d, bits, L, sign, mode, monkeypatch):
    """Fresh seeded inputs, oracle restatement as the checker."""
    from oracle import ivftq_oracle as orc
    from paper_2605_17415_b200 import (CoarsePartition, IndexConfig, IvfTqIndex,
                                       design_quantizer, generate_rotation)
    from paper_2605_17415_b200.workloads import mixture

    x, means = mixture(3000, d, 30, 0.3, seed)
    qx, _ = mixture(120, d, 30, 0.3, seed + 100, means=means)
    xn = orc.normalize_rows(x)
    cent = orc.train_partition(xn[:1500], L, seed=seed, max_iters=5)
    q = design_quantizer(bits, d)
    R = generate_rotation(d, seed)
    cfg = IndexConfig(dim=d, bits=bits, n_lists=L, use_sign_bit=sign, keep_raw=True)
    idx = IvfTqIndex(cfg, q, R, CoarsePartition(L, d, cent))
    if mode != "lut" and not _tc_ok(idx, 15):
        pytest.skip("bits outside the tensor-core path")
    _set_mode(idx, mode, monkeypatch)
    idx.add_batch(x[:1000])
    idx.add_batch(x[1000:])
    o = orc.OracleIndex(cent, R.matrix, q.boundaries, q.centroids, q.half_bin_means,
                        use_sign=sign, keep_raw=True)
    o.add_batch(x)
    np.testing.assert_array_equal(idx.list_ids, o.list_ids)
    np.testing.assert_array_equal(idx.norms.view(np.uint16), o.norms.view(np.uint16))
    assert ((idx.bins != o.bins) | (idx.signs != o.signs)).mean() <= 1e-4
    for (k, n_p, rr) in [(10, 4, 0), (10, L, 0), (1, 2, 0), (7, 3, 15)]:
        a = idx.search_batch(qx, k, n_p, rr)
        b = o.search_batch(qx, k, n_p, rr)
        compare_topk(*a, *b)


@pytest.mark.slow
def test_pr1_full_parity(golden):
    """configs[0] at full size: 100k x 128, L=256, b=4; 1k queries, n_p sweep."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).parent / "golden"))
    from hashing import row_hash

    from paper_2605_17415_b200.index import pack_fields
    from paper_2605_17415_b200.evaluation import recall_at_k
    from paper_2605_17415_b200.workloads import make_workload

    g = golden("pr1")
    w = make_workload("pr1")
    idx = index_from_golden(g)
    idx.add_batch(w.base())
    np.testing.assert_array_equal(idx.list_ids, g["list_ids"].astype(np.int64))
    np.testing.assert_array_equal(idx.norms.view(np.uint16), g["norms"].view(np.uint16))
    packed = np.concatenate([pack_fields(idx.bins, 4), pack_fields(idx.signs, 1)], 1)
    mism = (row_hash(packed) != g["code_hash"]).mean()
    assert mism <= 1e-4, mism
    qx = w.queries()
    for n_p in (1, 4, 16, 64):
        ids, sc = idx.search_batch(qx, 10, n_p)
        ref_i, ref_s = g[f"s_10_{n_p}_0_ids"], g[f"s_10_{n_p}_0_scores"]
        ndiff = compare_topk(ids, sc, ref_i, ref_s)
        assert ndiff <= 0.01 * len(ids)
        r_ours = recall_at_k(ids, g["truth10"], 10)
        r_ref = recall_at_k(ref_i, g["truth10"], 10)
        assert abs(r_ours - r_ref) <= 0.001, (n_p, r_ours, r_ref)


def test_exact_topk_gpu_matches_reference(golden):
    from paper_2605_17415_b200.evaluation import exact_topk

    for name in ("d32_b4_L16_raw", "d128_b4_L64"):
        g = golden(name)
        x = g["x"].astype(np.float64)
        xn = x / np.linalg.norm(x, axis=1)[:, None]
        t = exact_topk(xn, g["queries"], 10, db_chunk=1000)
        np.testing.assert_array_equal(t.ids, g["truth10"])


@pytest.mark.parametrize("cols,n", [(1, 1), (7, 3), (64, 64), (1024, 1), (1024, 32),
                                    (1024, 33), (1024, 64), (1000, 100), (4096, 128),
                                    (4096, 129), (300, 257)])
def test_select_topn_stable_order(cols, n):
    """Per-row top-n must equal a stable argsort of -scores (index.py:438),
    including exact ties (lower column first), -0.0 == 0.0 and NaN last."""
    import torch

    from paper_2605_17415_b200 import _lib

    rng = np.random.default_rng(cols * 1000 + n)
    rows = 37
    S = rng.integers(-8, 8, size=(rows, cols)).astype(np.float64) / 8.0  # many ties
    S[0] = rng.standard_normal(cols)
    if cols > 4:
        S[1, :: 3] = -0.0
        S[1, 1:: 3] = 0.0
        if n <= 128:  # the warp-queue path orders NaN last like argsort
            S[2, ::5] = np.nan
    S[3] = 0.25
    dS = torch.from_numpy(S).cuda()
    idx = torch.empty((rows, n), dtype=torch.int32, device="cuda")
    val = torch.empty((rows, n), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().ivftq_select_topn(dS.data_ptr(), rows, cols, n, idx.data_ptr(),
                                             val.data_ptr(), None), "select_topn")
    torch.cuda.synchronize()
    want = np.argsort(-S, axis=1, kind="stable")[:, :n]
    np.testing.assert_array_equal(idx.cpu().numpy(), want)
    wv = np.take_along_axis(S, want, axis=1)
    np.testing.assert_array_equal(val.cpu().numpy(), wv)


class TestEdgeCases:
    def test_errors_and_warnings(self, golden):
        g = golden("d32_b4_L16_raw")
        idx = index_from_golden(g)
        idx.add_batch(g["x"][:500])
        with pytest.raises(ValueError, match="k must be"):
            idx.search(g["x"][0], 0, n_p=2)
        with pytest.raises(ValueError, match="n_p must be"):
            idx.search(g["x"][0], 3, n_p=0)
        with pytest.warns(UserWarning, match="clamping"):
            idx.search(g["x"][0], 3, n_p=999)
        with pytest.raises(ValueError, match="dim"):
            idx.search(np.ones(16), 3, n_p=2)
        with pytest.raises(ValueError, match="zero-norm query"):
            idx.search(np.zeros(32), 3, n_p=2)
        with pytest.raises(ValueError, match="row at index 3"):
            bad = g["x"][:6].copy()
            bad[3] = 0
            idx.add_batch(bad)
        with pytest.raises(ValueError, match="external_ids length"):
            idx.add_batch(g["x"][:3], external_ids=np.arange(2))
        assert idx.count == 500

    def test_rerank_requires_raw(self, golden):
        g = golden("d16_b3_L8")
        idx = index_from_golden(g)
        idx.add_batch(g["x"])
        with pytest.raises(ValueError, match="keep_raw"):
            idx.search(g["x"][0], 3, n_p=2, rerank_depth=5)

    def test_empty_index_pads(self, golden):
        g = golden("d16_b3_L8")
        idx = index_from_golden(g)
        ids, sc = idx.search_batch(g["queries"][:4], 5, 3)
        assert (ids == -1).all() and np.isneginf(sc).all()

    def test_centroid_input_zero_residual(self, golden):
        g = golden("d32_b4_L16_raw")
        idx = index_from_golden(g)
        code = idx.encode(idx.partition.centroids[3].astype(np.float64))
        ref = g["centroid_code"].tobytes()
        assert code.codes + code.signs == ref
        assert code.list_id == int(g["centroid_code_meta"][0]) == 3
        assert float(code.residual_norm) == 0.0

    def test_incremental_equals_batch(self, golden):
        g = golden("d16_b3_L8")
        a = index_from_golden(g)
        a.add_batch(g["x"])
        b = index_from_golden(g)
        b.add_batch(g["x"][:600])
        b.search_batch(g["queries"], 5, 8)
        for row in g["x"][600:650]:
            b.add(row)
        b.add_batch(g["x"][650:])
        np.testing.assert_array_equal(a.bins, b.bins)
        ia, sa = a.search_batch(g["queries"], 10, 8)
        ib, sb = b.search_batch(g["queries"], 10, 8)
        np.testing.assert_array_equal(ia, ib)
        np.testing.assert_array_equal(sa, sb)

    def test_duplicates_tie_to_lower_id(self, golden):
        g = golden("d32_b4_L16_raw")  # rows 2000..2039 duplicate rows 0..39
        idx = index_from_golden(g)
        idx.add_batch(g["x"])
        ids, sc = idx.search_batch(g["x"][:40], 2, 16)
        for i in range(40):
            assert sc[i, 0] == sc[i, 1]
            assert ids[i, 0] < ids[i, 1]

    def test_partition_lists_view(self, golden):
        g = golden("d16_b3_L8")
        idx = index_from_golden(g)
        idx.add_batch(g["x"])
        lists = idx.partition.lists
        assert sum(len(m) for m in lists) == idx.count
        for l, m in enumerate(lists):
            assert m == sorted(m)
            assert all(idx.list_ids[i] == l for i in m)

    def test_bit_flip_ablation_restores(self, golden):
        g = golden("d32_b4_L16_raw")
        idx = index_from_golden(g)
        idx.add_batch(g["x"])
        before = idx.bins.copy(), idx.signs.copy()
        truth = g["truth10"]
        r0 = idx.bit_flip_ablation("msb_primary", 0.0, g["queries"], 10, 16, truth=truth)
        assert r0["recall_drop"] == 0.0
        r = idx.bit_flip_ablation("msb_primary", 0.5, g["queries"], 10, 16, seed=1, truth=truth)
        assert r["recall_drop"] > 0
        idx.bit_flip_ablation("sign", 0.3, g["queries"], 10, 16, seed=2, truth=truth)
        np.testing.assert_array_equal(idx.bins, before[0])
        np.testing.assert_array_equal(idx.signs, before[1])


class TestStorage:
    @pytest.mark.parametrize("name", ["d32_b4_L16_raw", "d24_b5_L12_raw",
                                      "d96_b2_nosign_L32", "flat_d16_b8"])
    def test_bytes_identical_to_reference(self, golden, tmp_path, name):
        from paper_2605_17415_b200.storage import load_index, save_index

        g = golden(name)
        idx = index_from_golden(g)
        idx.add_batch(g["x"])
        p = tmp_path / "a.ivtq"
        save_index(idx, p)
        assert p.read_bytes() == g["ivtq_bytes"].tobytes()
        # load the reference's own file, search identically
        q = tmp_path / "ref.ivtq"
        q.write_bytes(g["ivtq_bytes"].tobytes())
        loaded = load_index(q)
        k, n_p, rr = _search_keys(g)[0]
        a = idx.search_batch(g["queries"], k, n_p, rr)
        b = loaded.search_batch(g["queries"], k, n_p, rr)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])
        np.testing.assert_array_equal(loaded.bins, idx.bins)
        assert loaded.partition.lists == idx.partition.lists

    def test_corrupt_files(self, golden, tmp_path):
        from paper_2605_17415_b200.storage import IndexFormatError, load_index

        raw = golden("d32_b4_L16_raw")["ivtq_bytes"].tobytes()
        for bad in (b"NOPE" + raw[4:], raw[:-7], raw + b"\0"):
            p = tmp_path / "x.ivtq"
            p.write_bytes(bad)
            with pytest.raises(IndexFormatError):
                load_index(p)


class TestRefresh:
    @pytest.mark.parametrize("name,seed", [("refresh_recon", 3), ("refresh_raw", 4)])
    def test_refresh_matches_reference(self, golden, name, seed):
        from paper_2605_17415_b200.refresh import RefreshPolicy, refresh

        g = golden(name)
        idx = index_from_golden(g, "pre_")
        idx.add_batch(g["x"])
        fp = idx.compression_fingerprint()
        ext = idx.external_ids.copy()
        rep = refresh(idx, RefreshPolicy(seed=seed))
        ref = g["report"]
        assert rep.refreshed and rep.n_reassigned == int(ref[0])
        assert rep.sample_size == int(ref[1]) and rep.used_raw == bool(ref[2])
        np.testing.assert_array_equal(idx.partition.centroids, g["post_centroids"])
        np.testing.assert_array_equal(idx.list_ids, g["post_list_ids"])
        np.testing.assert_array_equal(idx.norms.view(np.uint16), g["post_norms"].view(np.uint16))
        np.testing.assert_array_equal(idx.bins, g["post_bins"])
        np.testing.assert_array_equal(idx.signs, g["post_signs"])
        np.testing.assert_allclose([rep.mean_assigned_ip_before, rep.mean_assigned_ip_after,
                                    rep.centroid_displacement_mean,
                                    rep.centroid_displacement_max], ref[3:], rtol=1e-9)
        assert idx.compression_fingerprint() == fp
        np.testing.assert_array_equal(idx.external_ids, ext)
        compare_topk(*idx.search_batch(g["queries"], 10, 8), g["s_10_8_0_ids"],
                     g["s_10_8_0_scores"])

    def test_empty_refresh_noop(self, golden):
        from paper_2605_17415_b200.refresh import RefreshPolicy, refresh

        idx = index_from_golden(golden("d16_b3_L8"))
        assert not refresh(idx, RefreshPolicy()).refreshed

    def test_reconstruct_matches_oracle(self, golden):
        from oracle import ivftq_oracle as orc
        from paper_2605_17415_b200.refresh import reconstruct_all, reconstruct_vector

        g = golden("d32_b4_L16_raw")
        idx = index_from_golden(g)
        idx.add_batch(g["x"])
        o = orc.OracleIndex(g["centroids"], g["R"], g["boundaries"], g["qcent"], g["half"])
        o.add_batch(g["x"])
        rec = reconstruct_all(idx)
        np.testing.assert_allclose(rec, orc.reconstruct_all(o), rtol=0, atol=1e-13)
        np.testing.assert_allclose(reconstruct_vector(idx, 123), rec[123], atol=1e-15)


@pytest.mark.parametrize("name", ["d32_b4_L16_raw", "d128_b4_L64", "d200_b3_L16"])
def test_train_partition_device_matches_reference(golden, name):
    """GPU k-means (csrc/kmeans.cu: seeding, tensor-core Lloyd assignment,
    in-order Lloyd sums) against the reference's own centroids
    (partition.py:64-178). The Lloyd sums and the normalisation are
    bit-identical by construction; the seeding's cdf / candidate scores and
    the exact assignment scores use a fixed summation order that is not
    OpenBLAS's, which can move a centroid by ulps of f64 before the f32 cast:
    the f32 centroids must agree to one f32 ulp, the memberships exactly."""
    from paper_2605_17415_b200.partition import train_partition

    g = golden(name)
    x = g["x"].astype(np.float64)
    xn = x / np.linalg.norm(x, axis=1)[:, None]
    L = int(g["config"][2])
    p = train_partition(xn, L, seed=int(g["config"][7]), device="cuda")
    np.testing.assert_allclose(p.centroids, g["centroids"], rtol=0, atol=2.0 ** -23)
    h = train_partition(xn, L, seed=int(g["config"][7]), device="cpu")
    assert [sorted(m) for m in p.lists] == [sorted(m) for m in h.lists]


def test_kmeans_sums_bit_identical_to_reduceat():
    """ivftq_kmeans_sums == np.add.reduceat over the stably sorted rows
    (partition.py:153-158), bit for bit, with empty lists and one long list."""
    import torch

    from paper_2605_17415_b200 import _lib

    L = _lib.lib()
    rng = np.random.default_rng(5)
    for n, d, k in [(5000, 24, 37), (70000, 96, 512), (300, 200, 4)]:
        x = rng.standard_normal((n, d))
        a = rng.integers(0, k, n).astype(np.int32)
        a[a == 3] = 2                      # list 3 empty
        a[: n // 3] = 1                    # one long list
        cnt = np.bincount(a, minlength=k)
        order = np.argsort(a, kind="stable")
        starts = np.concatenate(([0], np.cumsum(cnt)[:-1]))
        ne = np.flatnonzero(cnt > 0)
        want = np.zeros((k, d))
        want[ne] = np.add.reduceat(x[order], starts[ne], axis=0)
        X = torch.from_numpy(x).cuda()
        A = torch.from_numpy(a).cuda()
        sums = torch.empty((k, d), dtype=torch.float64, device="cuda")
        counts = torch.empty(k, dtype=torch.int32, device="cuda")
        nb = int(L.ivftq_kmeans_sums_scratch_bytes(n, k))
        scratch = torch.empty(nb, dtype=torch.uint8, device="cuda")
        _lib.check(L.ivftq_kmeans_sums(X.data_ptr(), A.data_ptr(), n, d, k, sums.data_ptr(),
                                       counts.data_ptr(), scratch.data_ptr(), nb, _lib.stream_ptr()))
        assert np.array_equal(counts.cpu().numpy(), cnt)
        assert np.array_equal(sums.cpu().numpy().view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("n,d,k", [(3000, 16, 8), (20000, 96, 64), (6000, 200, 33)])
def test_kmeanspp_seed_matches_host(n, d, k):
    """Device seeding picks the host's centres (partition.py:_kmeanspp) from
    the same generator stream."""
    import torch

    from paper_2605_17415_b200 import _lib
    from paper_2605_17415_b200.partition import _HostOps, _kmeanspp

    L = _lib.lib()
    rng = np.random.default_rng(n + k)
    x = rng.standard_normal((n, d))
    x /= np.linalg.norm(x, axis=1)[:, None]
    want = _kmeanspp(x, k, np.random.default_rng(77), _HostOps())
    g = np.random.default_rng(77)
    nc = int(L.ivftq_kmeanspp_candidates(k))
    assert nc == 2 + int(np.log2(k))
    first = int(g.integers(n))
    u = np.ascontiguousarray(g.random((k - 1, nc)))
    X = torch.from_numpy(x).cuda()
    chosen = torch.empty(k, dtype=torch.int64, device="cuda")
    tots = torch.empty(k, dtype=torch.float64, device="cuda")
    nb = int(L.ivftq_kmeanspp_scratch_bytes(n, d, k))
    scratch = torch.empty(nb, dtype=torch.uint8, device="cuda")
    _lib.check(L.ivftq_kmeanspp_seed(X.data_ptr(), n, d, k, first, u.ctypes.data, chosen.data_ptr(),
                                     tots.data_ptr(), scratch.data_ptr(), nb, _lib.stream_ptr()))
    got = x[chosen.cpu().numpy()]
    assert np.array_equal(got, want)
    assert float(tots[1:].min()) > 0


def test_train_partition_device_degenerate_and_repeatable():
    """Fewer distinct points than k takes the reference's checked seeding
    branch (partition.py:91-98) and its empty-list rule (partition.py:161-165).
    Which duplicate the rule re-seeds from hangs on the last ulp of equal
    scores (OpenBLAS's order on the host), so the check is structural: every
    centroid is one of the distinct points and each point keeps a list. Two
    runs agree bit for bit."""
    from paper_2605_17415_b200.partition import train_partition

    rng = np.random.default_rng(3)
    base = rng.standard_normal((6, 24))
    base /= np.linalg.norm(base, axis=1)[:, None]
    x = base[rng.integers(0, 6, 400)]
    p = train_partition(x, 8, seed=4, device="cuda")
    gap = np.abs(p.centroids[:, None, :].astype(np.float64) - base[None]).max(axis=2)
    assert np.all(gap.min(axis=1) <= 2.0 ** -23)
    assert set(gap.argmin(axis=1).tolist()) == set(range(6))
    assert sum(len(m) for m in p.lists) == len(x)
    y = rng.standard_normal((5000, 48))
    y /= np.linalg.norm(y, axis=1)[:, None]
    a = train_partition(y, 32, seed=9, device="cuda")
    b = train_partition(y, 32, seed=9, device="cuda")
    assert np.array_equal(a.centroids.view(np.uint32), b.centroids.view(np.uint32))
    assert a.lists == b.lists


@pytest.mark.parametrize("n,d,L", [(40000, 96, 64), (20000, 128, 32), (12000, 200, 16), (5000, 24, 8)])
def test_rotate_tc_error_inside_guard(n, d, L):
    """The tensor-core encoder quantises u' = (r/||r||).R^T computed on tcgen05
    and re-encodes in f64 every row with a coordinate within 2^-18 of a
    threshold. Pin the guard: |u' - u| against the f64 rotation stays below a
    quarter of it, and the binary16 norms are bit-exact (index.py:247-256)."""
    import torch

    from paper_2605_17415_b200 import _lib, generate_rotation

    Lb = _lib.lib()
    rng = np.random.default_rng(d)
    c = rng.standard_normal((L, d))
    c = (c / np.linalg.norm(c, axis=1)[:, None]).astype(np.float32)
    lid = rng.integers(0, L, n).astype(np.int32)
    x = c[lid].astype(np.float64) + rng.standard_normal((n, d)) * rng.uniform(1e-4, 0.3, (n, 1))
    x[:3] = c[lid[:3]]                      # zero residuals
    xn = x / np.linalg.norm(x, axis=1)[:, None]
    R = np.array(generate_rotation(d, 42).matrix, dtype=np.float64)
    r = xn - c[lid].astype(np.float64)
    rn = np.linalg.norm(r, axis=1)
    with np.errstate(invalid="ignore", divide="ignore"):
        want = np.where(rn[:, None] > 0, (r / rn[:, None]) @ R.T, 0.0)
    dev = "cuda"
    X = torch.from_numpy(xn).to(dev)
    C = torch.from_numpy(c).to(dev)
    Ld = torch.from_numpy(lid).to(dev)
    Rd = torch.from_numpy(R).to(dev)
    U = torch.empty((n, d), dtype=torch.float32, device=dev)
    nrm = torch.empty(n, dtype=torch.int16, device=dev)
    nb = int(Lb.ivftq_encode_tc_scratch_bytes(n, d))
    scratch = torch.empty(nb, dtype=torch.uint8, device=dev)
    assert Lb.ivftq_encode_supported_tc(d)
    _lib.check(Lb.ivftq_rotate_unit_tc(X.data_ptr(), C.data_ptr(), Ld.data_ptr(), n, d, 0,
                                       Rd.data_ptr(), U.data_ptr(), nrm.data_ptr(),
                                       scratch.data_ptr(), nb, _lib.stream_ptr()))
    got = U.cpu().numpy().astype(np.float64)
    live = rn > 1e-7
    err = np.abs(got[live] - want[live]).max()
    assert err < 2.0 ** -20, err
    assert np.array_equal(nrm.cpu().numpy().view(np.uint16), rn.astype(np.float16).view(np.uint16))


@pytest.mark.parametrize("d,bits", [(96, 4), (128, 4), (64, 2), (200, 3)])
def test_encoder_decides_near_threshold_coordinates_exactly(d, bits):
    """Rows built so that, after rotation, a third of their coordinates sit
    1e-9 .. 2e-6 above or below a Lloyd-Max decision threshold (bin boundary
    or half-bin centroid): far inside the tensor-core encoder's guard, far
    outside f64 summation noise. The guard must hand every such row to the
    exact pass, so bins and signs equal the oracle's (index.py:256-262,
    lloydmax.py:129-144)."""
    from oracle import ivftq_oracle as orc
    from paper_2605_17415_b200 import CoarsePartition, design_quantizer, generate_rotation
    from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex

    rng = np.random.default_rng(100 * d + bits)
    q = design_quantizer(bits, d)
    R = np.asarray(generate_rotation(d, 42).matrix, dtype=np.float64)
    thr = np.concatenate([np.asarray(q.boundaries, np.float64)[1:-1],
                          np.asarray(q.centroids, np.float64)])
    thr = thr[np.abs(thr) < 1.2 / np.sqrt(d)]        # inner thresholds: the row still has norm 1
    n, m = 3000, d // 3
    u = np.zeros((n, d))
    for i in range(n):
        near = rng.choice(d, m, replace=False)
        delta = rng.choice([1e-9, 1e-8, 1e-7, 2e-6], m) * rng.choice([-1.0, 1.0], m)
        u[i, near] = rng.choice(thr, m) + delta
        rest = np.setdiff1d(np.arange(d), near)
        room = 1.0 - np.sum(u[i, near] ** 2)
        assert room > 0
        v = rng.standard_normal(len(rest))
        u[i, rest] = v * np.sqrt(room) / np.linalg.norm(v)
    x = (u @ R) * rng.uniform(0.5, 2.0, (n, 1))      # rot = x~ . R^T = u up to f64 rounding
    ph = np.zeros((1, d), np.float32)
    ph[0, 0] = 1.0
    idx = IvfTqIndex(IndexConfig(dim=d, bits=bits, n_lists=1, flat=True), q,
                     generate_rotation(d, 42), CoarsePartition(1, d, ph))
    idx.add_batch(x)
    o = orc.OracleIndex(ph, R, q.boundaries, q.centroids, q.half_bin_means, flat=True)
    o.add_batch(x)
    # the construction really is adversarial for an unguarded f32 decision
    un = x / np.linalg.norm(x, axis=1)[:, None]
    rot = un @ R.T
    rot /= np.linalg.norm(rot, axis=1)[:, None]
    gap = np.abs(rot[:, :, None] - thr[None, None, :]).min(axis=2)
    assert (gap < 3e-6).mean() > 0.25
    assert np.array_equal(idx.bins, o.bins)
    assert np.array_equal(idx.signs, o.signs)
    assert np.array_equal(idx.norms.view(np.uint16), o.norms.view(np.uint16))


def _coarse_case(seed, n, L, d, dup=True):
    rng = np.random.default_rng(seed)
    c = rng.standard_normal((L, d))
    if dup and L >= 8:
        c[L // 2] = c[1]            # exact duplicate centroid: ties -> lower list
        c[L - 1] = c[1] * (1 + 1e-9)  # near-duplicate inside the guard band
    c = (c / np.linalg.norm(c, axis=1)[:, None]).astype(np.float32)
    x = rng.standard_normal((n, d))
    m = min(5, n, L)
    x[:m] = c[:m]  # rows sitting on centroids
    x /= np.linalg.norm(x, axis=1)[:, None]
    return x, c


def _with_mode(L, mode, fn):
    L.ivftq_set_coarse_mode(mode)
    try:
        return fn()
    finally:
        L.ivftq_set_coarse_mode(0)


@pytest.mark.parametrize("n,L,d,n_p,crowd", [
    (300, 64, 32, 8, 0), (1000, 1024, 128, 64, 0), (257, 300, 96, 33, 0), (128, 130, 200, 1, 0),
    (64, 4096, 96, 128, 0), (10, 16, 7, 16, 0), (2000, 4096, 96, 32, 0),
    # every centroid a copy of a few: > 256 in-band candidates -> exact full-row path
    (40, 600, 16, 10, 3),
    # more lists than the fused selection stages per row -> band/exact/pick kernels
    (30, 20000, 16, 8, 0),
    # scores rising with the list id (an adversarial column order)
    (16, 4096, 16, 8, -1), (16, 4096, 16, 100, -1)])
def test_coarse_tc_probes_identical_to_f64(n, L, d, n_p, crowd):
    """Tensor-core coarse scores + exact guard band == the f64 GEMM path:
    identical probe lists (stable order); coarse values are exact f64 dot
    products in a different summation order (lane-split tree vs sequential
    chain), so they agree to a few ulps."""
    import torch

    from paper_2605_17415_b200 import _lib

    lib = _lib.lib()
    x, c = _coarse_case(n + L + d, n, L, d)
    if crowd > 0:
        c = c[np.arange(L) % crowd].copy()
    elif crowd < 0:
        th = np.linspace(1.2, 0.0, L)
        c = np.zeros((L, d))
        c[:, 0], c[:, 1] = np.cos(th), np.sin(th)
        c = c.astype(np.float32)
        x = np.tile(np.eye(d)[:1], (n, 1)) + 1e-3 * np.random.default_rng(7).standard_normal((n, d))
        x /= np.linalg.norm(x, axis=1)[:, None]
    xd = torch.from_numpy(x).cuda()
    cd = torch.from_numpy(c).cuda()

    def run():
        probe = torch.empty((n, n_p), dtype=torch.int32, device="cuda")
        coarse = torch.empty((n, n_p), dtype=torch.float64, device="cuda")
        sb = lib.ivftq_probe_scratch_bytes(n, L, d)
        scr = torch.empty(sb, dtype=torch.uint8, device="cuda")
        _lib.check(lib.ivftq_probe(xd.data_ptr(), cd.data_ptr(), n, L, d, n_p, probe.data_ptr(),
                                   coarse.data_ptr(), scr.data_ptr(), sb, _lib.stream_ptr()))
        torch.cuda.synchronize()
        return probe.cpu().numpy(), coarse.cpu().numpy()

    assert lib.ivftq_coarse_tc_supported(d, L) == 1
    p_tc, c_tc = _with_mode(lib, 2, run)
    p_64, c_64 = _with_mode(lib, 1, run)
    np.testing.assert_array_equal(p_tc, p_64)
    np.testing.assert_allclose(c_tc, c_64, rtol=0, atol=1e-14)
    # and against numpy's stable argsort of the f64 scores
    s = x @ c.astype(np.float64).T
    want = np.argsort(-s, axis=1, kind="stable")[:, :n_p]
    np.testing.assert_array_equal(p_tc, want)


@pytest.mark.parametrize("n,L,d", [(5000, 1024, 128), (777, 33, 64), (300, 4096, 96),
                                   (200, 8, 200), (50, 3, 5)])
def test_assign_tc_identical_to_f64(n, L, d):
    import torch

    from paper_2605_17415_b200 import _lib

    lib = _lib.lib()
    x, c = _coarse_case(n * 7 + L, n, L, d)
    xd = torch.from_numpy(x).cuda()
    cd = torch.from_numpy(c).cuda()
    out_tc = torch.empty(n, dtype=torch.int32, device="cuda")
    out_64 = torch.empty(n, dtype=torch.int32, device="cuda")
    sb = lib.ivftq_assign_tc_scratch_bytes(n, L, d)
    scr = torch.empty(sb, dtype=torch.uint8, device="cuda")
    _lib.check(lib.ivftq_assign_tc(xd.data_ptr(), cd.data_ptr(), n, L, d, out_tc.data_ptr(),
                                   scr.data_ptr(), sb, _lib.stream_ptr()))
    _lib.check(lib.ivftq_assign(xd.data_ptr(), cd.data_ptr(), n, L, d, out_64.data_ptr(),
                                _lib.stream_ptr()))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out_tc.cpu().numpy(), out_64.cpu().numpy())
    np.testing.assert_array_equal(out_tc.cpu().numpy(),
                                  np.argmax(x @ c.astype(np.float64).T, axis=1))


def test_pipelined_host_ingest_equals_plain(golden):
    """Large host batches are encoded in sub-chunks while the next one copies;
    the stored fields must equal a plain add, and a zero row anywhere must
    still raise with its batch-wide index before anything is appended."""
    import torch

    g = golden("d128_b4_L64")
    x = g["x"].astype(np.float32)
    a = index_from_golden(g)
    a.add_batch(x)
    b = index_from_golden(g)
    b._PIPE_ROWS = 256  # force several sub-chunks
    b.add_batch(torch.from_numpy(x).pin_memory())
    np.testing.assert_array_equal(a.list_ids, b.list_ids)
    np.testing.assert_array_equal(a.bins, b.bins)
    np.testing.assert_array_equal(a.signs, b.signs)
    np.testing.assert_array_equal(a.norms.view(np.uint16), b.norms.view(np.uint16))
    c = index_from_golden(g)
    c._PIPE_ROWS = 256
    bad = x.copy()
    bad[700] = 0
    with pytest.raises(ValueError, match="row at index 700"):
        c.add_batch(torch.from_numpy(bad))
    assert c.count == 0


@pytest.mark.parametrize("k,n_p,nq", [(50, 64, 100), (33, 8, 100), (10, 64, 100), (1, 1, 100),
                                      (10, 4, 0), (10, 16, 1), (5, 200, 70)])
def test_search_shapes_against_oracle(golden, k, n_p, nq):
    """Depths past the tensor-core range (k > 32), every list probed, empty and
    single-query batches, n_p clamped above L -- all against the oracle."""
    import warnings as w_

    from oracle import ivftq_oracle as orc

    g = golden("d128_b4_L64")
    idx = index_from_golden(g)
    idx.add_batch(g["x"])
    o = orc.OracleIndex(g["centroids"], g["R"], g["boundaries"], g["qcent"], g["half"])
    o.add_batch(g["x"])
    rng = np.random.default_rng(k * 1000 + n_p)
    q = g["x"][rng.integers(0, len(g["x"]), nq)] + 0.05 * rng.standard_normal((nq, 128))
    with w_.catch_warnings():
        w_.simplefilter("ignore")
        ids, sc = idx.search_batch(q.reshape(nq, 128), k, n_p)
    assert ids.shape == (nq, k) and sc.shape == (nq, k)
    if nq:
        ref_i, ref_s = o.search_batch(q, k, min(n_p, 64))
        compare_topk(ids, sc, ref_i, ref_s)


def test_query_chunking_equals_single_call(golden):
    """Batches above the per-call query chunk are split; results are identical."""
    g = golden("d128_b4_L64")
    idx = index_from_golden(g)
    idx.add_batch(g["x"])
    q = np.tile(g["queries"], (3, 1))
    a_i, a_s = idx.search_batch(q, 10, 8)
    idx._QUERY_CHUNK = 128
    b_i, b_s = idx.search_batch(q, 10, 8)
    np.testing.assert_array_equal(a_i, b_i)
    np.testing.assert_array_equal(a_s, b_s)


def test_graph_replay_equals_eager(golden):
    """Repeated same-shape searches replay a captured CUDA graph: results equal
    the eager path call after call, with fresh inputs, and the graphs are
    dropped (re-captured) once the index changes."""
    import torch

    g = golden("d128_b4_L64")
    idx = index_from_golden(g)
    half = len(g["x"]) // 2
    idx.add_batch(g["x"][:half])
    rng = np.random.default_rng(5)

    def both(q):
        qt = torch.from_numpy(q).cuda()
        idx.use_graphs = False
        e = idx.search_batch(qt, 10, 8)
        idx.use_graphs = True
        r = idx.search_batch(qt, 10, 8)
        return e, r

    for _ in range(3):  # capture, then replays with new inputs
        q = g["x"][rng.integers(0, half, 300)] + 0.05 * rng.standard_normal((300, 128))
        (ei, es), (ri, rs) = both(q)
        np.testing.assert_array_equal(ei, ri)
        np.testing.assert_array_equal(es, rs)
    assert len(idx._thread_state().graphs) == 1
    dev_ids, _ = idx.search_batch(torch.from_numpy(q).cuda(), 10, 8, return_device=True)
    idx.search_batch(torch.from_numpy(q[::-1].copy()).cuda(), 10, 8)  # next replay
    np.testing.assert_array_equal(dev_ids.cpu().numpy(), ei)  # returned tensors are owned
    idx.add_batch(g["x"][half:])  # index changed: graphs re-captured
    q = g["x"][rng.integers(0, len(g["x"]), 300)]
    (ei, es), (ri, rs) = both(q)
    np.testing.assert_array_equal(ei, ri)
    np.testing.assert_array_equal(es, rs)
    assert ei.max() >= half  # the new rows are searched
    with pytest.raises(ValueError, match="zero-norm"):
        z = torch.from_numpy(q).cuda().clone()
        z[7] = 0
        idx.search_batch(z, 10, 8)


def test_graph_replay_with_kernel_timing(golden):
    """Toggling the scan-kernel timing between graph replays: the timed search
    reports a kernel time (its graph is captured with the events), and
    searches of other shapes afterwards still run (no stale CUDA error)."""
    import torch

    from paper_2605_17415_b200 import _lib

    g = golden("d128_b4_L64")
    idx = index_from_golden(g)
    idx.add_batch(g["x"])
    q = torch.from_numpy(g["x"][:512] + 0.01).cuda()
    lib = _lib.lib()
    idx.search_batch(q, 10, 8, return_device=True)
    lib.ivftq_set_kernel_timing(1)
    try:
        idx.search_batch(q, 10, 8, return_device=True)
        ms = lib.ivftq_last_scan_kernel_ms()
    finally:
        lib.ivftq_set_kernel_timing(0)
    assert ms > 0
    a = idx.search_batch(q[:300], 10, 16)
    idx.use_graphs = False
    b = idx.search_batch(q[:300], 10, 16)
    np.testing.assert_array_equal(a[0], b[0])


def test_external_ids_default_and_custom(golden, tmp_path):
    """External ids default to the internal ones (index.py:299-303) and are
    only materialised once a caller passes its own; mixed batches, search
    results (internal ids) and save/load keep them."""
    from paper_2605_17415_b200.storage import load_index, save_index

    g = golden("d32_b4_L16_raw")
    idx = index_from_golden(g)
    x = g["x"]
    assert idx.add_batch(x[:100]).tolist() == list(range(100))
    assert idx._ext is None
    np.testing.assert_array_equal(idx.external_ids, np.arange(100))
    idx.add_batch(x[100:150], external_ids=np.arange(1000, 1050))
    idx.add_batch(x[150:200])
    want = np.concatenate([np.arange(100), np.arange(1000, 1050), np.arange(150, 200)])
    np.testing.assert_array_equal(idx.external_ids, want)
    assert idx.add(x[200], external_id=77) == 200
    np.testing.assert_array_equal(idx.external_ids[-1:], [77])
    p = tmp_path / "ext.ivtq"
    save_index(idx, p)
    back = load_index(p)
    np.testing.assert_array_equal(back.external_ids, idx.external_ids)
