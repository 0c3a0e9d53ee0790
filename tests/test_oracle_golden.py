"""Pin the CPU oracle (oracle/ivftq_oracle.py) to the reference's outputs.

Golden vectors come from running the reference itself
(tests/golden/make_golden.py). Inline known-answer tests restate the
reference's own KATs (test_index.py:30-46, test_lloydmax.py:150-190,
test_evaluation.py:44-55).
"""

import numpy as np
import pytest

from oracle import ivftq_oracle as orc

SMALL = ["d32_b4_L16_raw", "d16_b3_L8", "d24_b5_L12_raw", "d96_b2_nosign_L32",
         "d200_b3_L16", "d64_b8_L8", "d40_b1_L4", "d128_b4_L64", "flat_d16_b8"]


def oracle_from(g, prefix=""):
    cfg = g[prefix + "config"]
    return orc.OracleIndex(g[prefix + "centroids"], g[prefix + "R"],
                           g[prefix + "boundaries"], g[prefix + "qcent"],
                           g[prefix + "half"], use_sign=bool(cfg[3]),
                           flat=bool(cfg[5]), keep_raw=bool(cfg[4]))


def search_keys(g):
    out = []
    for k in g:
        if k.startswith("s_") and k.endswith("_ids"):
            _, kk, p, rr, _ = k.split("_")
            out.append((int(kk), int(p), int(rr)))
    return out


@pytest.mark.parametrize("name", SMALL)
def test_oracle_encode_matches_reference(golden, name):
    g = golden(name)
    o = oracle_from(g)
    o.add_batch(g["x"])
    np.testing.assert_array_equal(o.list_ids, g["list_ids"])
    np.testing.assert_array_equal(o.norms.view(np.uint16), g["norms"].view(np.uint16))
    np.testing.assert_array_equal(o.bins, g["bins"])
    np.testing.assert_array_equal(o.signs, g["signs"])


@pytest.mark.parametrize("name", SMALL)
def test_oracle_search_matches_reference(golden, name):
    g = golden(name)
    o = oracle_from(g)
    o.add_batch(g["x"])
    if g["config"][4]:
        np.testing.assert_array_equal(o.raw, g["raw"])
    for (k, n_p, rr) in search_keys(g):
        ids, sc = o.search_batch(g["queries"], k, n_p, rr)
        np.testing.assert_array_equal(ids, g[f"s_{k}_{n_p}_{rr}_ids"])
        np.testing.assert_allclose(sc, g[f"s_{k}_{n_p}_{rr}_scores"], rtol=1e-12,
                                   atol=0)


@pytest.mark.parametrize("name", ["d32_b4_L16_raw", "d16_b3_L8", "d200_b3_L16"])
def test_oracle_kmeans_matches_reference(golden, name):
    g = golden(name)
    cfg = g["config"]
    xn = orc.normalize_rows(g["x"])
    # IvfTqIndex.build normalises then trains with default 25 iterations
    cent = orc.train_partition(xn, int(cfg[2]), seed=int(cfg[7]))
    np.testing.assert_array_equal(cent, g["centroids"])


def test_oracle_probes_match_reference(golden):
    g = golden("d128_b4_L64")
    o = oracle_from(g)
    probe, coarse = o.probes(g["queries"], 64)
    np.testing.assert_array_equal(probe, g["probe_all"][:, :64])
    np.testing.assert_allclose(coarse, np.take_along_axis(g["coarse"], probe, 1),
                               rtol=0, atol=1e-15)


@pytest.mark.parametrize("name", ["refresh_recon", "refresh_raw"])
def test_oracle_refresh_matches_reference(golden, name):
    g = golden(name)
    o = oracle_from(g, "pre_")
    o.add_batch(g["x"])
    np.testing.assert_array_equal(o.bins, g["pre_bins"])
    n_lists = int(g["pre_config"][2])
    used_raw = bool(g["report"][2])
    if used_raw:
        src = o.raw.astype(np.float64)
        src = src / np.linalg.norm(src, axis=1)[:, None]
    else:
        src = orc.reconstruct_all(o)
    n = o.count
    sample = min(n, max(100 * n_lists, n // 10))
    seed = 3 if name == "refresh_recon" else 4
    rng = np.random.default_rng(seed)
    ids = orc.stratified_sample_ids(o.members(), n, n_lists, sample, rng)
    np.testing.assert_array_equal(ids, g["sample_ids"])
    cent = orc.train_partition(src[ids], n_lists, seed=seed)
    np.testing.assert_array_equal(cent, g["post_centroids"])
    orc.refresh_encode(o, src, cent)
    np.testing.assert_array_equal(o.list_ids, g["post_list_ids"])
    np.testing.assert_array_equal(o.bins, g["post_bins"])
    np.testing.assert_array_equal(o.signs, g["post_signs"])
    np.testing.assert_array_equal(o.norms.view(np.uint16),
                                  g["post_norms"].view(np.uint16))
    np.testing.assert_array_equal(np.concatenate(o.members()), g["post_lists"])
    ids_, sc = o.search_batch(g["queries"], 10, 8)
    np.testing.assert_array_equal(ids_, g["s_10_8_0_ids"])


def test_oracle_exact_topk_and_recall(golden):
    g = golden("d32_b4_L16_raw")
    xn = orc.normalize_rows(g["x"])
    t = orc.exact_topk(xn, g["queries"], 10)
    np.testing.assert_array_equal(t, g["truth10"])
    assert orc.recall_at_k(t, g["truth10"], 10) == 1.0


class TestKnownAnswers:
    def test_packing_kat(self):
        # test_index.py:39-42: fields [0x3, 0xA] at width 4 -> byte 0xA3
        assert orc.pack_fields(np.array([[0x3, 0xA]], np.uint8), 4).tolist() == [[0xA3]]

    @pytest.mark.parametrize("width", [1, 2, 3, 4, 5, 7, 8])
    def test_pack_round_trip(self, width):
        rng = np.random.default_rng(width)
        v = rng.integers(0, 1 << width, size=(50, 37), dtype=np.uint8)
        p = orc.pack_fields(v, width)
        assert p.shape == (50, -(-37 * width // 8))
        np.testing.assert_array_equal(orc.unpack_fields(p, width, 37), v)

    def test_quantize_kats(self, golden):
        t = golden("tables")
        bnd, cent = t["b4_d32_bnd"], t["b4_d32_cent"]
        # test_lloydmax.py:150-167: centroid -> (k, 1); 0.0 -> bin 8; huge -> top
        for kk in range(16):
            b, s = orc.quantize(np.array([cent[kk]]), bnd, cent)
            assert (int(b[0]), int(s[0])) == (kk, 1)
        b, _ = orc.quantize(np.array([0.0, -0.0, 10.0, -10.0]), bnd, cent)
        assert b.tolist() == [8, 8, 15, 0]
        # boundary tie -> upper bin
        b, _ = orc.quantize(bnd[1:-1], bnd, cent)
        assert b.tolist() == list(range(1, 16))

    def test_golden_packing_matches_reference_file(self, golden):
        # codes inside the reference's own .ivtq bytes (storage.py:282-283)
        g = golden("d24_b5_L12_raw")
        n, d, bits = len(g["list_ids"]), 24, 5
        raw = g["ivtq_bytes"].tobytes()
        cb = -(-bits * d // 8)
        sb = -(-d // 8)
        tail = 4 * n * d  # raw store at the end
        codes = np.frombuffer(raw[-(tail + n * (cb + sb)):-(tail + n * sb)], np.uint8)
        np.testing.assert_array_equal(codes.reshape(n, cb),
                                      orc.pack_fields(g["bins"], bits))


@pytest.mark.slow
def test_oracle_pr1_encode_and_search(golden):
    """Full PR1 config (100k x 128, L=256): encode + search at n_p 16."""
    from paper_2605_17415_b200.workloads import make_workload
    import sys
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).parent / "golden"))
    g = golden("pr1")
    w = make_workload("pr1")
    o = oracle_from(g)
    o.add_batch(w.base())
    np.testing.assert_array_equal(o.list_ids, g["list_ids"].astype(np.int64))
    np.testing.assert_array_equal(o.norms.view(np.uint16), g["norms"].view(np.uint16))
    packed = np.concatenate([orc.pack_fields(o.bins, 4), orc.pack_fields(o.signs, 1)], 1)
    from hashing import row_hash
    np.testing.assert_array_equal(row_hash(packed), g["code_hash"])
    ids, sc = o.search_batch(w.queries(), 10, 16)
    np.testing.assert_array_equal(ids, g["s_10_16_0_ids"])
    np.testing.assert_allclose(sc, g["s_10_16_0_scores"], rtol=1e-12)
