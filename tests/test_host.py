"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
host-side numerics helpers match numpy bit-for-bit, host modules match the
reference's fixed inputs, and the API validates like the reference."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2605_17415_b200 import _lib
from paper_2605_17415_b200.quantizer import design_quantizer
from paper_2605_17415_b200.rotation import generate_rotation

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    return _lib.load()


def test_library_exports_every_header_symbol(lib):
    header = (ROOT / "include" / "ivftq_b200.h").read_text()
    declared = set(re.findall(r"\b(ivftq_[a-z0-9_]+)\s*\(", header))
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    assert lib.ivftq_abi_version() == 3


def test_code_layout(lib):
    from paper_2605_17415_b200.store import code_layout

    assert code_layout(96, 4, True) == (5, 6, 16)
    assert code_layout(128, 4, True) == (5, 6, 22)
    assert code_layout(200, 3, True) == (4, 8, 25)
    assert code_layout(200, 2, True) == (3, 10, 20)
    assert code_layout(64, 8, True) == (9, 3, 22)
    assert code_layout(16, 4, False) == (5, 6, 3)


def test_host_double_to_half_matches_numpy(lib):
    rng = np.random.default_rng(0)
    x = np.concatenate([
        rng.uniform(0, 2, 200000), rng.uniform(0, 1e-4, 100000),
        np.exp(rng.uniform(-40, 12, 100000)),
        [0.0, -0.0, 1.0, 65504.0, 65519.99, 65520.0, 1e6, 2 ** -24, 2 ** -25,
         2 ** -25 * 1.0000001, 2 ** -14, 2 ** -14 * (1 - 2 ** -12), 0.5 + 2 ** -12,
         0.5 + 3 * 2 ** -12, np.inf, -np.inf, -1.5, -2 ** -20, 6.1e-5, 5.96e-8]])
    # exact ties at every binary16 rounding boundary
    h = np.arange(0, 0x7bff, dtype=np.uint16).view(np.float16).astype(np.float64)
    mids = (h[:-1] + h[1:]) / 2
    x = np.concatenate([x, mids, -mids])
    out = np.zeros(len(x), dtype=np.uint16)
    assert lib.ivftq_host_double_to_half(x.ctypes.data, len(x), out.ctypes.data) == 0
    np.testing.assert_array_equal(out, x.astype(np.float16).view(np.uint16))


@pytest.mark.parametrize("d", [2, 3, 7, 8, 9, 16, 31, 96, 128, 129, 200, 257, 1000])
def test_host_row_norms_match_numpy_pairwise(lib, d):
    rng = np.random.default_rng(d)
    x = rng.standard_normal((300, d)) * np.exp(rng.uniform(-5, 5, (300, 1)))
    out = np.zeros(300)
    lib.ivftq_host_row_norms(x.ctypes.data, 300, d, out.ctypes.data)
    np.testing.assert_array_equal(out, np.linalg.norm(x, axis=1))


@pytest.mark.parametrize("bits", [1, 2, 3, 4, 5, 6])
def test_quantizer_tables_bit_identical(golden, bits):
    t = golden("tables")
    for d in (16, 32, 96, 128, 200):
        q = design_quantizer(bits, d)
        np.testing.assert_array_equal(q.boundaries, t[f"b{bits}_d{d}_bnd"])
        np.testing.assert_array_equal(q.centroids, t[f"b{bits}_d{d}_cent"])
        np.testing.assert_array_equal(q.half_bin_means, t[f"b{bits}_d{d}_half"])
        np.testing.assert_array_equal([q.distortion, q.distortion_sign], t[f"b{bits}_d{d}_dist"])


@pytest.mark.parametrize("d", [16, 24, 32, 96, 128, 200])
def test_rotation_bit_identical(golden, d):
    np.testing.assert_array_equal(generate_rotation(d, 42).matrix, golden("tables")[f"rot_{d}"])


@pytest.mark.parametrize("name", ["d32_b4_L16_raw", "d16_b3_L8", "d200_b3_L16"])
def test_train_partition_bit_identical(golden, name):
    from paper_2605_17415_b200.partition import train_partition

    g = golden(name)
    x = g["x"].astype(np.float64)
    xn = x / np.linalg.norm(x, axis=1)[:, None]
    p = train_partition(xn, int(g["config"][2]), seed=int(g["config"][7]))
    np.testing.assert_array_equal(p.centroids, g["centroids"])


def test_pack_unpack_kat_and_round_trip():
    from paper_2605_17415_b200.index import pack_fields, unpack_fields

    assert pack_fields(np.array([[0x3, 0xA]], np.uint8), 4).tolist() == [[0xA3]]
    for w in (1, 2, 3, 4, 5, 7, 8):
        rng = np.random.default_rng(w)
        v = rng.integers(0, 1 << w, size=(200, 37), dtype=np.uint8)
        np.testing.assert_array_equal(unpack_fields(pack_fields(v, w), w, 37), v)
    with pytest.raises(ValueError):
        pack_fields(np.zeros((1, 4), np.uint8), 9)


def test_config_validation():
    from paper_2605_17415_b200.index import IndexConfig

    for kw in (dict(dim=1, bits=4, n_lists=4), dict(dim=8, bits=0, n_lists=4),
               dict(dim=8, bits=9, n_lists=4), dict(dim=8, bits=4, n_lists=0),
               dict(dim=8, bits=4, n_lists=2, flat=True)):
        with pytest.raises(ValueError):
            IndexConfig(**kw)
    c = IndexConfig(dim=8, bits=4, n_lists=2)
    assert (c.use_sign_bit, c.keep_raw, c.flat, c.rotation_seed, c.kmeans_seed) == (
        True, False, False, 42, 42)


def test_no_gpu_means_loud_failure():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.lib()


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2605_17415_b200"
    for p in pkg.rglob("*.py"):
        assert not re.search(r"^\s*(from|import)\s+\.*oracle", p.read_text(), re.M), p
        assert "ivftq_oracle" not in p.read_text(), p


def test_load_rejects_out_of_range_list_id(golden, tmp_path):
    """A corrupt list id fails cleanly before any device work (ADVICE r1:
    the id would index device list buffers)."""
    import struct

    from paper_2605_17415_b200.storage import _CFG, IndexFormatError, load_index

    raw = bytearray(golden("d32_b4_L16_raw")["ivtq_bytes"].tobytes())
    dim, bits, n_lists, flags, _, _, count = struct.unpack_from(_CFG, raw, 6)
    lv = 1 << bits
    off = 6 + struct.calcsize(_CFG) + 8 * (lv + 1 + lv + 2 * lv) + 16 + 8 * dim * dim \
        + 4 * n_lists * dim
    for bad in (n_lists, 0x80000000):
        b = bytearray(raw)
        struct.pack_into("<I", b, off + 4 * 3, bad)  # list id of vector 3
        p = tmp_path / "x.ivtq"
        p.write_bytes(bytes(b))
        with pytest.raises(IndexFormatError, match="list id .* of vector 3 out of range"):
            load_index(p)
