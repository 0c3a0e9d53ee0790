"""ctypes binding of libivftq_b200.so (the C ABI in include/ivftq_b200.h).

This is the host side of the drop-in boundary: Python owns every device
buffer (torch tensors used purely as allocations) and passes raw pointers and
the current CUDA stream. There is no CPU fallback: if the library or a GPU is
missing, `lib()` raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "lib" / "libivftq_b200.so"

IVFTQ_F32 = 0
IVFTQ_F64 = 1

_vp = C.c_void_p
_i32 = C.c_int
_i64 = C.c_int64
_sz = C.c_size_t


class IvftqStore(C.Structure):
    """Mirror of `ivftq_store` (include/ivftq_b200.h)."""

    _fields_ = [
        ("dim", C.c_int32),
        ("bits", C.c_int32),
        ("use_sign", C.c_int32),
        ("n_lists", C.c_int32),
        ("field_bits", C.c_int32),
        ("fields_per_word", C.c_int32),
        ("words_per_vec", C.c_int32),
        ("max_list_size", C.c_int32),
        ("list_offset", _vp),
        ("list_size", _vp),
        ("codes", _vp),
        ("norms", _vp),
        ("ids", _vp),
        ("capacity", C.c_int64),
    ]


_SIGS = {
    "ivftq_last_error": (C.c_char_p, []),
    "ivftq_abi_version": (_i32, []),
    "ivftq_launch_count": (C.c_ulonglong, []),
    "ivftq_note_graph_launches": (None, [C.c_ulonglong]),
    "ivftq_code_layout": (_i32, [_i32, _i32, _i32, C.POINTER(_i32), C.POINTER(_i32),
                                 C.POINTER(_i32)]),
    "ivftq_host_double_to_half": (_i32, [_vp, _i64, _vp]),
    "ivftq_host_row_norms": (_i32, [_vp, _i64, _i32, _vp]),
    "ivftq_normalize_rows": (_i32, [_vp, _i32, _i64, _i32, _vp, _vp, _vp]),
    "ivftq_gemm_nt": (_i32, [_vp, _vp, _i32, _i64, _i32, _i32, _vp, _i32, _vp]),
    "ivftq_assign": (_i32, [_vp, _vp, _i64, _i32, _i32, _vp, _vp]),
    "ivftq_residuals": (_i32, [_vp, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp]),
    "ivftq_quantize_pack": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "ivftq_encode_scratch_bytes": (_sz, [_i64, _i32, _i32]),
    "ivftq_encode_supported_tc": (_i32, [_i32]),
    "ivftq_encode_tc_scratch_bytes": (_sz, [_i64, _i32]),
    "ivftq_rotate_unit_tc": (_i32, [_vp, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "ivftq_encode_tail_tc": (_i32, [_vp, _vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp,
                                    _vp, _vp, _vp, _sz, _vp]),
    "ivftq_encode": (_i32, [_vp, _i32, _i64, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _vp,
                            _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "ivftq_pack_codes": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp]),
    "ivftq_histogram": (_i32, [_vp, _i64, _i32, _vp, _vp]),
    "ivftq_append": (_i32, [C.POINTER(IvftqStore), _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "ivftq_relayout": (_i32, [C.POINTER(IvftqStore), C.POINTER(IvftqStore), _vp, _vp]),
    "ivftq_export_codes": (_i32, [C.POINTER(IvftqStore), _vp, _i64, _i64, _vp, _vp, _vp]),
    "ivftq_xor_codes": (_i32, [C.POINTER(IvftqStore), _vp, _i64, _vp, _i32, _i32, _vp]),
    "ivftq_select_topn": (_i32, [_vp, _i64, _i32, _i32, _vp, _vp, _vp]),
    "ivftq_probe_scratch_bytes": (_sz, [_i64, _i32, _i32]),
    "ivftq_assign_tc_scratch_bytes": (_sz, [_i64, _i32, _i32]),
    "ivftq_assign_tc": (_i32, [_vp, _vp, _i64, _i32, _i32, _vp, _vp, _sz, _vp]),
    "ivftq_assign_tc64": (_i32, [_vp, _vp, _i64, _i32, _i32, _vp, _vp, _sz, _vp]),
    "ivftq_kmeanspp_candidates": (_i32, [_i32]),
    "ivftq_kmeanspp_scratch_bytes": (_sz, [_i64, _i32, _i32]),
    "ivftq_kmeanspp_seed": (_i32, [_vp, _i64, _i32, _i32, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "ivftq_kmeans_sums_scratch_bytes": (_sz, [_i64, _i32]),
    "ivftq_kmeans_sums": (_i32, [_vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _sz, _vp]),
    "ivftq_rowdot64": (_i32, [_vp, _vp, _vp, _i64, _i32, _vp, _vp]),
    "ivftq_lists_differ": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "ivftq_set_coarse_mode": (_i32, [_i32]),
    "ivftq_coarse_tc_supported": (_i32, [_i32, _i32]),
    "ivftq_coarse_prep_bytes": (_sz, [_i32, _i32]),
    "ivftq_coarse_prepare": (_i32, [_vp, _i32, _i32, _vp, _vp]),
    "ivftq_probe": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _sz, _vp]),
    "ivftq_probe_prepared": (_i32, [_vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _sz,
                                    _vp]),
    "ivftq_scan_scratch_bytes": (_sz, [_i64, _i32, _i32, _i32]),
    "ivftq_scan_topk": (_i32, [C.POINTER(IvftqStore), _vp, _vp, _vp, _vp, _i64, _i32, _i32,
                               _vp, _vp, _vp, _sz, _vp]),
    "ivftq_scan_topk_lut": (_i32, [C.POINTER(IvftqStore), _vp, _vp, _vp, _vp, _i64, _i32, _i32,
                                   _vp, _vp, _vp, _sz, _vp]),
    "ivftq_scan_topk_tc": (_i32, [C.POINTER(IvftqStore), _vp, _vp, _vp, _vp, _i64, _i32, _i32,
                                  _vp, _vp, _vp, _sz, _vp]),
    "ivftq_scan_tc_supported": (_i32, [_i32, _i32, _i32]),
    "ivftq_get_kernel_timing": (_i32, []),
    "ivftq_set_kernel_timing": (_i32, [_i32]),
    "ivftq_last_scan_kernel_ms": (C.c_double, []),
    "ivftq_last_scan_kernel": (C.c_char_p, []),
    "ivftq_scan_tc_scratch_bytes": (_sz, [_i64, _i32, _i32, _i32]),
    "ivftq_rerank": (_i32, [_vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp]),
    "ivftq_decode_scratch_bytes": (_sz, [_i64, _i32]),
    "ivftq_rowdot": (_i32, [_vp, _vp, _vp, _i64, _i32, _vp, _vp]),
    "ivftq_decode": (_i32, [C.POINTER(IvftqStore), _vp, _vp, _i64, _vp, _vp, _vp, _i32, _i32,
                            _vp, _vp, _sz, _vp]),
}

EXPORTS = tuple(_SIGS)

_LIB = None


class IvftqError(RuntimeError):
    """A C-ABI call returned an error code."""


def load(path: str | os.PathLike | None = None):
    """Load the shared library (no GPU needed) and bind every signature."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path else Path(os.environ.get("IVFTQ_LIB", LIB_PATH))
    if not p.exists():
        raise FileNotFoundError(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _LIB = lib
    return lib


def check(rc: int, what: str = ""):
    if rc != 0:
        msg = load().ivftq_last_error().decode(errors="replace")
        raise IvftqError(f"{what}: {msg} (code {rc})")


def lib():
    """The loaded library; requires a CUDA device for any compute entry point."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2605_17415_b200 needs a CUDA GPU (B200); no CPU fallback")
    return load()


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
