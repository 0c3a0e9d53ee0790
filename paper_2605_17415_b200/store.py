"""Device-resident inverted lists (host-side owner of the `ivftq_store` buffers).

Replaces the reference's per-vector `_Rows` buffers plus the Python member
lists (index.py:130-159, 177-185, 300-308; partition.py:34). Layout (see
include/ivftq_b200.h): list l owns the slot segment [offset_l, offset_l+cap_l),
multiples of 128 slots; codes are interleaved in 32-slot blocks (word w of
slot s at codes[((s/32)*W + w)*32 + s%32]) so one warp reads a word of 32
vectors as one 128-byte transaction. Growth re-lays lists into a larger pool
(amortised: capacity grows to 1.25x the need) with one device copy kernel.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib

_SEG = 128  # slot granularity of list segments (one tensor-core M tile)


def code_layout(dim: int, bits: int, use_sign: bool) -> tuple[int, int, int]:
    """(field_bits, fields_per_word, words_per_vec) of the device code layout."""
    fb, fpw, w = C.c_int(), C.c_int(), C.c_int()
    _lib.check(_lib.load().ivftq_code_layout(dim, bits, int(use_sign), C.byref(fb),
                                             C.byref(fpw), C.byref(w)), "code_layout")
    return fb.value, fpw.value, w.value


class DeviceStore:
    def __init__(self, dim: int, bits: int, use_sign: bool, n_lists: int, device):
        self.dim, self.bits, self.use_sign, self.n_lists = dim, bits, bool(use_sign), n_lists
        self.device = device
        self.field_bits, self.fields_per_word, self.words_per_vec = code_layout(dim, bits, use_sign)
        self.sizes = np.zeros(n_lists, dtype=np.int64)
        self.caps = np.zeros(n_lists, dtype=np.int64)
        self.offsets = np.zeros(n_lists, dtype=np.int64)
        self._alloc(0)
        self._sync_meta()

    # -- buffers -------------------------------------------------------------
    def _alloc(self, capacity: int):
        W = self.words_per_vec
        self.capacity = int(capacity)
        self.codes = torch.zeros((max(capacity, 32) // 32, W, 32), dtype=torch.int32,
                                 device=self.device)
        self.norms = torch.zeros(max(capacity, 32), dtype=torch.int16, device=self.device)
        self.ids = torch.full((max(capacity, 32),), -1, dtype=torch.int32, device=self.device)

    def _sync_meta(self):
        self.offsets_d = torch.from_numpy(self.offsets.copy()).to(self.device)
        self.sizes_d = torch.from_numpy(self.sizes.astype(np.int32)).to(self.device)
        self._struct = None

    def struct(self) -> _lib.IvftqStore:
        if self._struct is None:
            s = _lib.IvftqStore()
            s.dim, s.bits, s.use_sign, s.n_lists = self.dim, self.bits, int(self.use_sign), self.n_lists
            s.field_bits, s.fields_per_word = self.field_bits, self.fields_per_word
            s.words_per_vec = self.words_per_vec
            s.max_list_size = int(self.sizes.max()) if self.n_lists else 0
            s.list_offset = self.offsets_d.data_ptr()
            s.list_size = self.sizes_d.data_ptr()
            s.codes = self.codes.data_ptr()
            s.norms = self.norms.data_ptr()
            s.ids = self.ids.data_ptr()
            s.capacity = self.capacity
            self._struct = s
        return self._struct

    # -- growth --------------------------------------------------------------
    def reserve(self, incoming: np.ndarray, slot_of: torch.Tensor):
        """Make room for `incoming[l]` more vectors in each list l."""
        need = self.sizes + incoming
        if np.all(need <= self.caps):
            return
        grow = need > self.caps
        new_caps = self.caps.copy()
        want = need + need // 4
        new_caps[grow] = ((np.maximum(want[grow], 1) + _SEG - 1) // _SEG) * _SEG
        new_off = np.concatenate(([0], np.cumsum(new_caps)[:-1])).astype(np.int64)
        old = DeviceStore.__new__(DeviceStore)
        old.__dict__.update(self.__dict__)
        old._struct = None
        self.caps = new_caps
        self.offsets = new_off
        self._alloc(int(new_caps.sum()))
        self._sync_meta()
        if old.sizes.sum() > 0:
            lib = _lib.lib()
            _lib.check(lib.ivftq_relayout(C.byref(old.struct()), C.byref(self.struct()),
                                          slot_of.data_ptr(), _lib.stream_ptr()), "relayout")

    def set_sizes(self, sizes: np.ndarray):
        self.sizes = sizes.astype(np.int64)
        self.sizes_d.copy_(torch.from_numpy(self.sizes.astype(np.int32)))
        self._struct = None

    def reset(self):
        self.sizes[:] = 0
        self.caps[:] = 0
        self.offsets[:] = 0
        self._alloc(0)
        self._sync_meta()

    def nbytes(self) -> int:
        return (self.codes.numel() * 4 + self.norms.numel() * 2 + self.ids.numel() * 4)
