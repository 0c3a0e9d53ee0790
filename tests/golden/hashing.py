"""Per-row 64-bit polynomial hash used to pin large code matrices compactly."""

import numpy as np

HASH_P = np.uint64(0x9E3779B97F4A7C15)


def row_hash(packed: np.ndarray) -> np.ndarray:
    """Hash of each row of a (n, B) uint8 matrix (arithmetic wraps mod 2^64)."""
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    n, b = packed.shape
    h = np.zeros(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for j in range(b):
            h = h * HASH_P + packed[:, j].astype(np.uint64) + np.uint64(1)
    return h
