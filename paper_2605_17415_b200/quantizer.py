"""Lloyd-Max scalar quantizer for N(0, 1/d) with half-bin means (host side).

The codebook is a fixed input of the hot path: it is
designed once on the CPU from the published Lloyd-Max fixed point and shipped
to the device as f64 tables. This module restates lloydmax.py:159-235 so that
`IvfTqIndex.build` needs no reference import; tests/test_host.py checks its
tables bit-for-bit against the reference's (tests/golden/tables.npz).

Design (standard normal, then scaled by 1/sqrt(d)):
  c_i <- E[Z | t_i <= Z <= t_{i+1}] with t the midpoints of neighbouring
  c's, E[Z | a<=Z<=b] = (phi(a) - phi(b)) / (Phi(b) - Phi(a)); start at the
  Gaussian quantiles (i+1/2)/2^b; re-symmetrise c <- (c - reverse(c))/2 each
  step; stop when max |c_new - c| < tol.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.special import ndtr, ndtri

__all__ = ["ScalarQuantizer", "QuantizerConvergenceError", "design_quantizer"]


class QuantizerConvergenceError(RuntimeError):
    """Lloyd iteration did not converge (lloydmax.py:34-44)."""

    def __init__(self, bits: int, last_delta: float, max_iters: int):
        self.bits, self.last_delta, self.max_iters = bits, last_delta, max_iters
        super().__init__(
            f"Lloyd iteration for bits={bits} did not converge after "
            f"{max_iters} iterations (last centroid movement {last_delta:.3e})")


def _pdf(z: np.ndarray) -> np.ndarray:
    out = np.zeros_like(z, dtype=np.float64)
    ok = np.isfinite(z)
    out[ok] = np.exp(-0.5 * z[ok] ** 2) / np.sqrt(2.0 * np.pi)
    return out


def _moments(a: np.ndarray, b: np.ndarray):
    """(P, M1, M2) of N(0,1) on [a, b]; infinite ends handled exactly."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    fa, fb = _pdf(a), _pdf(b)
    p = ndtr(b) - ndtr(a)
    m1 = fa - fb
    za = np.zeros_like(fa)
    za[np.isfinite(a)] = a[np.isfinite(a)] * fa[np.isfinite(a)]
    zb = np.zeros_like(fb)
    zb[np.isfinite(b)] = b[np.isfinite(b)] * fb[np.isfinite(b)]
    return p, m1, p + za - zb


def _cond_mean(a, b):
    p, m1, _ = _moments(a, b)
    return m1 / p


def _mse(a, b, rep) -> float:
    p, m1, m2 = _moments(a, b)
    return float(np.sum(m2 - 2.0 * rep * m1 + rep * rep * p))


@dataclass(frozen=True)
class ScalarQuantizer:
    """Converged codebook for N(0, 1/dim) (lloydmax.py:89-156)."""

    bits: int
    dim: int
    boundaries: np.ndarray  # (2^b + 1,), -inf .. +inf
    centroids: np.ndarray  # (2^b,)
    half_bin_means: np.ndarray  # (2^b, 2)
    distortion: float
    distortion_sign: float

    def __post_init__(self):
        for name in ("boundaries", "centroids", "half_bin_means"):
            getattr(self, name).setflags(write=False)

    @property
    def n_levels(self) -> int:
        return 1 << self.bits

    @property
    def per_coord_distortion(self) -> float:
        return self.distortion / self.dim

    @property
    def per_coord_distortion_sign(self) -> float:
        return self.distortion_sign / self.dim

    def reconstruction_table(self, use_sign: bool) -> np.ndarray:
        """(2^b, 2) half-bin means, or (2^b,) centroids (lloydmax.py:146-150)."""
        return self.half_bin_means if use_sign else self.centroids

    def levels(self, use_sign: bool) -> np.ndarray:
        """Flattened f64 table indexed by the device field value bin*2+sign.

        Without the sign bit both halves of a bin map to its centroid, which is
        `reconstruction_table(False)[bin]` (lloydmax.py:146-150).
        """
        if use_sign:
            return np.ascontiguousarray(self.half_bin_means, dtype=np.float64).ravel()
        return np.repeat(np.asarray(self.centroids, dtype=np.float64), 2)


def design_quantizer(bits: int, dim: int, tol: float = 1e-10,
                     max_iters: int = 1_000_000) -> ScalarQuantizer:
    if not 1 <= bits <= 8:
        raise ValueError(f"bits must be in [1, 8], got {bits}")
    if dim < 1:
        raise ValueError(f"dim must be >= 1, got {dim}")
    if tol <= 0:
        raise ValueError(f"tol must be positive, got {tol}")
    k = 1 << bits
    c = ndtri((np.arange(k) + 0.5) / k)
    c = 0.5 * (c - c[::-1])
    delta = np.inf
    converged = False
    for _ in range(max_iters):
        mid = 0.5 * (c[:-1] + c[1:])
        lo = np.concatenate(([-np.inf], mid))
        hi = np.concatenate((mid, [np.inf]))
        nxt = _cond_mean(lo, hi)
        nxt = 0.5 * (nxt - nxt[::-1])
        delta = float(np.max(np.abs(nxt - c)))
        c = nxt
        if delta < tol:
            converged = True
            break
    if not converged:
        raise QuantizerConvergenceError(bits, delta, max_iters)
    mid = 0.5 * (c[:-1] + c[1:])
    lo = np.concatenate(([-np.inf], mid))
    hi = np.concatenate((mid, [np.inf]))
    h_lo = _cond_mean(lo, c)
    h_hi = _cond_mean(c, hi)
    half = np.stack([h_lo, h_hi], axis=1)
    dist = _mse(lo, hi, c)
    dist_s = _mse(lo, c, h_lo) + _mse(c, hi, h_hi)
    s = 1.0 / np.sqrt(float(dim))
    return ScalarQuantizer(bits=bits, dim=dim,
                           boundaries=np.concatenate(([-np.inf], mid * s, [np.inf])),
                           centroids=c * s, half_bin_means=half * s,
                           distortion=dist, distortion_sign=dist_s)
