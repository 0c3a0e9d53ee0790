"""Seeded synthetic workloads for the BASELINE.json configs.

No public dataset is used: the reference's own generators
(`ivftq.data_io.make_sift_like` / `make_synthetic_clusters`, data_io.py:111-173)
produce different distributions, so these mixtures are this repo's own, with the
shapes, sizes and value distributions BASELINE.json names:

    Mixture(N, d, K, sigma): means ~ N(0, I_d) (K of them), labels ~ U{0..K-1},
    x = means[label] + sigma * N(0, I_d), float32.

Queries use the same means with a separate RNG stream. Noise is drawn in
float32 row chunks so 10M-row configs never hold a float64 copy; the chunked
stream equals a single draw (numpy Generator fills sequentially).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["Workload", "WORKLOADS", "mixture", "make_workload"]

_CHUNK = 1 << 20


def mixture(
    n: int,
    d: int,
    k: int,
    sigma: float,
    seed: int,
    means: np.ndarray | None = None,
    mean_seed: int | None = None,
    norm_sigma: float = 0.0,
) -> tuple[np.ndarray, np.ndarray]:
    """Gaussian-mixture rows (float32) and the component means used.

    Args:
        means: Reuse these component means (queries share the base means).
        mean_seed: Seed for drawing means when `means` is None (defaults to seed).
        norm_sigma: If > 0, scale each row by a log-normal(0, norm_sigma) norm
            (config C4; the reference normalises rows, so this changes nothing
            the index sees).
    """
    if means is None:
        mrng = np.random.default_rng(seed if mean_seed is None else mean_seed)
        means = mrng.standard_normal((k, d))
    rng = np.random.default_rng(seed + 7919)
    labels = rng.integers(0, len(means), n)
    out = np.empty((n, d), dtype=np.float32)
    for s in range(0, n, _CHUNK):
        e = min(n, s + _CHUNK)
        noise = rng.standard_normal((e - s, d), dtype=np.float32)
        out[s:e] = (means[labels[s:e]] + sigma * noise).astype(np.float32)
    if norm_sigma > 0:
        nrng = np.random.default_rng(seed + 104729)
        for s in range(0, n, _CHUNK):
            e = min(n, s + _CHUNK)
            rn = np.linalg.norm(out[s:e].astype(np.float64), axis=1)
            scale = np.exp(norm_sigma * nrng.standard_normal(e - s)) / rn
            out[s:e] = (out[s:e] * scale[:, None]).astype(np.float32)
    return out, means


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config with its recorded seeds."""

    name: str
    n: int
    d: int
    components: int
    sigma: float
    n_lists: int
    bits: int
    n_queries: int
    k: int
    nprobe: tuple[int, ...]
    kmeans_iters: int = 10
    kmeans_sample: int | None = None  # train on a seeded subsample of this size
    base_seed: int = 1234
    query_seed: int = 4321
    query_shift: float = 0.0  # C4: per-component query mean offset scale
    norm_sigma: float = 0.0  # C4: log-normal base norms
    notes: str = ""
    extra: dict = field(default_factory=dict)

    def base(self, n: int | None = None) -> np.ndarray:
        x, _ = mixture(n or self.n, self.d, self.components, self.sigma,
                       self.base_seed, norm_sigma=self.norm_sigma)
        return x

    def queries(self, nq: int | None = None) -> np.ndarray:
        mrng = np.random.default_rng(self.base_seed)
        means = mrng.standard_normal((self.components, self.d))
        if self.query_shift > 0:
            srng = np.random.default_rng(self.query_seed + 1)
            means = means + self.query_shift * srng.standard_normal(means.shape)
        q, _ = mixture(nq or self.n_queries, self.d, self.components, self.sigma,
                       self.query_seed, means=means)
        return q


WORKLOADS = {
    "pr1": Workload("pr1", 100_000, 128, 256, 0.3, 256, 4, 1_000, 10, (16,),
                    notes="configs[0]: PR1 oracle scale"),
    "c2": Workload("c2", 1_000_000, 128, 1000, 0.3, 1024, 4, 10_000, 10,
                   (1, 4, 16, 64), kmeans_sample=100_000,
                   notes="configs[1]: k-means on a seeded 100k subsample"),
    "c3": Workload("c3", 10_000_000, 96, 4096, 0.3, 4096, 4, 10_000, 10,
                   (16, 32, 64, 128), kmeans_sample=1_000_000,
                   notes="configs[2]: sigma unspecified, 0.3 recorded"),
    "c4": Workload("c4", 10_000_000, 200, 4096, 0.3, 4096, 4, 10_000, 10, (64,),
                   kmeans_sample=1_000_000, query_shift=0.5, norm_sigma=0.25,
                   notes="configs[3]: queries from means + 0.5*N(0,1) offsets"),
    "c5": Workload("c5", 10_000_000, 96, 4096, 0.3, 4096, 4, 10_000, 10, (32,),
                   kmeans_sample=1_000_000,
                   notes="configs[4]: stream of 1M batches, L=4096 recorded"),
}


def make_workload(name: str, **overrides) -> Workload:
    """A named workload, optionally with fields overridden (scaled-down tests)."""
    import dataclasses

    return dataclasses.replace(WORKLOADS[name], **overrides)
