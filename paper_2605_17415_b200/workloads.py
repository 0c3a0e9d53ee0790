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

The 10M-row configs (`threads > 1`) draw each 1M-row chunk from its own child
stream (`SeedSequence(seed).spawn`), so the chunks fill in parallel threads
(numpy releases the GIL while a Generator fills an array); the rows depend only
on the seed, never on the thread count.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
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
    threads: int = 1,
) -> tuple[np.ndarray, np.ndarray]:
    """Gaussian-mixture rows (float32) and the component means used.

    Args:
        means: Reuse these component means (queries share the base means).
        mean_seed: Seed for drawing means when `means` is None (defaults to seed).
        norm_sigma: If > 0, scale each row by a log-normal(0, norm_sigma) norm
            (config C4; the reference normalises rows, so this changes nothing
            the index sees).
        threads: > 1 selects the chunk-parallel stream (see module docstring).
    """
    if threads > 1:
        return _mixture_parallel(n, d, k, sigma, seed, means, mean_seed, norm_sigma, threads)
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


def _mixture_parallel(n, d, k, sigma, seed, means, mean_seed, norm_sigma, threads):
    if means is None:
        mrng = np.random.default_rng(seed if mean_seed is None else mean_seed)
        means = mrng.standard_normal((k, d))
    out = np.empty((n, d), dtype=np.float32)
    starts = list(range(0, n, _CHUNK))
    kids = np.random.SeedSequence([seed, 7919]).spawn(len(starts))

    def fill(i):
        s = starts[i]
        e = min(n, s + _CHUNK)
        rng = np.random.default_rng(kids[i])
        labels = rng.integers(0, len(means), e - s)
        noise = rng.standard_normal((e - s, d), dtype=np.float32)
        out[s:e] = (means[labels] + sigma * noise).astype(np.float32)
        if norm_sigma > 0:
            rn = np.linalg.norm(out[s:e].astype(np.float64), axis=1)
            scale = np.exp(norm_sigma * rng.standard_normal(e - s)) / rn
            out[s:e] = (out[s:e] * scale[:, None]).astype(np.float32)

    with ThreadPoolExecutor(max(1, min(threads, len(starts)))) as ex:
        list(ex.map(fill, range(len(starts))))
    return out, means


def gen_threads() -> int:
    return max(1, min(16, os.cpu_count() or 1))


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
    parallel: bool = False  # chunk-parallel generation (10M-row configs)
    extra: dict = field(default_factory=dict)

    def base(self, n: int | None = None) -> np.ndarray:
        x, _ = mixture(n or self.n, self.d, self.components, self.sigma,
                       self.base_seed, norm_sigma=self.norm_sigma,
                       threads=gen_threads() if self.parallel else 1)
        return x

    def queries(self, nq: int | None = None) -> np.ndarray:
        mrng = np.random.default_rng(self.base_seed)
        means = mrng.standard_normal((self.components, self.d))
        if self.query_shift > 0:
            srng = np.random.default_rng(self.query_seed + 1)
            means = means + self.query_shift * srng.standard_normal(means.shape)
        q, _ = mixture(nq or self.n_queries, self.d, self.components, self.sigma,
                       self.query_seed, means=means,
                       threads=gen_threads() if self.parallel else 1)
        return q


WORKLOADS = {
    "pr1": Workload("pr1", 100_000, 128, 256, 0.3, 256, 4, 1_000, 10, (16,),
                    notes="configs[0]: PR1 oracle scale"),
    "c2": Workload("c2", 1_000_000, 128, 1000, 0.3, 1024, 4, 10_000, 10,
                   (1, 4, 16, 64), kmeans_sample=100_000,
                   notes="configs[1]: k-means on a seeded 100k subsample"),
    # C3: the north_star target. k-means (reference algorithm, host f64) runs on
    # a seeded 32,768-row subsample (8 rows per list) so the bench's two arms
    # train the identical centroids on the host in ~half a minute.
    "c3": Workload("c3", 10_000_000, 96, 4096, 0.3, 4096, 4, 10_000, 10,
                   (16, 32, 64, 128), kmeans_sample=32_768, parallel=True,
                   notes="configs[2]: sigma unspecified, 0.3 recorded"),
    # C3 with overlapping clusters: 1024 mixture components spread over 4096
    # lists and sigma 0.6, so true neighbours straddle lists and recall rises
    # with n_p (the C3 mixture puts every neighbour in the nearest list).
    "c3_hard": Workload("c3_hard", 10_000_000, 96, 1024, 1.0, 4096, 4, 10_000, 10,
                        (1, 4, 16, 32, 64, 128), kmeans_sample=32_768, parallel=True,
                        notes="harder C3 variant: K=1024 components, sigma 1.0, sweep from n_p=1"),
    "c4": Workload("c4", 10_000_000, 200, 4096, 0.3, 4096, 4, 10_000, 10, (64,),
                   kmeans_sample=32_768, query_shift=0.5, norm_sigma=0.25, parallel=True,
                   notes="configs[3]: queries from means + 0.5*N(0,1) offsets"),
    "c5": Workload("c5", 10_000_000, 96, 4096, 0.3, 4096, 4, 10_000, 10, (32,),
                   kmeans_sample=1_000_000, parallel=True,
                   notes="configs[4]: stream of 1M batches, L=4096 recorded"),
}


def make_workload(name: str, **overrides) -> Workload:
    """A named workload, optionally with fields overridden (scaled-down tests)."""
    import dataclasses

    return dataclasses.replace(WORKLOADS[name], **overrides)
