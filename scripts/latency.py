"""Single-query and small-batch search latency through the public API (C2 scale)."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_17415_b200 import CoarsePartition, design_quantizer, generate_rotation
from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex
from paper_2605_17415_b200.workloads import mixture
n, d, L = 1_000_000, 128, 1024
x, means = mixture(n, d, 1000, 0.3, 1)
q, _ = mixture(1000, d, 1000, 0.3, 2, means=means)
rng = np.random.default_rng(0)
cent = x[rng.choice(n, L, replace=False)].astype(np.float64)
cent = (cent / np.linalg.norm(cent, axis=1)[:, None]).astype(np.float32)
idx = IvfTqIndex(IndexConfig(dim=d, bits=4, n_lists=L), design_quantizer(4, d),
                 generate_rotation(d, 42), CoarsePartition(L, d, cent))
idx.add_batch(torch.from_numpy(x).pin_memory())
q = np.concatenate([q, q])  # fixed-size windows at any offset
for graphs in (True, False):
    idx.use_graphs = graphs
    for bs in (1, 8, 64, 256):
        for n_p in (16, 64):
            idx.search_batch(q[:bs], 10, n_p)
            idx.search_batch(q[bs:2 * bs], 10, n_p)
            t0 = time.perf_counter()
            reps = 50
            for r in range(reps):
                o = (r * bs) % 1000
                idx.search_batch(q[o:o + bs], 10, n_p)
            dt = (time.perf_counter() - t0) / reps
            print(f"graphs {int(graphs)} batch {bs:4d} n_p {n_p:3d}: {dt*1e3:.3f} ms per call, "
                  f"{bs/dt:,.0f} queries/s", flush=True)
