"""Host-side cost of one end-to-end search_batch call (pinned host queries ->
numpy results) at C2, phase by phase, against the device time of the replay."""
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
q, _ = mixture(10000, d, 1000, 0.3, 2, means=means)
rng = np.random.default_rng(0)
cent = x[rng.choice(n, L, replace=False)].astype(np.float64)
cent = (cent / np.linalg.norm(cent, axis=1)[:, None]).astype(np.float32)
idx = IvfTqIndex(IndexConfig(dim=d, bits=4, n_lists=L), design_quantizer(4, d), generate_rotation(d, 42), CoarsePartition(L, d, cent))
idx.add_batch(torch.from_numpy(x).pin_memory())
qpin = torch.from_numpy(q).pin_memory()
for _ in range(3):
    idx.search_batch(qpin, 10, 64)
import cProfile, pstats
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20):
    idx.search_batch(qpin, 10, 64)
print("per call wall", (time.perf_counter() - t) / 20 * 1e3, "ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    idx.search_batch(qpin, 10, 64)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
