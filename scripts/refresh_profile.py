"""Host-side profile of one refresh() on a C5-sized index (cProfile, cumulative)."""
import cProfile, pstats, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2605_17415_b200 import CoarsePartition, design_quantizer, generate_rotation
from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex
from paper_2605_17415_b200.refresh import RefreshPolicy, refresh
from paper_2605_17415_b200.workloads import mixture
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
d, L = 96, 4096
x, means = mixture(n, d, L, 0.3, 1)
rng = np.random.default_rng(0)
cent = x[rng.choice(n, L, replace=False)].astype(np.float64)
cent = (cent / np.linalg.norm(cent, axis=1)[:, None]).astype(np.float32)
idx = IvfTqIndex(IndexConfig(dim=d, bits=4, n_lists=L), design_quantizer(4, d), generate_rotation(d, 42), CoarsePartition(L, d, cent))
for s in range(0, n, 1_000_000):
    idx.add_batch(x[s:s + 1_000_000])
torch.cuda.synchronize()
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
rep = refresh(idx, RefreshPolicy(seed=0))
torch.cuda.synchronize()
pr.disable()
print("refresh", time.perf_counter() - t, "s", rep.sample_size)
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
