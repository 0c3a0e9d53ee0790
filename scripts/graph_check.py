import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
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
Qd = torch.from_numpy(q).cuda()
for n_p in (8, 64):
    for graphs in (True, False):
        idx.use_graphs = graphs
        for r in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); t = time.perf_counter()
            e0.record(); idx.search_batch(Qd, 10, n_p, return_device=True); e1.record(); torch.cuda.synchronize()
            print(n_p, graphs, r, round(e0.elapsed_time(e1), 3), "ms gpu", round((time.perf_counter()-t)*1e3, 3), "ms host", len(getattr(idx._thread_state(), 'graphs', {}) or {}), flush=True)
