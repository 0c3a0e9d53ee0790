"""End-to-end add_batch rate from pinned host rows vs the host->device copy rate,
for several pipeline sub-chunk sizes (C2 shape)."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_17415_b200 import CoarsePartition, design_quantizer, generate_rotation
from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex
from paper_2605_17415_b200.workloads import mixture
n, d, L = 1_000_000, 128, 1024
x, _ = mixture(n, d, 1000, 0.3, 1)
rng = np.random.default_rng(0)
cent = x[rng.choice(n, L, replace=False)].astype(np.float64)
cent = (cent / np.linalg.norm(cent, axis=1)[:, None]).astype(np.float32)
pinned = torch.from_numpy(x).pin_memory()
dev = torch.device("cuda")
buf = torch.empty_like(pinned, device=dev)
torch.cuda.synchronize()
t0 = time.perf_counter(); buf.copy_(pinned, non_blocking=True); torch.cuda.synchronize()
print(f"H2D {pinned.numel()*4/1e9:.2f} GB in {(time.perf_counter()-t0)*1e3:.1f} ms")
for sub in (1 << 16, 1 << 17, 1 << 18):
    for rep in range(2):
        idx = IvfTqIndex(IndexConfig(dim=d, bits=4, n_lists=L), design_quantizer(4, d),
                         generate_rotation(d, 42), CoarsePartition(L, d, cent))
        idx._PIPE_ROWS = sub
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        idx.add_batch(pinned)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"sub-chunk {sub}: {dt*1e3:.1f} ms, {n/dt/1e6:.1f} M adds/s")
