"""Run-to-run spread of one 1M-row add_batch into a fresh index (C2 shape),
host and device clocks, with and without the caching allocator warm."""
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
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
keep = []
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    idx = IvfTqIndex(IndexConfig(dim=d, bits=4, n_lists=L), design_quantizer(4, d),
                     generate_rotation(d, 42), CoarsePartition(L, d, cent))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    idx.add_batch(pinned)
    e1.record()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"rep {rep}: host {dt*1e3:.1f} ms  event {e0.elapsed_time(e1):.1f} ms  "
          f"reserved {torch.cuda.memory_reserved()/1e9:.2f} GB", flush=True)
    if rep % 2:
        keep.append(idx)  # alternate: some indexes stay alive
