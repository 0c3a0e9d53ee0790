"""Host-clock phases of one 1M-row pinned add_batch at C2 (encode pipeline vs append)."""
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
for rep in range(3):
    idx = IvfTqIndex(IndexConfig(dim=d, bits=4, n_lists=L), design_quantizer(4, d),
                     generate_rotation(d, 42), CoarsePartition(L, d, cent))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    words, lids, nrm, xn = idx._encode_host_pipelined(pinned)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    idx._append_encoded(words, lids, nrm, xn)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"encode issue {1e3*(t1-t0):.1f} ms (incl. final flag sync), drain {1e3*(t2-t1):.1f}, append {1e3*(t3-t2):.1f}, total {1e3*(t3-t0):.1f}")
