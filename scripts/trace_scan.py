"""Run one C2-like batched search with the scan_tc timeline trace enabled."""
import os, sys, time
os.environ["IVFTQ_NO_GRAPH"] = "1"  # a graph replay would skip the host-side trace dump
from pathlib import Path
# the timeline instrumentation only exists in the trace build (make -C paper_2605_17415_b200/csrc trace)
os.environ.setdefault("IVFTQ_LIB", str(Path(__file__).resolve().parents[1] / "paper_2605_17415_b200" / "lib" / "libivftq_b200_trace.so"))
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_17415_b200 import CoarsePartition, design_quantizer, generate_rotation
from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex
from paper_2605_17415_b200.workloads import mixture
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
n_p = int(sys.argv[2]) if len(sys.argv) > 2 else 64
d = int(sys.argv[3]) if len(sys.argv) > 3 else 128
L = int(sys.argv[4]) if len(sys.argv) > 4 else 1024
nq = 10_000
x, means = mixture(n, d, L, 0.3, 1)
q, _ = mixture(nq, d, L, 0.3, 2, means=means)
rng = np.random.default_rng(0)
cent = x[rng.choice(n, L, replace=False)].astype(np.float64)
cent = (cent / np.linalg.norm(cent, axis=1)[:, None]).astype(np.float32)
idx = IvfTqIndex(IndexConfig(dim=d, bits=4, n_lists=L), design_quantizer(4, d),
                 generate_rotation(d, 42), CoarsePartition(L, d, cent))
idx.add_batch(x)
qd = torch.from_numpy(q).cuda()
idx.search_batch(qd, 10, n_p, return_device=True)
torch.cuda.synchronize()
os.environ["IVFTQ_TRACE"] = "gpurun_out/trace.txt"
idx.search_batch(qd, 10, n_p, return_device=True)
torch.cuda.synchronize()
print("sizes", idx._store.sizes.min(), idx._store.sizes.mean(), idx._store.sizes.max())
