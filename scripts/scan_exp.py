"""Scan-kernel timing on a C3-shaped index with the library named by IVFTQ_LIB
(used with the experiment builds of `make exp`, whose results are invalid:
they compile one role's work out to show which role bounds the tile period).

  IVFTQ_LIB=paper_2605_17415_b200/lib/libivftq_b200_exp_noepi.so python scripts/scan_exp.py [n] [n_p] [d] [L]
"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2605_17415_b200 import CoarsePartition, _lib, design_quantizer, generate_rotation  # noqa: E402
from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex  # noqa: E402
from paper_2605_17415_b200.workloads import mixture  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
n_p = int(sys.argv[2]) if len(sys.argv) > 2 else 32
d = int(sys.argv[3]) if len(sys.argv) > 3 else 96
L = int(sys.argv[4]) if len(sys.argv) > 4 else 4096
nq = 10_000
x, means = mixture(n, d, L, 0.3, 1)
q, _ = mixture(nq, d, L, 0.3, 2, means=means)
rng = np.random.default_rng(0)
cent = x[rng.choice(n, L, replace=False)].astype(np.float64)
cent = (cent / np.linalg.norm(cent, axis=1)[:, None]).astype(np.float32)
idx = IvfTqIndex(IndexConfig(dim=d, bits=4, n_lists=L), design_quantizer(4, d),
                 generate_rotation(d, 42), CoarsePartition(L, d, cent))
for s in range(0, n, 1_000_000):
    idx.add_batch(x[s:s + 1_000_000])
qd = torch.from_numpy(q).cuda()
lib = _lib.lib()
lib.ivftq_set_kernel_timing(1)
ts = []
for r in range(6):
    idx.search_batch(qd, 10, n_p, return_device=True)
    torch.cuda.synchronize()
    ts.append(lib.ivftq_last_scan_kernel_ms())
print(f"{os.path.basename(os.environ.get('IVFTQ_LIB', 'default'))} n={n} n_p={n_p} d={d} L={L} "
      f"scan_ms median={np.median(ts[1:]):.4f} all={[round(t, 4) for t in ts]}", flush=True)
