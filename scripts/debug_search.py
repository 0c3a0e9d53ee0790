"""Stage-by-stage search debug on a synthetic index (run with CUDA_LAUNCH_BLOCKING=1)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17415_b200 import CoarsePartition, design_quantizer, generate_rotation  # noqa
from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex  # noqa
from paper_2605_17415_b200.workloads import mixture  # noqa

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000
d, L = 128, 1024
x, means = mixture(n, d, 1000, 0.3, 1)
q, _ = mixture(nq, d, 1000, 0.3, 2, means=means)
rng = np.random.default_rng(0)
cent = x[rng.choice(n, L, replace=False)].astype(np.float64)
cent = (cent / np.linalg.norm(cent, axis=1)[:, None]).astype(np.float32)
idx = IvfTqIndex(IndexConfig(dim=d, bits=4, n_lists=L), design_quantizer(4, d),
                 generate_rotation(d, 42), CoarsePartition(L, d, cent))
t0 = time.time()
idx.add_batch(x)
torch.cuda.synchronize()
print("added", n, time.time() - t0, "max list", idx._store.sizes.max(), flush=True)
for n_p in (1, 4, 16, 64):
    for nqq in (100, nq):
        try:
            ids, sc = idx.search_batch(q[:nqq], 10, n_p)
            torch.cuda.synchronize()
            print("ok n_p", n_p, "nq", nqq, ids[0, :3], flush=True)
        except Exception as e:  # noqa
            print("FAIL n_p", n_p, "nq", nqq, repr(e)[:300], flush=True)
            raise
