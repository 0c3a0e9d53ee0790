"""Standalone ivftq_select_topn timing on C2-like coarse score rows (10k x 1024, n=64)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_17415_b200 import _lib
L = _lib.lib()
rows, cols = 10000, 1024
rng = np.random.default_rng(0)
c = rng.standard_normal((cols, 128)); c /= np.linalg.norm(c, axis=1)[:, None]
q = c[rng.integers(0, cols, rows)] + 0.3 * rng.standard_normal((rows, 128))
q /= np.linalg.norm(q, axis=1)[:, None]
S = torch.from_numpy(q @ c.T).cuda()
for n in (1, 16, 64):
    idx = torch.empty((rows, n), dtype=torch.int32, device="cuda")
    val = torch.empty((rows, n), dtype=torch.float64, device="cuda")
    run = lambda: _lib.check(L.ivftq_select_topn(S.data_ptr(), rows, cols, n, idx.data_ptr(), val.data_ptr(), None))
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record(); torch.cuda.synchronize()
    want = np.argsort(-S.cpu().numpy(), axis=1, kind="stable")[:, :n]
    ok = np.array_equal(idx.cpu().numpy(), want)
    print(f"n={n}: {e0.elapsed_time(e1)/10*1000:.1f} us per call, exact={ok}")
