"""Time ivftq_probe (f64 GEMM + select vs tensor-core + exact band) on random
unit queries/centroids of a given shape; both paths must return identical probes (coarse values to a few ulps)."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_17415_b200 import _lib

L_ = _lib.lib()
for (nq, L, d, n_p) in [(10000, 1024, 128, 64), (10000, 4096, 96, 32), (10000, 4096, 96, 128),
                        (10000, 4096, 200, 64)]:
    rng = np.random.default_rng(0)
    means = rng.standard_normal((L, d))
    c = means + 0.3 * rng.standard_normal((L, d))
    c = (c / np.linalg.norm(c, axis=1)[:, None]).astype(np.float32)
    q = means[rng.integers(0, L, nq)] + 0.3 * rng.standard_normal((nq, d))
    q /= np.linalg.norm(q, axis=1)[:, None]
    qd, cd = torch.from_numpy(q).cuda(), torch.from_numpy(c).cuda()
    sb = L_.ivftq_probe_scratch_bytes(nq, L, d)
    scr = torch.empty(sb, dtype=torch.uint8, device="cuda")
    res = {}
    for mode in (1, 2):
        L_.ivftq_set_coarse_mode(mode)
        pr = torch.empty((nq, n_p), dtype=torch.int32, device="cuda")
        co = torch.empty((nq, n_p), dtype=torch.float64, device="cuda")
        run = lambda: _lib.check(L_.ivftq_probe(qd.data_ptr(), cd.data_ptr(), nq, L, d, n_p, pr.data_ptr(),
                                                co.data_ptr(), scr.data_ptr(), sb, _lib.stream_ptr()))
        run(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record(); torch.cuda.synchronize()
        res[mode] = (e0.elapsed_time(e1) / 5, pr.cpu().numpy(), co.cpu().numpy())
    L_.ivftq_set_coarse_mode(0)
    same = np.array_equal(res[1][1], res[2][1]) and np.allclose(res[1][2], res[2][2], rtol=0, atol=1e-14)
    print(f"nq={nq} L={L} d={d} n_p={n_p}: f64 {res[1][0]:.3f} ms, tc {res[2][0]:.3f} ms, identical={same}")
