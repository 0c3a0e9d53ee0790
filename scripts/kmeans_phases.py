"""Device k-means phases at the C5 refresh shape: seeding, one Lloyd assignment, one Lloyd update."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2605_17415_b200 import _lib
L = _lib.lib()
n, d, k = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (411644, 96, 4096)))
rng = np.random.default_rng(0)
x = rng.standard_normal((n, d)); x /= np.linalg.norm(x, axis=1)[:, None]
X = torch.from_numpy(x).cuda()
nc = int(L.ivftq_kmeanspp_candidates(k))
u = np.ascontiguousarray(rng.random((k - 1, nc)))
chosen = torch.empty(k, dtype=torch.int64, device="cuda")
tots = torch.empty(k, dtype=torch.float64, device="cuda")
nb = int(L.ivftq_kmeanspp_scratch_bytes(n, d, k))
scratch = torch.empty(nb, dtype=torch.uint8, device="cuda")
def timed(fn, reps=2):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best
ts = timed(lambda: _lib.check(L.ivftq_kmeanspp_seed(X.data_ptr(), n, d, k, 5, u.ctypes.data, chosen.data_ptr(), tots.data_ptr(), scratch.data_ptr(), nb, _lib.stream_ptr())))
cent = X[chosen].clone()
ab = max(int(L.ivftq_assign_tc_scratch_bytes(n, k, d)), int(L.ivftq_kmeans_sums_scratch_bytes(n, k)))
sc2 = torch.empty(ab, dtype=torch.uint8, device="cuda")
a = torch.empty(n, dtype=torch.int32, device="cuda")
ta = timed(lambda: _lib.check(L.ivftq_assign_tc64(X.data_ptr(), cent.data_ptr(), n, k, d, a.data_ptr(), sc2.data_ptr(), ab, _lib.stream_ptr())))
sums = torch.empty((k, d), dtype=torch.float64, device="cuda"); cnt = torch.empty(k, dtype=torch.int32, device="cuda")
tu = timed(lambda: _lib.check(L.ivftq_kmeans_sums(X.data_ptr(), a.data_ptr(), n, d, k, sums.data_ptr(), cnt.data_ptr(), sc2.data_ptr(), ab, _lib.stream_ptr())))
print(f"n={n} d={d} k={k}: seeding {ts*1e3:.1f} ms ({ts/(k-1)*1e6:.1f} us/step), assign {ta*1e3:.2f} ms, sums {tu*1e3:.2f} ms")
