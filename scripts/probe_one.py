"""One shape of ivftq_probe in a chosen coarse mode (for ncu captures):
python scripts/probe_one.py NQ L D NP MODE [REPS]"""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_17415_b200 import _lib

nq, L, d, n_p, mode = (int(a) for a in sys.argv[1:6])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
lib = _lib.lib()
rng = np.random.default_rng(0)
means = rng.standard_normal((L, d))
c = means + 0.3 * rng.standard_normal((L, d))
c = (c / np.linalg.norm(c, axis=1)[:, None]).astype(np.float32)
q = means[rng.integers(0, L, nq)] + 0.3 * rng.standard_normal((nq, d))
q /= np.linalg.norm(q, axis=1)[:, None]
qd, cd = torch.from_numpy(q).cuda(), torch.from_numpy(c).cuda()
sb = lib.ivftq_probe_scratch_bytes(nq, L, d)
scr = torch.empty(sb, dtype=torch.uint8, device="cuda")
pr = torch.empty((nq, n_p), dtype=torch.int32, device="cuda")
co = torch.empty((nq, n_p), dtype=torch.float64, device="cuda")
lib.ivftq_set_coarse_mode(mode)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(reps):
    e0.record()
    _lib.check(lib.ivftq_probe(qd.data_ptr(), cd.data_ptr(), nq, L, d, n_p, pr.data_ptr(),
                               co.data_ptr(), scr.data_ptr(), sb, _lib.stream_ptr()))
    e1.record()
    torch.cuda.synchronize()
    print(f"rep {i}: {e0.elapsed_time(e1) * 1000:.1f} us", flush=True)
