"""CUDA-event timeline of one C2 search step (10k queries, n_p=64), phase by
phase, replaying IvfTqIndex.search_batch's device sequence on the current
stream: normalize | probe | rotate | scan (regroup + seed + scan + merge)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_17415_b200 import CoarsePartition, design_quantizer, generate_rotation, _lib
from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex
from paper_2605_17415_b200.workloads import mixture

n, d, L, n_p, nq = 1_000_000, 128, 1024, 64, 10_000
x, means = mixture(n, d, 1000, 0.3, 1)
q, _ = mixture(nq, d, 1000, 0.3, 2, means=means)
rng = np.random.default_rng(0)
cent = x[rng.choice(n, L, replace=False)].astype(np.float64)
cent = (cent / np.linalg.norm(cent, axis=1)[:, None]).astype(np.float32)
idx = IvfTqIndex(IndexConfig(dim=d, bits=4, n_lists=L), design_quantizer(4, d),
                 generate_rotation(d, 42), CoarsePartition(L, d, cent))
idx.add_batch(x)
qd = torch.from_numpy(q).cuda()
lib = _lib.lib()
for rep in range(4):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    qn, bad, _ = idx._normalize_queries_device(qd)
    ev[1].record()
    probe = torch.empty((nq, n_p), dtype=torch.int32, device="cuda")
    coarse = torch.empty((nq, n_p), dtype=torch.float64, device="cuda")
    pb = lib.ivftq_probe_scratch_bytes(nq, L, d)
    pscr = torch.empty(pb, dtype=torch.uint8, device="cuda")
    _lib.check(lib.ivftq_probe(qn.data_ptr(), idx._cent.data_ptr(), nq, L, d, n_p,
                               probe.data_ptr(), coarse.data_ptr(), pscr.data_ptr(), pb,
                               _lib.stream_ptr()))
    ev[2].record()
    qrot = torch.empty((nq, d), dtype=torch.float32, device="cuda")
    idx._rotate(qn, nq, qrot)
    ev[3].record()
    ids, sc = idx._scan(qn, nq, probe, coarse, n_p, 10, qrot)
    ev[4].record()
    torch.cuda.synchronize()
    t = [ev[i].elapsed_time(ev[i + 1]) * 1000 for i in range(4)]
    print(f"normalize {t[0]:.0f} us | probe {t[1]:.0f} | rotate {t[2]:.0f} | scan+regroup+merge {t[3]:.0f} | total {sum(t):.0f}")
