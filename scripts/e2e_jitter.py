"""Per-step distribution of the end-to-end search time (pinned host queries ->
numpy results) at C2, to separate host jitter from device time."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_17415_b200 import CoarsePartition, design_quantizer, generate_rotation
from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex
from paper_2605_17415_b200.workloads import mixture
n, d, L, nq = 1_000_000, 128, 1024, 10_000
x, means = mixture(n, d, 1000, 0.3, 1)
q, _ = mixture(nq, d, 1000, 0.3, 2, means=means)
rng = np.random.default_rng(0)
cent = x[rng.choice(n, L, replace=False)].astype(np.float64)
cent = (cent / np.linalg.norm(cent, axis=1)[:, None]).astype(np.float32)
idx = IvfTqIndex(IndexConfig(dim=d, bits=4, n_lists=L), design_quantizer(4, d),
                 generate_rotation(d, 42), CoarsePartition(L, d, cent))
idx.add_batch(torch.from_numpy(x).pin_memory())
qpin = torch.from_numpy(q).pin_memory()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(5):
    idx.search_batch(qpin, 10, 64)
ev, host = [], []
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 60):
    flush.fill_(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    idx.search_batch(qpin, 10, 64)
    e1.record()
    torch.cuda.synchronize()
    host.append((time.perf_counter() - t0) * 1e3)
    ev.append(e0.elapsed_time(e1))
ev, host = np.array(ev), np.array(host)
for name, a in (("event", ev), ("host", host)):
    print(name, "mean %.3f p50 %.3f p90 %.3f max %.3f" % (a.mean(), np.median(a), np.percentile(a, 90), a.max()))
print("per-step event ms:", " ".join("%.2f" % v for v in ev))
