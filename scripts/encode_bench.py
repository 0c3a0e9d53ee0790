"""Device-resident encode rate (ivftq_encode on rows already in HBM), CUDA events.
  python scripts/encode_bench.py [n] [d] [L]      (IVFTQ_ENCODE_F64=1: the f64 tail)"""
import os, sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_17415_b200 import CoarsePartition, design_quantizer, generate_rotation
from paper_2605_17415_b200.index import IndexConfig, IvfTqIndex
from paper_2605_17415_b200.workloads import mixture
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
L = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
x, _ = mixture(n, d, L, 0.3, 1)
rng = np.random.default_rng(0)
cent = x[rng.choice(n, L, replace=False)].astype(np.float64)
cent = (cent / np.linalg.norm(cent, axis=1)[:, None]).astype(np.float32)
idx = IvfTqIndex(IndexConfig(dim=d, bits=4, n_lists=L), design_quantizer(4, d),
                 generate_rotation(d, 42), CoarsePartition(L, d, cent))
xd = torch.from_numpy(x).cuda()
chunk = 250_000
ts = []
for rep in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(0, n, chunk):
        idx._encode_device(xd[s:s + chunk], defer_check=True)
    e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t = float(np.median(ts[1:]))
print(f"{'f64 tail' if os.environ.get('IVFTQ_ENCODE_F64') else 'tensor-core tail'} n={n} d={d} L={L}: "
      f"{t:.2f} ms per {n} rows = {n / t / 1e3:.1f} M adds/s (device encode, {chunk}-row chunks)")
