"""Standalone ivftq_gemm_nt timing at the C2 coarse shape (10k x 1024 x 128, f32 B, f64 C)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_17415_b200 import _lib
L = _lib.lib()
M, N, K = 10000, 1024, 128
A = torch.randn(M, K, dtype=torch.float64, device="cuda")
B = torch.randn(N, K, dtype=torch.float32, device="cuda")
Cm = torch.empty(M, N, dtype=torch.float64, device="cuda")
run = lambda: _lib.check(L.ivftq_gemm_nt(A.data_ptr(), B.data_ptr(), _lib.IVFTQ_F32, M, N, K, Cm.data_ptr(), _lib.IVFTQ_F64, None))
run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    run()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"gemm_nt {M}x{N}x{K}: {ms*1000:.1f} us, {2*M*N*K/ms/1e9:.1f} TFLOP/s")
