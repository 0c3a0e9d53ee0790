"""Summarise a scan_vq timeline (IVFTQ_TRACE output of the trace build, CTA 0)."""
import sys

import numpy as np

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace.txt"
head = open(path).readline().strip()
a = np.loadtxt(path, comments="#", dtype=np.int64)
if a.ndim == 1:
    a = a[None]
t, prod, dec_e, mma_s, mma_e, epi_s, epi_e, dec_s, tile, nt, nq = a.T
n = len(a)
span = epi_e.max() - prod.min()
print(head)
print(f"tiles {n} items {(tile == 0).sum()} span {span} cycles, {span / n:.0f}/tile, nq median {np.median(nq):.0f}")
sl = slice(min(20, n // 4), n)
def med(x):
    return float(np.median(x[sl]))
print(f"durations: decode {med(dec_e - dec_s):.0f}  mma-issue {med(mma_e - mma_s):.0f}  epilogue {med(epi_e - epi_s):.0f}")
print(f"periods:   decode {med(np.diff(dec_e, prepend=dec_e[0])):.0f}  mma {med(np.diff(mma_s, prepend=mma_s[0])):.0f}  "
      f"epilogue {med(np.diff(epi_e, prepend=epi_e[0])):.0f}")
print(f"gaps: prod->dec_s {med(dec_s - prod):.0f}  dec_e->mma_s {med(mma_s - dec_e):.0f}  mma_e->epi_s {med(epi_s - mma_e):.0f}")
f = np.flatnonzero(tile == 0)[1:]
if len(f):
    print(f"item starts: mma gap {np.median(mma_s[f] - mma_s[f - 1]):.0f}  epi gap {np.median(epi_s[f] - epi_e[f - 1]):.0f}")
