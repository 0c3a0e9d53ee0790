"""Summarise the scan_tc timeline trace (IVFTQ_TRACE output of CTA 0)."""
import sys
import numpy as np
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace.txt"
rows = [list(map(int, l.split())) for l in open(path) if not l.startswith('#')]
a = np.array(rows, dtype=np.int64)
t, prod, ds, de, ms, me, es, ee, tile, nt, nqt = a.T
span = ee.max() - ds.min()
print(f"tiles {len(a)} items {(tile == 0).sum()} span {span} cycles, {span / len(a):.0f}/tile")
for lo, hi in [(0, 60), (60, 200), (200, len(a))]:
    sl = slice(lo, hi)
    print(f"[{lo},{hi}) dec {np.median((de - ds)[sl]):.0f} mma {np.median((me - ms)[sl]):.0f} "
          f"epi {np.median((ee - es)[sl]):.0f} | period dec {np.median(np.diff(de[sl])):.0f} "
          f"mma {np.median(np.diff(me[sl])):.0f} epi {np.median(np.diff(ee[sl])):.0f}")
idle = es[1:] - ee[:-1]
print("epi idle frac %.2f" % (idle[idle > 0].sum() / span))
didle = ds[1:] - de[:-1]
print("dec idle frac %.2f" % (didle[didle > 0].sum() / span))
f = np.flatnonzero(tile == 0)[1:]
print("item start: dec dur median %.0f, mma gap median %.0f, epi last-tile dur median %.0f" % (
    np.median((de - ds)[f]), np.median(ms[f] - me[f - 1]), np.median((ee - es)[f - 1])))
ok = ee > 0
g = np.diff(ee[ok])
ti = tile[ok][1:]
n = nt[ok][1:]
cats = {"first": ti == 0, "second": ti == 1, "third": ti == 2, "last": ti == n - 1,
        "mid": (ti > 2) & (ti < n - 1)}
tot = g.sum()
for k, m in cats.items():
    print(f"{k:7s} n={m.sum():4d} sum={g[m].sum():9d} ({100 * g[m].sum() / tot:4.1f}%) "
          f"mean={g[m].mean():7.0f}")
