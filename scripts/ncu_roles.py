"""Attribute ncu warp-stall samples of scan_tc_kernel to pipeline roles."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
lines = []
for r in rows[2:]:
    if not r[iex].isdigit():
        continue
    lines.append((int(r[ia], 16), int(r[iex]), r[isrc], {hdr[i]: float(r[i] or 0) for i in stall_cols}))
base = lines[0][0]
def first(pat):
    return [l[0] for l in lines if pat in l[2]]
marks = {"producer": first("UBLKCP"), "mma": first("UTCHMMA"), "a_build": first("F2F.F16.F32"),
         "epilogue": first("LDTM")}
for k, v in marks.items():
    print(k, [hex(x - base) for x in (v[:1] + v[-1:])])
# role boundaries: sort first-occurrence of each role
bounds = sorted((min(v), k) for k, v in marks.items() if v)
def role(a):
    r = "setup"
    for s, k in bounds:
        if a >= s - 0x600:  # include the role's loop head
            r = k
    return r
agg = collections.defaultdict(lambda: collections.Counter())
inst = collections.Counter()
for a, ex, src, st in lines:
    rl = role(a) if 'PHASECHK' not in src and 'YIELD' not in src else "spin:" + role(a)
    for k, v in st.items():
        agg[rl][k] += v
    inst[rl] += ex
for rl, c in agg.items():
    tot = sum(c.values())
    top = ", ".join(f"{k[6:]}={v:.0f}" for k, v in c.most_common(5))
    print(f"{rl:16s} inst={inst[rl]/1e6:7.1f}M samples={tot:8.0f}  {top}")
