"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

usage: python scripts/ncu_lines.py report.ncu-rep <cubin> <mangled-kernel-name> [top] [kernel-regex]

The report's SASS source page (ncu --page source --print-source sass) gives
per-instruction stall samples by absolute address; `nvdisasm -g` on the
kernel's cubin (cuobjdump -xelf all lib.so) gives per-offset source lines
(built with -lineinfo). Joined on offset-from-function-start.
"""
import collections
import csv
import io
import re
import subprocess
import sys


def line_map(cubin, fn):
    sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    out, cur, inside = {}, None, False
    for ln in sass.splitlines():
        if ln.startswith("//----") and ".text." in ln:
            inside = fn in ln
            continue
        if not inside:
            continue
        m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m:
            out[int(m.group(1), 16)] = cur
    return out


def main():
    rep, cubin, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    # optional 5th argument: kernel-name regex, for reports holding several kernels
    filt = ["-k", "regex:" + sys.argv[5]] if len(sys.argv) > 5 else []
    txt = subprocess.run(["ncu", "-i", rep, *filt, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    ia, iex, isrc = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Source")
    stall = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    lm = line_map(cubin, fn)
    base = None
    agg = collections.defaultdict(collections.Counter)
    ins = collections.Counter()
    srcs = {}
    for r in rows[2:]:
        if len(r) <= iex or not r[iex].strip().isdigit():
            continue
        a = int(r[ia], 16)
        if base is None:
            base = a
        key = lm.get(a - base, ("?", 0))
        ins[key] += int(r[iex])
        for i in stall:
            v = float(r[i] or 0)
            if v:
                agg[key][hdr[i][6:]] += v
        srcs.setdefault(key, r[isrc].strip())
    tot = sum(sum(c.values()) for c in agg.values())
    print(f"total stall samples {tot:.0f}")
    for key, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
        s = sum(c.values())
        reasons = ", ".join(f"{k}={v:.0f}" for k, v in c.most_common(3))
        print(f"{key[0]}:{key[1]:<5d} {100*s/tot:5.1f}%  inst={ins[key]/1e6:6.2f}M  {reasons}")


if __name__ == "__main__":
    main()
