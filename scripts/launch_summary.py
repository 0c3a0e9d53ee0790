"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv).

usage: python scripts/launch_summary.py launches.csv [--last N] [--md]

Groups launches by kernel (template arguments stripped), prints count, total
and mean duration and the share of the summed time. --last N keeps only the
last N launches (e.g. the timed steps of a bench run).
"""
import argparse
import csv
import re
from collections import OrderedDict


def short(name):
    name = re.sub(r"\(.*\)$", "", name)
    name = re.sub(r"^void ", "", name)
    base = name.split("<")[0].split("::")[-1]
    m = re.search(r"<(.*)>", name)
    if m and base.startswith(("scan_", "select", "merge")):
        base += "<" + m.group(1)[:24] + ">"
    return base


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] == "us":
            ns *= 1e3
        elif r["Metric Unit"] == "ms":
            ns *= 1e6
        rows.append((int(r["ID"]), short(r["Kernel Name"]), ns, r["Grid Size"], r["Block Size"]))
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--last", type=int, default=0)
    ap.add_argument("--md", action="store_true")
    a = ap.parse_args()
    rows = load(a.csv)
    if a.last:
        rows = rows[-a.last:]
    agg = OrderedDict()
    for _, k, ns, g, b in rows:
        e = agg.setdefault(k, [0, 0.0, g, b])
        e[0] += 1
        e[1] += ns
    tot = sum(e[1] for e in agg.values())
    items = sorted(agg.items(), key=lambda kv: -kv[1][1])
    if a.md:
        print("| kernel | launches | total us | mean us | share | grid | block |")
        print("|---|---:|---:|---:|---:|---|---|")
    for k, (c, ns, g, b) in items:
        if a.md:
            print(f"| {k} | {c} | {ns/1e3:.1f} | {ns/c/1e3:.1f} | {100*ns/tot:.1f}% | {g} | {b} |")
        else:
            print(f"{k:48s} {c:5d} {ns/1e3:10.1f}us {ns/c/1e3:9.1f}us {100*ns/tot:5.1f}%  {g} {b}")
    print(f"total {len(rows)} launches, {tot/1e3:.1f} us")


if __name__ == "__main__":
    main()
