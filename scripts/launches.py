"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: mean us and share per kernel."""
import collections
import csv
import sys

for fn in sys.argv[1:]:
    rows = [r for r in csv.reader(open(fn)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    d = collections.defaultdict(list)
    clk = collections.defaultdict(list)
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            d[r[ki][:48]].append(float(r[vi].replace(",", "")))
        elif r[mi] == "sm__cycles_elapsed.avg.per_second":
            clk[r[ki][:48]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    print(fn)
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        c = f" sm_clk={sum(clk[k]) / len(clk[k]) / 1e6:6.0f}MHz" if clk.get(k) else ""
        print(f"  {k:48s} n={len(v):3d} mean={sum(v) / len(v) / 1000:8.1f}us share={sum(v) / tot * 100:5.1f}%{c}")
