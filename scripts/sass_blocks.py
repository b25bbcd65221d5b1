"""Summarise an ncu --page source (SASS) CSV export by basic block: stall-sample share,
instruction mix.  Usage: ncu -i X.ncu-rep --page source --csv --print-source sass > s.csv;
python scripts/sass_blocks.py s.csv [min_share]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
hdr = rows[1]
data = rows[2:]
isrc = hdr.index("Source")
iss = hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
blocks, cur = [], None
for i, r in enumerate(data):
    ex = float(r[iex] or 0)
    s = float(r[iss] or 0)
    op = r[isrc].split()
    op = (op[1] if op and op[0].startswith('@') else (op[0] if op else '')).split('.')[0]
    if cur is None or ex != cur['ex']:
        cur = dict(start=i, ex=ex, n=0, s=0, ops=collections.Counter())
        blocks.append(cur)
    cur['n'] += 1
    cur['s'] += s
    cur['ops'][op] += 1
T = sum(b['s'] for b in blocks)
tot_ex = collections.Counter()
for r in data:
    op = r[isrc].split()
    op = (op[1] if op and op[0].startswith('@') else (op[0] if op else '')).split('.')[0]
    tot_ex[op] += float(r[iex] or 0)
print("samples", T, " warp-instructions", sum(tot_ex.values()))
print("top opcodes (executed):", {k: f"{v / 1e6:.2f}M" for k, v in tot_ex.most_common(12)})
for b in blocks:
    if b['s'] / T > thr:
        print(f"{b['start']:5d} n={b['n']:4d} exec={b['ex']:8.0f} samp%={100 * b['s'] / T:5.1f}  {dict(b['ops'].most_common(5))}")
