"""Per-source-line attribution of an ncu --set full capture: joins the SASS page of the report
(per-instruction executed counts and stall samples) with the line table nvdisasm -g prints for
the same function of the built library (built with -lineinfo).

usage: python scripts/sass_lines.py report.ncu-rep paper_1610_01050_b200/librsft.so [top]
The .so must be the one the capture ran (same build)."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def ncu_sass(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kname = rows[0][1] if rows and len(rows[0]) > 1 else ""
    hdr = rows[1]
    ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[2:] if len(r) > max(ie, ss)]
    return kname, [(int(r[0], 16), r[1].strip(), int(r[ie] or 0), int(r[ss] or 0)) for r in body]


def mangled_candidates(kname):
    m = re.search(r"(k_[A-Za-z0-9_]+)", kname)
    return m.group(1) if m else None


def line_table(so, short):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
    tables = {}
    for cub in os.listdir(tmp):
        txt = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
        fn, loc = None, None
        for line in txt.splitlines():
            m = re.match(r"^\.text\.(\S+):$", line)
            if m:
                fn = m.group(1)
                tables[fn] = []
                loc = None
                continue
            m = re.match(r'^\s*//## File "([^"]+)", line (\d+)', line)
            if m:
                loc = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                continue
            m = re.match(r"^\s*/\*([0-9a-f]+)\*/\s+(\S.*?);", line)
            if m and fn is not None:
                tables[fn].append((int(m.group(1), 16), loc, m.group(2)))
    return {k: v for k, v in tables.items() if short in k}


def main():
    rep, so = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    kname, sass = ncu_sass(rep)
    short = mangled_candidates(kname)
    tabs = line_table(so, short)
    # pick the function whose instruction count and opcodes match the capture
    best = None
    for fn, tab in tabs.items():
        if len(tab) != len(sass):
            continue
        same = sum(1 for (_, _, op), (_, s, _, _) in zip(tab, sass) if op.split()[0] in s)
        if best is None or same > best[1]:
            best = (fn, same)
    if best is None:
        sys.exit(f"no function of {so} matches the capture of {kname} ({len(sass)} instructions)")
    tab = tabs[best[0]]
    inst, stall = collections.Counter(), collections.Counter()
    for (_, loc, _), (_, _, ie, ss) in zip(tab, sass):
        inst[loc] += ie
        stall[loc] += ss
    ti, ts = sum(inst.values()) or 1, sum(stall.values()) or 1
    print(f"{kname}\n  function {best[0]} ({len(tab)} SASS instructions)")
    print(f"  {'line':28s} {'warp insts':>14s} {'%':>6s} {'stall smp':>10s} {'%':>6s}")
    for loc, v in sorted(inst.items(), key=lambda kv: -kv[1])[:top]:
        print(f"  {str(loc):28s} {v:14d} {100 * v / ti:6.1f} {stall[loc]:10d} {100 * stall[loc] / ts:6.1f}")


if __name__ == "__main__":
    main()
