"""Summarise an ncu --set full report (.ncu-rep) into a short text block for profiles/.
usage: python scripts/ncu_summary.py report.ncu-rep [algorithmic_bytes]"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes_read.sum.per_second", "DRAM read throughput"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active (of peak)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active (of 64/SM)"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe (of peak)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    algo = float(sys.argv[2]) if len(sys.argv) > 2 else None
    rows = ncu_csv(rep, "--page", "raw")
    d = dict(zip(rows[0], rows[2]))
    print(f"kernel: {d.get('Kernel Name', '?')[:100]}")
    units = dict(zip(rows[0], rows[1]))
    for k, name in KEYS:
        v = d.get(k)
        if v is None:
            continue
        print(f"  {name:32s} {v} {units.get(k, '')}")
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    rd = float(d.get("dram__bytes_read.sum", "nan")) * scale.get(units.get("dram__bytes_read.sum", "byte"), 1.0)
    wr = float(d.get("dram__bytes_write.sum", "nan")) * scale.get(units.get("dram__bytes_write.sum", "byte"), 1.0)
    print(f"  DRAM read+write bytes per launch  {rd + wr:.0f}")
    if algo:
        print(f"  DRAM traffic / algorithmic bytes  {(rd + wr) / algo:.3f}  (algorithmic {algo:.0f} B)")
    st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v)) for h, v in d.items()
          if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")
          and v.replace(".", "").isdigit()]
    st.sort(key=lambda x: -x[1])
    tot = sum(v for _, v in st) or 1
    print("  top stall reasons (share of samples): " + ", ".join(f"{h} {v / tot * 100:.0f}%" for h, v in st[:6]))
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    ops = collections.Counter()
    for r in src[2:]:
        if len(r) > 5 and r[1].strip():
            t = r[1].split()
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            ops[op] += int(r[5] or 0)
    ev = {k: ops.get(k, 0) for k in ("UTMALDG", "FFMA2", "FMUL2", "SYNCS", "LDS", "STG", "SHFL")}
    print("  SASS executed (warp insts): " + ", ".join(f"{k} {v}" for k, v in ev.items()))


if __name__ == "__main__":
    main()
