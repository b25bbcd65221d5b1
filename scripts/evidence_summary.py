"""Turn one evidence session's outputs (gpurun_out/<dir>: bench lines, launch lists with DRAM bytes,
ncu summaries) into a markdown summary and the per-step DRAM traffic table bench.py reports.

    python scripts/evidence_summary.py gpurun_out/bm profiles/r02b_summary.md [--traffic profiles/traffic.json]
"""
import collections
import csv
import glob
import json
import os
import sys

# the roofline's "dominant kernel" per workload: fused plans time the whole rsft_run call (every kernel
# of the step), split plans time rsft_execute (the fold + outer-FFT kernels)
def in_roofline(wl, kernel):
    return "split" in kernel if wl in ("c3_3d", "c5_cube") else True


def last_json(path):
    try:
        with open(path) as f:
            lines = [ln for ln in f.read().strip().splitlines() if ln.startswith("{")]
        return json.loads(lines[-1]) if lines else None
    except OSError:
        return None


def launch_table(fn):
    rows = [r for r in csv.reader(open(fn)) if len(r) > 10]
    if not rows:
        return {}
    hdr = rows[0]
    ki, vi, mi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"), hdr.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki]
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for i, m in per.items():
        for k, v in m.items():
            agg[names[i]][k].append(v)
    return agg


def main():
    src, out = sys.argv[1], sys.argv[2]
    traffic_path = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    L = []
    L.append(f"# Evidence summary ({os.path.basename(src.rstrip('/'))}; B200, one GPU)\n")
    smoke = os.path.join(src, "smoke.log")
    if os.path.exists(smoke):
        L.append("Smoke: " + " / ".join(ln.strip() for ln in open(smoke) if ln.strip()) + "\n")
    pt = os.path.join(src, "pytest_gpu.log")
    if os.path.exists(pt):
        tail = [ln.strip() for ln in open(pt) if ln.strip()][-2:]
        L.append("GPU tests (`pytest -m gpu`): " + " ".join(tail) + "\n")
    L.append("## Bench lines\n")
    L.append("| line | value | ms / step (median, p90) | roofline kernel | frac of measured peak | clocks |")
    L.append("|---|---|---|---|---|---|")
    for name in ["c4", "c4_two", "c1", "c2", "c3", "c5", "ref"]:
        d = last_json(os.path.join(src, f"bench_{name}.json"))
        if not d or "value" not in d:
            continue
        r = d.get("roofline") or {}
        st = d.get("step_ms") or {}
        ck = d.get("clocks") or {}
        L.append(f"| {name} ({d.get('config', {}).get('workload', '')}) | {d['value']:.4g} {d.get('unit', '')} | "
                 f"{d.get('ms_per_step', 0):.4f} ({st.get('median', 0):.4f}, {st.get('p90', 0):.4f}) | "
                 f"{str(r.get('kernel', ''))[:60]} | {r.get('frac', float('nan')):.3f} | "
                 f"{ck.get('sm_mhz', '')} MHz {ck.get('reasons', '')} |")
        if name == "c4":
            e = d.get("e2e") or {}
            cb = d.get("cpu_baseline") or {}
            L.append(f"\nc4 e2e (rsft_run_host, host buffers): {e.get('value', 0):.4g} {e.get('unit', '')}; "
                     f"CPU oracle: {cb.get('value', 0):.4g} {cb.get('unit', '')} on {cb.get('cores')} cores\n")
    L.append("\n## Step composition (ncu launch lists: cold-cache, serialised -- shares, not absolutes)\n")
    traffic = {}
    for fn in sorted(glob.glob(os.path.join(src, "launches_*.csv"))):
        wl = os.path.basename(fn)[len("launches_"):-4]
        agg = launch_table(fn)
        if not agg:
            continue
        tot = sum(sum(m.get("gpu__time_duration.sum", [])) for m in agg.values())
        L.append("```")
        L.append(fn)
        byts = 0.0
        for k, m in sorted(agg.items(), key=lambda x: -sum(x[1].get("gpu__time_duration.sum", []))):
            t = m.get("gpu__time_duration.sum", [])
            rd, wr = m.get("dram__bytes_read.sum", []), m.get("dram__bytes_write.sum", [])
            extra = ""
            if rd and wr:
                per = (sum(rd) + sum(wr)) / len(rd)
                if in_roofline(wl, k):
                    byts += per
                extra = f" dram/launch={per / 1e9:7.3f} GB"
            L.append(f"  {k[:56]:56s} n={len(t):3d} mean={sum(t) / len(t) / 1000:9.1f}us "
                     f"share={sum(t) / tot * 100:5.1f}%{extra}")
        L.append("```")
        if byts and not wl.startswith("bart"):
            traffic[wl] = int(byts)
    L.append("\n## ncu --set full captures (per-source-line attribution in the matching .lines.txt)\n")
    L.append("| capture | duration | DRAM read | DRAM read throughput | issue active | top stalls |")
    L.append("|---|---|---|---|---|---|")
    for fn in sorted(glob.glob(os.path.join(src, "prof_*.summary.txt"))):
        txt = open(fn).read()
        dur = next((ln.split("duration", 1)[1].strip() for ln in txt.splitlines() if ln.strip().startswith("duration")), "")
        rd = next((ln.split("DRAM read", 1)[1].strip() for ln in txt.splitlines() if ln.strip().startswith("DRAM read ")), "")
        thr = next((ln.split("throughput", 1)[1].strip() for ln in txt.splitlines() if "DRAM read throughput" in ln), "")
        iss = next((ln.split("peak)", 1)[1].strip() for ln in txt.splitlines() if "issue active" in ln), "")
        stl = next((ln.split(":", 1)[1].strip()[:80] for ln in txt.splitlines() if "top stall" in ln), "")
        L.append(f"| {os.path.basename(fn)[5:-12]} | {dur} | {rd} | {thr} | {iss} | {stl} |")
    L.append("\n## Bartlett (Alg. 2) vs RSFT segment mode, like for like (T = L segments per frame)\n")
    L.append("| shape | Bartlett frames/s | Bartlett HBM (design bytes / time, of peak) | RSFT segment mode frames/s | ratio |")
    L.append("|---|---|---|---|---|")
    for wl in ["c1_1d", "c2_2d", "c4_batched_2d", "c3_3d"]:
        b = last_json(os.path.join(src, f"bart_{wl}.json"))
        sg = last_json(os.path.join(src, f"seg_{wl}.json"))
        if not b or not sg:
            continue
        L.append(f"| {wl} | {b['value']:.4g} | {b['hbm']['design_frac']:.2f} ({b['hbm']['passes_over_input']} pass(es)) | "
                 f"{sg['value']:.4g} | {sg['value'] / b['value']:.1f}x |")
    with open(out, "w") as f:
        f.write("\n".join(L) + "\n")
    if traffic_path and traffic:
        old = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
        old.update(traffic)
        old["_source"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per step of the roofline's kernels (the "
                          f"whole rsft_run call for fused plans, the fold + outer-FFT kernels for split plans), mean "
                          f"per launch, from the launch lists in {src} (ncu --metrics, --clock-control none); "
                          f"committed as profiles/r02d_launches_*.csv")
        json.dump(old, open(traffic_path, "w"), indent=1)
    print("\n".join(L))


if __name__ == "__main__":
    main()
