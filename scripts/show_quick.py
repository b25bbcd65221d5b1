"""Summarise gpurun_out/ quick-loop results (bench lines, parity tail, launch list)."""
import csv
import json
import os

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
for f in ["q_bench.json", "q_bench_c5.json"]:
    try:
        d = json.loads(open(os.path.join(OUT, f)).read().strip().splitlines()[-1])
        r = d["roofline"]
        print(f, round(d["value"], 1), d["unit"], "ms/step", round(d["ms_per_step"], 4), "roof", round(r["achieved"]),
              round(r["frac"], 3), "k1 ms", round(r["avg_launch_ms"], 4), d.get("clocks", {}).get("sm_mhz"))
    except Exception as e:
        print(f, "ERR", e)
try:
    print(open(os.path.join(OUT, "q_parity.log")).read().strip().splitlines()[-1])
except Exception as e:
    print("parity ERR", e)
try:
    rows = [r for r in csv.DictReader(l for l in open(os.path.join(OUT, "q_launches.csv")) if not l.startswith("=="))]
    seen = {}
    for x in rows:
        seen[x["Kernel Name"][:70]] = x["Metric Value"]
    for k, v in seen.items():
        print(f"  {v:>10} ns  {k}")
except Exception as e:
    print("launches ERR", e)
