"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
total device time, launches, mean -- which kernels a setup + solve step spends its
time in, without the CUDA-event profiler's per-launch brackets.
usage: python tools/launch_summary.py gpurun_out/launches.csv [out.txt]"""
import csv
import sys
from collections import defaultdict

rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    us = v / 1000.0 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1000.0)
    rows.append((int(r["ID"]), r["Kernel Name"], r.get("Grid Size", ""), us))
agg = defaultdict(lambda: [0, 0.0])
for _, k, _, us in rows:
    agg[k][0] += 1
    agg[k][1] += us
tot = sum(v[1] for v in agg.values())
out = [f"# {len(rows)} launches, {tot / 1000:.3f} ms device time (sum of serialised launch durations)",
       "# kernel  launches  total_ms  mean_us  share"]
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"{k}\t{n}\t{us / 1000:.3f}\t{us / n:.1f}\t{100 * us / tot:.1f}%")
text = "\n".join(out)
print(text)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(text + "\n")
