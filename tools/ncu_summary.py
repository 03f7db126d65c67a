"""Summarise ncu --set full reports (gpurun_out/<tag>_*.ncu-rep) into one table per
launch: duration, DRAM bytes (read + write), achieved DRAM GB/s, memory / compute
throughput, occupancy, registers -- the per-launch 'traffic' that bench.py reports."""
import csv
import glob
import io
import json
import re
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
want = {"Duration": "dur", "DRAM Throughput": "dram_pct", "Memory Throughput": "mem",
        "Compute (SM) Throughput": "sm_pct", "Achieved Occupancy": "occ", "Registers Per Thread": "regs",
        "Grid Size": "grid", "L2 Hit Rate": "l2hit", "L1/TEX Hit Rate": "l1hit"}
rows = []
CAPTURES = ("gs", "gs_seg", "lfmis", "evolution", "spgemm_hash", "spgemm_sort", "arnoldi", "masked", "relax0",
            "jacobi", "prolong", "sell_spmv", "vcycle_fused", "count")
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1.0, "nsecond": 1.0, "us": 1e3,
         "usecond": 1e3, "ms": 1e6, "msecond": 1e6}
reps = [f"gpurun_out/{tag}_{c}.ncu-rep" for c in CAPTURES if glob.glob(f"gpurun_out/{tag}_{c}.ncu-rep")]
reps += sorted(r for r in glob.glob(f"gpurun_out/{tag}_*.ncu-rep") if r not in reps)
for rep in reps:
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    launches = {}
    for r in csv.reader(io.StringIO(det)):
        if len(r) < 15 or r[0] == "ID":
            continue
        # ncu's --kernel-name-base function leaves "unnamed>::" (anonymous namespace) prefixes
        base = r[4][:r[4].index("(")] if "(" in r[4] else r[4]
        name = base.replace("void ", "").replace("amgcu::<unnamed>::", "").replace("unnamed>::", "")
        d = launches.setdefault(r[0], {"kernel": name, "report": rep})
        if r[12] in want:
            key = want[r[12]]
            if key == "mem" and "mem" in d:
                key = "mem_gbs" if "byte/s" in r[13] else key
            d[key] = (r[14], r[13])
    rr = list(csv.reader(io.StringIO(raw)))
    if rr:
        hdr, units = rr[0], rr[1]
        for r in rr[2:]:
            d = launches.get(r[0])
            if d is None:
                continue
            def num(name, r=r):
                try:
                    k = hdr.index(name)
                    return float(r[k].replace(",", "")) * SCALE.get(units[k], 1.0)
                except (ValueError, IndexError):
                    return 0.0
            d["dram_bytes"] = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
            d["ns"] = num("gpu__time_duration.sum")
    rows.extend(launches.values())
print(f"| kernel | grid | duration | DRAM bytes | DRAM GB/s | DRAM % | L2 hit | SM % | occupancy | regs |")
print("|---|---|---|---|---|---|---|---|---|---|")
traffic = {}
for d in rows:
    ns = d.get("ns", 0.0)
    by = d.get("dram_bytes", 0.0)
    gbs = by / ns if ns else 0.0
    def g(k):
        v = d.get(k)
        return f"{v[0]} {v[1]}".strip() if v else ""
    print(f"| {d['kernel']} | {g('grid')} | {ns / 1e3:.1f} us | {by / 1e6:.1f} MB | {gbs:.0f} | {g('dram_pct')} | "
          f"{g('l2hit')} | {g('sm_pct')} | {g('occ')} | {g('regs')} |")
    traffic.setdefault(d["kernel"], []).append({"grid": g("grid"), "ns": ns, "dram_bytes": by})
json.dump(traffic, open(f"profiles/{tag}_traffic.json", "w"), indent=1)
