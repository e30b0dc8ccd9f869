"""Summarise an ncu report: key SOL metrics + top stall reasons + hottest SASS lines."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = ["Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Memory Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Achieved Active Warps Per SM", "Theoretical Occupancy", "Executed Instructions",
        "Dynamic Shared Memory Per Block", "Grid Size", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
kernel = None
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Kernel Name") != kernel:
        kernel = d.get("Kernel Name")
        print("==", kernel[:150])
    if d.get("Metric Name") in want:
        print(f"  {d['Metric Name']:<40} {d['Metric Unit']:<12} {d['Metric Value']}")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# one section per kernel: a "Kernel Name" row, a header row, then SASS lines
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1] if len(r) > 1 else "?", "hdr": None, "data": []}
        sections.append(cur)
    elif cur is not None and cur["hdr"] is None:
        cur["hdr"] = r
    elif cur is not None and len(r) == len(cur["hdr"]):
        cur["data"].append(dict(zip(cur["hdr"], r)))
key = "Warp Stall Sampling (All Samples)"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
for sec in sections:
    data, hdr = sec["data"], sec["hdr"]
    print("== SASS hot spots:", sec["name"][:120])
    tot = sum(float(d[key] or 0) for d in data) or 1
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = sorted(((sum(float(d[c] or 0) for d in data) / tot * 100, c) for c in stall_cols), reverse=True)[:8]
    print("  stalls:", ", ".join(f"{c[6:]} {v:.1f}%" for v, c in agg))
    for d in sorted(data, key=lambda d: -float(d[key] or 0))[:n]:
        st = max(((float(d[c] or 0), c) for c in stall_cols))
        print(f"  {float(d[key])/tot*100:5.1f}% {d['Instructions Executed']:>9} {d['Source'][:58]:<58} {st[1][6:]}")
