"""Launch-share table from an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python tools/launch_shares.py profiles/ncu_r01_bench_launches.csv [top_n]
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[1:]:
    name = r[ki]
    for pre in ("void ", ):
        if name.startswith(pre):
            name = name[len(pre):]
    name = name.split("(")[0] if name.startswith("stc::") else name[:80]
    tot[name] += float(r[vi]) / 1000.0
    cnt[name] += 1
total = sum(tot.values())
print("| share | launches | µs/launch | kernel |")
print("|---|---|---|---|")
for name, us in tot.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 10):
    print(f"| {100 * us / total:5.1f}% | {cnt[name]} | {us / cnt[name]:.1f} | `{name}` |")
