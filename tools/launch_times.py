"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name + grid."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, gi, vi = hdr.index("Kernel Name"), hdr.index("Grid Size"), hdr.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows:
    agg[(r[ki].split("(")[0][-40:], r[gi])].append(float(r[vi]) / 1000)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[0]:40s} {k[1]:14s} n={len(v):4d} mean={sum(v) / len(v):7.2f}us tot={sum(v):8.1f}us {100 * sum(v) / tot:5.1f}%")
print(f"total {tot:.1f} us")
