#!/usr/bin/env python3
"""SASS instruction census per kernel of libdsinf.so (cuobjdump -sass): tcgen05 (UTC*MMA, LDTM),
TMA (UTMALDG / UTMAPF / UBLKCP), warp MMA (HMMA / IMMA), barriers (SYNCS) and LDSM counts.
  python tools/sass_census.py [paper_2207_00032_b200/libdsinf.so] > profiles/r2_sass_census.txt"""
import collections
import re
import subprocess
import sys

OPS = ["UTCHMMA", "UTCIMMA", "UTCQMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMAPF", "UBLKCP", "HMMA", "IMMA", "SYNCS", "LDSM"]
lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2207_00032_b200/libdsinf.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
kernels = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        kernels[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9]+)", line)
    if m and m.group(1) in OPS:
        kernels[cur][m.group(1)] += 1
names = subprocess.run(["c++filt"], input="\n".join(kernels), capture_output=True, text=True).stdout.splitlines()
print(f"SASS instruction census of {lib} (cuobjdump -sass, sm_100a)")
print("kernel (demangled prefix) : " + " ".join(OPS))
for (k, c), n in zip(kernels.items(), names):
    if c:
        print(n + " : " + " ".join(f"{op}={c[op]}" for op in OPS if c[op]))
