#!/usr/bin/env python3
"""Stall-reason shares and SASS opcode mix of the kernels in an ncu report."""
import collections
import csv
import io
import subprocess
import sys

path = sys.argv[1]
raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
seen = set()
for r in rows[2:]:
    name = r[h.index("Kernel Name")].split("(")[0].split("::")[-1]
    if name in seen:
        continue
    seen.add(name)
    st = [(h[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i].replace(",", "") or 0))
          for i in range(len(h))
          if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")]
    tot = sum(v for _, v in st) or 1
    print(name, "stalls:", " ".join(f"{k}={v / tot:.2f}" for k, v in sorted(st, key=lambda x: -x[1])[:8]))
src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr_i = next(k for k, r in enumerate(rows) if "Source" in r)
h = rows[hdr_i]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ops, stall = collections.Counter(), collections.Counter()
for r in rows[hdr_i + 1:]:
    if len(r) <= iE or r[0] == "Kernel Name":
        continue
    try:
        n, w = int(r[iE]), int(r[iW])
    except ValueError:
        continue
    op = r[iS].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    ops[o] += n
    stall[o] += w
tot, totw = sum(ops.values()) or 1, sum(stall.values()) or 1
print("opcode mix (share of executed, share of stall samples):")
print("  " + "  ".join(f"{o}={n / tot:.3f}/{stall[o] / totw:.3f}" for o, n in ops.most_common(16)))
