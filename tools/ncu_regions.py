#!/usr/bin/env python3
"""Per-loop breakdown of one kernel's SASS from an ncu report's source page: every
backward branch closes a region; prints warp-instructions executed and stall samples per
region (to tell which role / K phase of a warp-specialised kernel costs what).
  python tools/ncu_regions.py REPORT.ncu-rep KERNEL_REGEX [launch_skip]"""
import csv
import io
import re
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kre}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
# the page lists one block per function of the module ("Kernel Name", header, rows):
# keep the block of the kernel itself
blocks, cur = [], None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Kernel Name":
        cur = [r[1], []]
        blocks.append(cur)
    elif cur is not None and r:
        cur[1].append(r)
name, rows = next(b for b in blocks if re.search(kre, b[0]))
lines = [name]
hdr, rows = rows[0], rows[1:]
ia, isrc, isam, iex = (hdr.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                              "Instructions Executed"))
ins = [(int(r[ia], 16), r[isrc].strip(), int(r[isam] or 0), int(r[iex] or 0)) for r in rows]
addr = {a: n for n, (a, *_) in enumerate(ins)}
tot_s = sum(x[2] for x in ins) or 1
tot_e = sum(x[3] for x in ins) or 1
loops = []
for n, (a, src, *_) in enumerate(ins):
    m = re.search(r"BRA.*?0x([0-9a-f]+)", src)
    if m and int(m.group(1), 16) < a and int(m.group(1), 16) in addr:
        if n - addr[int(m.group(1), 16)] < 1000:  # (long jumps back are error-path returns)
            loops.append((addr[int(m.group(1), 16)], n))
print(f"{lines[0][:120]}")
print(f"{'region':>14s} {'instrs':>7s} {'exec share':>10s} {'stall share':>11s}")
for s, e in loops:
    se = sum(x[3] for x in ins[s:e + 1])
    ss = sum(x[2] for x in ins[s:e + 1])
    if se / tot_e > 0.01 or ss / tot_s > 0.01:
        print(f"{s:6d}-{e:<7d} {e - s + 1:7d} {se / tot_e:10.3f} {ss / tot_s:11.3f}")
