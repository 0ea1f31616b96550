#!/usr/bin/env python3
"""Opcode evidence from the built library: per kernel of libhfb.so (cuobjdump -sass), the
count of the Blackwell-specific instructions (TMA loads / prefetches, mbarrier ops, TMEM
stores / loads / allocation) and of a few others, static (in the code, not executed).
  python tools/sass_opcodes.py [paper_1710_08616_b200/libhfb.so]"""
import re
import subprocess
import sys
from collections import Counter

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1710_08616_b200/libhfb.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = ["UTMALDG", "UTMAPF", "UBLKPF", "SYNCS", "STTM", "LDTM", "UTCATOMSWS", "ELECT",
        "LDGSTS", "BAR", "DFMA", "DADD", "DMUL", "MUFU"]
arch = re.search(r"arch = (\w+)", sass)
print(f"# {lib}: {arch.group(1) if arch else '?'}; static opcode counts per kernel")
print(f"{'kernel':58s} " + " ".join(f"{k:>7s}" for k in KEYS))
seen = set()
for f in re.split(r"\n\s+Function : ", sass)[1:]:
    name = f.split("\n")[0].strip()
    m = re.search(r"(k_[a-z0-9_]+)(I[^E]*E)?", name)
    if not m:
        continue
    dem = subprocess.run(["c++filt", name[name.find("_Z"):]], capture_output=True,
                         text=True).stdout.strip() if "_Z" in name else name
    dem = re.sub(r"\(.*", "", dem.replace("hfb::(anonymous namespace)::", ""))
    if dem in seen:  # the step kernels' second object: the tolerance (FMA) build
        dem += " [fma]"
    seen.add(dem)
    ops = Counter()
    for line in f.split("\n"):
        mm = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if mm:
            ops[mm.group(2)] += 1
    print(f"{dem[:58]:58s} " + " ".join(f"{ops.get(k, 0):7d}" for k in KEYS))
