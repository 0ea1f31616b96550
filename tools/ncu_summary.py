#!/usr/bin/env python3
"""Summarise an ncu report (or a launch-list CSV) into a small text table for profiles/.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [alg_bytes_per_launch kernel=bytes ...]
  python tools/ncu_summary.py --launches gpurun_out/launches.csv
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "dsmem"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("lts__t_bytes.sum", "l2_bytes"),
]


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit)
    return f * scale if scale else f


def report(path, alg):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    print(f"# ncu --set full summary of {path}")
    for r in rows[2:]:
        name = r[col["Kernel Name"]].split("(")[0].split("::")[-1]
        vals = {}
        for m, short in METRICS:
            if m in col:
                vals[short] = (r[col[m]], units[col[m]])
        t_ms = float(vals["time"][0].replace(",", "")) * (1e-3 if vals["time"][1] in ("usecond", "us") else
                                                           1.0 if vals["time"][1] in ("msecond", "ms") else 1e-6)
        rd = to_bytes(*vals["dram_rd"])
        wr = to_bytes(*vals["dram_wr"])
        line = [f"{name}", f"time={t_ms:.4f}ms", f"dram_rd={rd/1e6:.1f}MB", f"dram_wr={wr/1e6:.1f}MB",
                f"traffic={(rd+wr)/1e6:.1f}MB", f"dram_GBps={(rd+wr)/t_ms/1e6:.0f}"]
        for short in ("dram%", "sm%", "occ%", "fp64%", "regs", "dsmem", "block", "grid"):
            if short in vals:
                line.append(f"{short}={vals[short][0]}")
        if name in alg:
            line.append(f"alg={alg[name]/1e6:.1f}MB alg_GBps={alg[name]/t_ms/1e6:.0f}")
        print("  ".join(line))


def launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ci = {h: i for i, h in enumerate(hdr)}
    agg = defaultdict(lambda: [0, 0.0])
    unit = None
    for r in rows[1:]:
        if len(r) < len(hdr) or r[ci["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ci["Kernel Name"]].split("(")[0].split("::")[-1]
        unit = r[ci["Metric Unit"]]
        agg[name][0] += 1
        agg[name][1] += float(r[ci["Metric Value"]].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"# launch list {path} (gpu__time_duration.sum, {unit}; cold-cache, serialised)")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:40s} launches={n:4d} total={t:12.1f} avg={t/n:10.1f} share={t/tot:6.3f}")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        alg = {}
        for a in sys.argv[2:]:
            k, v = a.split("=")
            alg[k] = float(v)
        report(sys.argv[1], alg)
