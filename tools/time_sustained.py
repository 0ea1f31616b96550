#!/usr/bin/env python3
"""Sustained timing of the C4 full step (power-capped state): ~1 s of back-to-back steps
first, then 4 blocks of 50 steps (CUDA events) with the SM clock sampled by nvidia-smi.
  HFB_LIB=<lib> python tools/time_sustained.py [exact|fma] [entry]"""
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_1710_08616_b200 as hfb  # noqa: E402
from paper_1710_08616_b200 import synthetic  # noqa: E402

arith = sys.argv[1] if len(sys.argv) > 1 else "exact"
entry = sys.argv[2] if len(sys.argv) > 2 else "full_step"
nx, ny, nz = 1581, 1301, 58
eng = hfb.Engine("dycore")
eng.set_option("arith", arith)
for k, v in dict(nx=nx, ny=ny, nz=nz, nsteps=1).items():
    eng.set(k, v)
for k, v in dict(synthetic.DYCORE_SCALARS, **synthetic.PHYS_SCALARS).items():
    eng.set(k, v)
arrs = {k: synthetic.field((nz, nx, ny), *v, order="F") for k, v in synthetic.DYCORE_FILLS.items()}
arrs.update({k: synthetic.field((nx, ny), *v, order="F") for k, v in synthetic.PHYS_FILLS.items()})
for k, a in arrs.items():
    eng.bind(k, a)
    eng.copy_to_device(k)
s = torch.cuda.ExternalStream(eng.stream)
t0 = time.perf_counter()
while time.perf_counter() - t0 < 1.0:
    for _ in range(20):
        eng.enqueue(entry)
    eng.synchronize()
out = []
for blk in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(50):
        eng.enqueue(entry)
    e1.record(s)
    eng.synchronize()
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip()
    out.append(f"{e0.elapsed_time(e1) / 50:.4f}@{clk}")
print(f"{entry} [{arith}] sustained ms/step (block@MHz): {' '.join(out)}")
