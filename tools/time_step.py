#!/usr/bin/env python3
"""ms per dycore step (CUDA events on the engine stream) for quick A/B experiments."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_1710_08616_b200 as hfb  # noqa: E402
from paper_1710_08616_b200 import synthetic  # noqa: E402

import numpy as np  # noqa: E402

nx, ny, nz = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (512, 512, 58)))
app = sys.argv[4] if len(sys.argv) > 4 else "dycore"
full = app == "full"  # the full timestep: dycore + column physics (full_step)
if full:
    app = "dycore"
eng = hfb.Engine(app)
for k, v in dict(nx=nx, ny=ny, nz=nz, nsteps=1).items():
    eng.set(k, v)
if app == "dycore":
    for k, v in synthetic.DYCORE_SCALARS.items():
        eng.set(k, v)
    arrs = {k: synthetic.field((nz, nx, ny), *v, order="F")
            for k, v in synthetic.DYCORE_FILLS.items()}
    entry, bpp = "dycore_step", 88
    if full:
        eng.set("ch", 0.05)
        eng.set("rrelax", 0.01)
        arrs["tsfc"] = synthetic.field((nx, ny), 13, 300.0, 2.0, order="F")
        arrs["colm"] = synthetic.field((nx, ny), 14, 300.0, 0.5, order="F")
        entry = "full_step"
else:
    eng.set("coef", 0.1)
    arrs = {"t_old": synthetic.field((nz, nx, ny), 1, 280.0, 10.0, order="F"),
            "t_new": np.zeros((nz, nx, ny), order="F")}
    entry, bpp = "diffuse_step", 24
for k, a in arrs.items():
    eng.bind(k, a)
    eng.copy_to_device(k)
s = torch.cuda.ExternalStream(eng.stream)
for _ in range(5):
    eng.enqueue(entry)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 40
e0.record(s)
for _ in range(n):
    eng.enqueue(entry)
e1.record(s)
eng.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"{app} {nx}x{ny}x{nz}: {ms:.4f} ms/step  {nx*ny*nz/ms*1e3:.3e} pt/s  "
      f"{bpp*nx*ny*nz/ms/1e6:.0f} GB/s(alg)")
