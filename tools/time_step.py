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
arith = sys.argv[5] if len(sys.argv) > 5 else "exact"
full = app == "full"  # the full timestep: dycore + column physics (full_step)
asuca = app == "asuca"  # the ASUCA time scheme (asuca_step)
rk3 = app == "rk3"  # Wicker-Skamarock RK3 of the dycore step (rk3_step)
if full or asuca or rk3:
    app = "dycore"
eng = hfb.Engine(app)
if app == "dycore":
    eng.set_option("arith", arith)
    if len(sys.argv) > 7:  # kernel variant (hfb_set_option "variant")
        eng.set_option("variant", sys.argv[7])
    if len(sys.argv) > 6 and sys.argv[6] != "0":  # A/B build only (libhfb_variants.so):
        eng.set_option("debug_skip", sys.argv[6])     # 1 = no advection, 2 = no acoustic
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
    if asuca:
        kdmp = nz - max(1, nz // 4)
        for k, v in dict(nsound=6, nbnd=8, kdmp=kdmp).items():
            eng.set(k, v)
        for k, v in dict(rdmp=0.2, rnbnd=1.0 / 8, rnzd=1.0 / (nz - kdmp)).items():
            eng.set(k, v)
        entry, bpp = "asuca_step", 2496
    if rk3:
        entry, bpp = "rk3_step", 88 + 2 * 128
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
print(f"{entry} [{arith}] {nx}x{ny}x{nz}: {ms:.4f} ms/step  {nx*ny*nz/ms*1e3:.3e} pt/s  "
      f"{bpp*nx*ny*nz/ms/1e6:.0f} GB/s(alg)")
if asuca:  # per-kernel device times of 3 more steps (CUDA events around every launch)
    eng.profile(True, clear=True)
    eng.profile(True)
    for _ in range(3):
        eng.enqueue(entry)
    eng.synchronize()
    eng.profile(False)
    pts = nx * ny * nz
    for kname, b in (("asuca_tend", 80), ("asuca_acoustic_a", 80), ("asuca_acoustic_b", 112),
                     ("asuca_stage_end", 48)):
        t, n = eng.kernel_time(kname)
        if n:
            print(f"  {kname}: {n // 3} launches/step, {t / n:.4f} ms each, "
                  f"{b * pts / (t / n) / 1e6:.0f} GB/s(alg, {b} B/pt)")
