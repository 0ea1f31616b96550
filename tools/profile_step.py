#!/usr/bin/env python3
"""Minimal driver for ncu: set up one app on cuda:0 and run a few stream-only steps.

  python tools/profile_step.py [--app dycore|diffusion] [--nx 512 --ny 512 --nz 58] [--steps 3]
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_1710_08616_b200 as hfb  # noqa: E402
from paper_1710_08616_b200 import synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--app", default="dycore")
ap.add_argument("--nx", type=int, default=512)
ap.add_argument("--ny", type=int, default=512)
ap.add_argument("--nz", type=int, default=58)
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()

eng = hfb.Engine(a.app)
shape = (a.nz, a.nx, a.ny)
for k, v in dict(nx=a.nx, ny=a.ny, nz=a.nz, nsteps=1).items():
    eng.set(k, v)
if a.app == "dycore":
    for k, v in synthetic.DYCORE_SCALARS.items():
        eng.set(k, v)
    arrs = {k: synthetic.field(shape, *v, order="F") for k, v in synthetic.DYCORE_FILLS.items()}
    entry = "dycore_step"
elif a.app == "diffusion":
    eng.set("coef", 0.1)
    arrs = {"t_old": synthetic.field(shape, 1, 280.0, 10.0, order="F"),
            "t_new": np.zeros(shape, order="F")}
    entry = "diffuse_step"
else:
    raise SystemExit("app must be dycore or diffusion")
for k, v in arrs.items():
    eng.bind(k, v)
    eng.copy_to_device(k)
for _ in range(a.steps):
    eng.enqueue(entry)
eng.synchronize()
print("done", a.app, shape, a.steps)
