#!/usr/bin/env python3
"""Minimal driver for ncu: set up one app on cuda:0 and run a few stream-only steps.

  python tools/profile_step.py [--app dycore|diffusion] [--entry full_step|dycore_step|rk3_step]
                               [--nx 1581 --ny 1301 --nz 58] [--steps 3] [--variant V]
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
ap.add_argument("--entry", default="full_step")
ap.add_argument("--variant", default=None)
ap.add_argument("--nx", type=int, default=1581)
ap.add_argument("--ny", type=int, default=1301)
ap.add_argument("--nz", type=int, default=58)
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()

eng = hfb.Engine(a.app)
if a.variant:
    eng.set_option("variant", a.variant)
shape = (a.nz, a.nx, a.ny)
for k, v in dict(nx=a.nx, ny=a.ny, nz=a.nz, nsteps=1).items():
    eng.set(k, v)
if a.app == "dycore":
    for k, v in dict(synthetic.DYCORE_SCALARS, **synthetic.PHYS_SCALARS).items():
        eng.set(k, v)
    arrs = {k: synthetic.field(shape, *v, order="F") for k, v in synthetic.DYCORE_FILLS.items()}
    entry = a.entry
    if entry == "asuca_step":
        for k, v in synthetic.asuca_params(a.nz).items():
            eng.set(k, v)
    if entry == "full_step":
        arrs.update({k: synthetic.field((a.nx, a.ny), *v, order="F")
                     for k, v in synthetic.PHYS_FILLS.items()})
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
