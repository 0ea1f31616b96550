#!/usr/bin/env python3
"""Small dycore step through the C ABI (for compute-sanitizer runs of the step kernel)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "tests", ROOT / "oracle"):
    sys.path.insert(0, str(p))
import numpy as np
import paper_1710_08616_b200 as hfb
import oracle
from cases import DYCORE_FILLS, DYCORE_SCALARS

nx, ny, nz = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (64, 48, 58)
arrs = {k: oracle.fill((nz, nx, ny), *DYCORE_FILLS[k]) for k in DYCORE_FILLS}
ref = {k: v.copy() for k, v in arrs.items()}
oracle.dycore_run(1, DYCORE_SCALARS, *(ref[k] for k in ("rho", "th", "u", "v", "w", "p")))
with hfb.Engine("dycore", device=0) as eng:
    for k, v in dict(nx=nx, ny=ny, nz=nz, nsteps=1).items():
        eng.set(k, v)
    for k, v in DYCORE_SCALARS.items():
        eng.set(k, v)
    for k, a in arrs.items():
        eng.bind(k, a)
    eng.run("main")
for k in ("th", "u", "v", "w", "p"):
    d = np.flatnonzero(arrs[k].view(np.uint64) != ref[k].view(np.uint64))
    print(k, "mismatches", d.size, d[:5])
