#!/usr/bin/env python3
"""One asuca_step on cuda:0 vs the oracle (debugging / compute-sanitizer runs).
  python tools/debug_asuca.py nx ny nz [nsteps] [nbnd] [nsound]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "tests", ROOT / "oracle"):
    sys.path.insert(0, str(p))
import numpy as np  # noqa: E402

from cases import _asu  # noqa: E402
from golden_io import make_inputs, run_oracle  # noqa: E402
from test_gpu_parity import run_engine  # noqa: E402

a = [int(x) for x in sys.argv[1:]]
nx, ny, nz = a[:3]
nsteps = a[3] if len(a) > 3 else 1
nbnd = a[4] if len(a) > 4 else 2
nsound = a[5] if len(a) > 5 else 6
case = _asu("dbg", nx, ny, nz, nsteps, nbnd=nbnd, nsound=nsound)
gpu = make_inputs(case)
ora = {k: v.copy() for k, v in gpu.items()}
run_oracle(case, ora)
run_engine(case, gpu)
for k in ("rho", "th", "u", "v", "w", "p"):
    d = np.argwhere(gpu[k].view(np.uint64) != ora[k].view(np.uint64))
    print(k, "mismatches:", len(d), "first (k,i,j):", d[:3].tolist() if len(d) else "")
