"""Fixture loading and input synthesis shared by the parity tests (test infrastructure)."""
import json
from pathlib import Path

import numpy as np

from cases import APPS, CASE_BY_NAME, CASES
import oracle

GOLDEN = Path(__file__).resolve().parent / "golden"
PARAMS = {"ntlm": 4}  # module parameters (sf_state.h90:3)


def _eval(expr, env):
    return int(eval(expr, {}, env))  # dims are simple integer expressions


def decl(app, name, ints):
    """(shape, lower) of a module array from its declared dims."""
    env = dict(PARAMS, **ints)
    shape, lower = [], []
    for d in APPS[app].arrays[name]:
        lo, hi = (d.split(":") if ":" in d else ("1", d))
        lo, hi = _eval(lo, env), _eval(hi, env)
        shape.append(hi - lo + 1)
        lower.append(lo)
    return tuple(shape), tuple(lower)


def make_inputs(case, order="C"):
    """Module arrays of the case in declared shape; unset arrays are zero-filled."""
    arrs = {}
    for name in APPS[case.app].arrays:
        shape, lower = decl(case.app, name, case.ints)
        if name in case.fills:
            seed, off, scale = case.fills[name]
            arrs[name] = oracle.fill(shape, seed, off, scale, order=order)
        else:
            arrs[name] = np.zeros(shape, order=order)
    return arrs


def load_golden(name):
    z = np.load(GOLDEN / f"{name}.npz")
    meta = json.loads(bytes(z["meta"]).decode())
    out = {k[4:]: z[k] for k in z.files if k.startswith("out.")}
    init = {k[5:]: z[k] for k in z.files if k.startswith("init.")}
    extra = {k: z[k] for k in z.files if k.startswith("out_accsim.")}
    return meta, out, init, extra


def run_oracle(case, arrs):
    """Execute the app's `main` through the C restatement, in place; returns scalars."""
    a, i, r = arrs, case.ints, case.reals
    if case.app == "diffusion":
        oracle.diffusion_run(i["nsteps"], r["coef"], a["t_old"], a["t_new"])
    elif case.app == "damping":
        oracle.damping(i["nx_mn"], i["nx_mx"], i["ny_mn"], i["ny_mx"], i["nz_mn"], i["nz_mx"],
                       r["tratio_bnd"], r["mtratio_bnd"], a["dens_ref_f"], a["dens_ptb_damp"],
                       a["dens_ptb_bnd"])
    elif case.app == "bounded":
        oracle.bounded(a["a"], a["b"])
    elif case.app == "surface_flux":
        oracle.surface_flux_main(i["tile_land"], a["cover_frac"], a["wind_speed"],
                                 a["flx_sum_x"], a["flx_sum_y"])
    elif case.app == "reduction":
        return {"total": oracle.grid_total(a["y"], 0.0, mode=0),
                "total_accsim": oracle.grid_total(a["y"], 0.0, mode=1)}
    elif case.app == "dycore":
        oracle.dycore_run(i["nsteps"], r, a["rho"], a["th"], a["u"], a["v"], a["w"], a["p"])
    elif case.app == "dycore_rk3":
        oracle.rk3_run(i["nsteps"], r, a["rho"], a["th"], a["u"], a["v"], a["w"], a["p"])
    elif case.app == "dycore_full":
        oracle.full_run(i["nsteps"], r, a["rho"], a["th"], a["u"], a["v"], a["w"], a["p"],
                        a["tsfc"], a["colm"])
    elif case.app == "asuca":
        oracle.asuca_run(i["nsteps"], r, i, a["rho"], a["th"], a["u"], a["v"], a["w"], a["p"])
    else:
        raise KeyError(case.app)
    return {}


def bits_equal(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))
