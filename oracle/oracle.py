"""ctypes front-end of the CPU restatement (oracle/liboracle.so). TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module, and only as the checker or the timed CPU baseline —
never as the product path.

All arrays are numpy float64 arrays shaped by the DECLARED dims of the
Hybrid-Fortran object, e.g. t_old(nz,nx,ny) -> shape (nz, nx, ny); any strides are
accepted (the reference's ArrayValue order is C order over those dims,
/root/reference/proj/src/interp.cpp:485-494; the Fortran KIJ order is F order).
`lower` gives the declared lower bounds (default 1).
"""
import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"
HFT_REF = HERE / "_ref" / "hft_ref"


class View(ctypes.Structure):
    _fields_ = [("p", ctypes.c_void_p), ("off", ctypes.c_int64), ("sk", ctypes.c_int64),
                ("si", ctypes.c_int64), ("sj", ctypes.c_int64), ("sl", ctypes.c_int64)]


class DynParams(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
                ("dt", ctypes.c_double), ("rdx", ctypes.c_double), ("rdy", ctypes.c_double),
                ("rdz", ctypes.c_double), ("cs2", ctypes.c_double), ("grav", ctypes.c_double),
                ("th0", ctypes.c_double)]


class AsucaParams(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
                ("dt", ctypes.c_double), ("rdx", ctypes.c_double), ("rdy", ctypes.c_double),
                ("rdz", ctypes.c_double), ("cs2", ctypes.c_double), ("grav", ctypes.c_double),
                ("th0", ctypes.c_double), ("nsound", ctypes.c_int64), ("nbnd", ctypes.c_int64),
                ("kdmp", ctypes.c_int64), ("rdmp", ctypes.c_double), ("rnbnd", ctypes.c_double),
                ("rnzd", ctypes.c_double)]


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", str(HERE), "oracle"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        i64, dbl, V = ctypes.c_int64, ctypes.c_double, View
        L.ora_diffusion_run.argtypes = [i64, i64, i64, i64, dbl, V, V]
        L.ora_damping.argtypes = [i64] * 6 + [dbl, dbl, V, V, V]
        L.ora_bounded.argtypes = [i64, i64, V, V]
        L.ora_sf_setup.argtypes = [i64, i64, i64, V]
        L.ora_sf_physics_run.argtypes = [i64, i64, i64, V, V, V, V]
        L.ora_grid_total.argtypes = [i64, i64, i64, dbl, V, ctypes.c_int]
        L.ora_grid_total.restype = dbl
        L.ora_dycore_run.argtypes = [i64, ctypes.POINTER(DynParams), V, V, V, V, V, V]
        L.ora_dycore_run.restype = ctypes.c_int
        L.ora_rk3_run.argtypes = [i64, ctypes.POINTER(DynParams), V, V, V, V, V, V]
        L.ora_asuca_run.argtypes = [i64, ctypes.POINTER(AsucaParams), V, V, V, V, V, V]
        L.ora_asuca_run.restype = ctypes.c_int
        L.ora_rk3_run.restype = ctypes.c_int
        L.ora_full_run.argtypes = [i64, ctypes.POINTER(DynParams), dbl, dbl] + [V] * 8
        L.ora_full_run.restype = ctypes.c_int
        L.ora_fill.argtypes = [ctypes.c_void_p, i64, ctypes.c_uint64, dbl, dbl]
        L.ora_splitmix64.argtypes = [ctypes.c_uint64]
        L.ora_splitmix64.restype = ctypes.c_uint64
        L.ora_set_threads.argtypes = [ctypes.c_int]
        L.ora_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def view(a, lower=None):
    """Strided view of a declared-shape array. Rank 2 arrays map to (i, j);
    rank 3 to (k|lt, i, j); rank 4 to (k, i, j, l)."""
    assert a.dtype == np.float64
    st = [s // 8 for s in a.strides]
    lower = list(lower) if lower is not None else [1] * a.ndim
    if a.ndim == 2:
        sk, si, sj, sl = 0, st[0], st[1], 0
        lk, li, lj, ll = 0, lower[0], lower[1], 0
    elif a.ndim == 3:
        sk, si, sj, sl = st[0], st[1], st[2], 0
        lk, li, lj, ll = lower[0], lower[1], lower[2], 0
    else:
        sk, si, sj, sl = st
        lk, li, lj, ll = lower
    off = -(lk * sk + li * si + lj * sj + ll * sl)
    return View(a.ctypes.data, off, sk, si, sj, sl)


def fill(shape, seed, offset, scale, order="C"):
    """SURVEY §8(d) synthetic field over the declared shape (flat = row-major index)."""
    n = int(np.prod(shape))
    flat = np.empty(n, np.float64)
    lib().ora_fill(flat.ctypes.data, n, seed, offset, scale)
    a = flat.reshape(shape)
    return np.asfortranarray(a) if order == "F" else a


def set_threads(n):
    lib().ora_set_threads(int(n))


def num_threads():
    return lib().ora_num_threads()


# --- per-app entry points (semantics of `main` in each app) -------------------------

def diffusion_run(nsteps, coef, t_old, t_new):
    nz, nx, ny = t_old.shape
    lib().ora_diffusion_run(nsteps, nx, ny, nz, coef, view(t_old), view(t_new))


def damping(nx_mn, nx_mx, ny_mn, ny_mx, nz_mn, nz_mx, tratio_bnd, mtratio_bnd,
            dens_ref_f, dens_ptb_damp, dens_ptb_bnd):
    lo3 = (nz_mn, nx_mn, ny_mn)
    lib().ora_damping(nx_mn, nx_mx, ny_mn, ny_mx, nz_mn, nz_mx, tratio_bnd, mtratio_bnd,
                      view(dens_ref_f, lo3), view(dens_ptb_damp, lo3),
                      view(dens_ptb_bnd, lo3 + (1,)))


def bounded(a, b):
    nx, ny = a.shape
    lib().ora_bounded(nx, ny, view(a), view(b))


def surface_flux_main(tile_land, cover_frac, wind_speed, flx_sum_x, flx_sum_y):
    ntlm, nx, ny = cover_frac.shape
    lib().ora_sf_setup(ntlm, nx, ny, view(cover_frac))
    lib().ora_sf_physics_run(nx, ny, tile_land, view(cover_frac), view(wind_speed),
                             view(flx_sum_x), view(flx_sum_y))


def grid_total(y, total=0.0, mode=0):
    nz, nx, ny = y.shape
    return lib().ora_grid_total(nx, ny, nz, total, view(y), mode)


def dycore_run(nsteps, params, rho, th, u, v, w, p):
    nz, nx, ny = th.shape
    prm = DynParams(nx, ny, nz, params["dt"], params["rdx"], params["rdy"], params["rdz"],
                    params["cs2"], params["grav"], params["th0"])
    rc = lib().ora_dycore_run(nsteps, ctypes.byref(prm), view(rho), view(th), view(u),
                              view(v), view(w), view(p))
    if rc:
        raise RuntimeError(f"ora_dycore_run failed ({rc})")


def full_run(nsteps, params, rho, th, u, v, w, p, tsfc, colm):
    """simulation_run_full: nsteps x (dycore_step; column_physics)."""
    nz, nx, ny = th.shape
    prm = DynParams(nx, ny, nz, params["dt"], params["rdx"], params["rdy"], params["rdz"],
                    params["cs2"], params["grav"], params["th0"])
    rc = lib().ora_full_run(nsteps, ctypes.byref(prm), params["ch"], params["rrelax"],
                            view(rho), view(th), view(u), view(v), view(w), view(p),
                            view(tsfc), view(colm))
    if rc:
        raise RuntimeError(f"ora_full_run failed ({rc})")


def rk3_run(nsteps, params, rho, th, u, v, w, p):
    """simulation_run_rk3: nsteps x rk3_step."""
    nz, nx, ny = th.shape
    prm = DynParams(nx, ny, nz, params["dt"], params["rdx"], params["rdy"], params["rdz"],
                    params["cs2"], params["grav"], params["th0"])
    rc = lib().ora_rk3_run(nsteps, ctypes.byref(prm), view(rho), view(th), view(u), view(v),
                           view(w), view(p))
    if rc:
        raise RuntimeError(f"ora_rk3_run failed ({rc})")


def asuca_run(nsteps, params, ints, rho, th, u, v, w, p):
    """simulation_run_asuca: nsteps x asuca_step (apps/dycore/asuca.h90). `params` holds
    the dyn_state reals (dt..th0, rdmp, rnbnd, rnzd), `ints` nsound, nbnd, kdmp."""
    nz, nx, ny = th.shape
    prm = AsucaParams(nx, ny, nz, params["dt"], params["rdx"], params["rdy"], params["rdz"],
                      params["cs2"], params["grav"], params["th0"], ints["nsound"],
                      ints["nbnd"], ints["kdmp"], params["rdmp"], params["rnbnd"],
                      params["rnzd"])
    rc = lib().ora_asuca_run(nsteps, ctypes.byref(prm), view(rho), view(th), view(u), view(v),
                             view(w), view(p))
    if rc:
        raise RuntimeError(f"ora_asuca_run failed ({rc})")
