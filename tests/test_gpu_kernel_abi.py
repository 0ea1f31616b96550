"""The generated-kernel ABI (include/hfb.h, codegen.cpp:397-519): what the reference's
generated host code would call instead of launching its CUDA-Fortran kernels. The test
plays that host code — transfers (hfrt_*), device views (hfb_device_array), then the
hfk<i>_<routine> launches with the generated grid/block and argument order, step by
step — and the result must equal the reference interpreter's goldens bit for bit."""
import ctypes

import numpy as np
import pytest

import paper_1710_08616_b200 as hfb
from paper_1710_08616_b200.runtime import lib
from cases import APPS, CASE_BY_NAME
from golden_io import bits_equal, decl, load_golden, make_inputs

pytestmark = pytest.mark.gpu


class Dim3(ctypes.Structure):
    _fields_ = [("x", ctypes.c_uint32), ("y", ctypes.c_uint32), ("z", ctypes.c_uint32)]


class HfbArray(ctypes.Structure):
    _fields_ = [("origin", ctypes.c_void_p), ("pitch", ctypes.c_int64),
                ("plane", ctypes.c_int64), ("volume", ctypes.c_int64),
                ("lower", ctypes.c_int64 * 4), ("upper", ctypes.c_int64 * 4),
                ("rank", ctypes.c_int32), ("roles", ctypes.c_int32), ("slot", ctypes.c_void_p)]


def device_array(eng, name):
    a = HfbArray()
    rc = lib().hfb_device_array(eng._h, eng.module.encode(), name.encode(), ctypes.byref(a))
    assert rc == 0, hfb.runtime.lib().hfb_last_error()
    return a


def grid_for(ex, ey):
    """The generated launch: ceiling(real(extent)/real(B)) per axis, block 32 x 4
    (codegen.cpp:421-434)."""
    return Dim3((ex + 31) // 32, (ey + 3) // 4, 1), Dim3(32, 4, 1)


def call(fn, *args):
    f = getattr(lib(), fn)
    f.restype = ctypes.c_int
    rc = f(*args)
    assert rc == 0, (fn, lib().hfb_last_error())


def engine_for(case, arrs):
    app = APPS[case.app]
    eng = hfb.Engine(app.prog)
    for k, v in case.ints.items():
        eng.set(k, int(v))
    for k, v in case.reals.items():
        eng.set(k, float(v))
    for name, a in arrs.items():
        eng.bind(name, a, lower=decl(case.app, name, case.ints)[1])
    for name in arrs:
        eng.copy_to_device(name)
    return eng


def finish(case, eng, arrs):
    eng.synchronize()
    for name in arrs:
        eng.copy_from_device(name)
    eng.close()
    _, out, _, _ = load_golden(case.name)
    for k in APPS[case.app].outputs:
        if k in arrs:
            assert bits_equal(arrs[k], out[k]), f"{case.name}: {k} differs"


@pytest.mark.parametrize("name", ["diffusion_37x21x9_s3", "diffusion_33x5x3_s2",
                                  "diffusion_1x1x3_s2"])
def test_diffusion_through_generated_kernel_abi(name):
    case = CASE_BY_NAME[name]
    arrs = make_inputs(case)
    eng = engine_for(case, arrs)
    i = case.ints
    t_new, t_old = device_array(eng, "t_new"), device_array(eng, "t_old")
    grid, block = grid_for(i["nx"], i["ny"])
    D = ctypes.c_double
    I32 = ctypes.c_int32
    for _ in range(i["nsteps"]):  # diffusion.h90:44-59: hfk0 then hfk1 every step
        call("hfk0_diffuse_step", grid, block, D(case.reals["coef"]), I32(0), I32(i["nx"]),
             I32(i["ny"]), I32(i["nz"]), t_new, t_old, None)
        call("hfk1_diffuse_step", grid, block, I32(0), I32(i["nx"]), I32(i["ny"]),
             I32(i["nz"]), t_new, t_old, None)
    finish(case, eng, arrs)


@pytest.mark.parametrize("name", ["damping_37x21x9", "damping_70x9x58_neg"])
def test_damping_through_generated_kernel_abi(name):
    case = CASE_BY_NAME[name]
    arrs = make_inputs(case)
    eng = engine_for(case, arrs)
    i, r = case.ints, case.reals
    grid, block = grid_for(i["nx_mx"] - i["nx_mn"] + 1, i["ny_mx"] - i["ny_mn"] + 1)
    I32 = ctypes.c_int32
    call("hfk0_lateral_and_upper_damping", grid, block, I32(0), ctypes.c_double(r["mtratio_bnd"]),
         I32(i["nx_mn"]), I32(i["nx_mx"]), I32(i["ny_mn"]), I32(i["ny_mx"]), I32(i["nz_mn"]),
         I32(i["nz_mx"]), ctypes.c_double(r["tratio_bnd"]), device_array(eng, "dens_ptb_bnd"),
         device_array(eng, "dens_ptb_damp"), device_array(eng, "dens_ref_f"), None)
    finish(case, eng, arrs)


@pytest.mark.parametrize("name", ["bounded_37x21", "bounded_3x3"])
def test_bounded_through_generated_kernel_abi(name):
    case = CASE_BY_NAME[name]
    arrs = make_inputs(case)
    eng = engine_for(case, arrs)
    nx, ny = case.ints["nx"], case.ints["ny"]
    grid, block = grid_for(max(nx - 2, 1), max(ny - 2, 1))  # startAt(2,2) endAt(nx-1,ny-1)
    call("hfk0_interior_update", grid, block, ctypes.c_int32(nx), ctypes.c_int32(ny),
         device_array(eng, "a"), device_array(eng, "b"), None)
    finish(case, eng, arrs)


@pytest.mark.parametrize("name", ["surface_flux_37x21_t1", "surface_flux_33x7_t3"])
def test_surface_flux_through_generated_kernel_abi(name):
    case = CASE_BY_NAME[name]
    arrs = make_inputs(case)
    arrs["cover_frac"] -= 0.5  # driver.h90 setup(): the host-side shift before the copy-in
    eng = engine_for(case, arrs)
    nx, ny = case.ints["nx"], case.ints["ny"]
    grid, block = grid_for(nx, ny)
    call("hfk0_sf_slab_flx_tile_run", grid, block, ctypes.c_int32(nx), ctypes.c_int32(ny),
         ctypes.c_int32(case.ints["tile_land"]), device_array(eng, "cover_frac"),
         device_array(eng, "flx_sum_x"), device_array(eng, "flx_sum_y"),
         device_array(eng, "wind_speed"), None)
    finish(case, eng, arrs)
