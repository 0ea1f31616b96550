"""Parity cases shared by the golden generator, the oracle tests and the GPU tests.

Each case names one Hybrid-Fortran app, its module scalars and the synthetic
fills of its module arrays (value = offset + scale * u(seed, flat),
flat = the logical row-major index over the declared dims). The golden fixtures
under tests/golden/ hold what the REFERENCE INTERPRETER produced for these
inputs (oracle/_ref/hft_ref, see tests/golden/make_golden.py).
"""
from dataclasses import dataclass, field
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
REF_APPS = Path("/root/reference/proj/tests/data/apps")  # generation time only
OWN_APPS = REPO / "apps"


@dataclass
class App:
    name: str
    sources: list          # (root, relative path); root "ref" or "own"
    module: str            # state module
    arrays: dict           # name -> tuple of declared-dim expressions (for shapes)
    outputs: list          # arrays/scalars compared after the run
    families: list = field(default_factory=list)
    entry: str = "main"
    backend: str = "cuda"
    program: str = ""      # runtime program name (default: the app name)

    @property
    def prog(self):
        return self.program or self.name


APPS = {
    "diffusion": App(
        "diffusion", [("ref", "diffusion/diffusion.h90")], "diff_state",
        {"t_old": ("nz", "nx", "ny"), "t_new": ("nz", "nx", "ny")},
        ["t_old", "t_new"]),
    "damping": App(
        "damping", [("ref", "damping/damping.h90")], "svar",
        {"dens_ref_f": ("nz_mn:nz_mx", "nx_mn:nx_mx", "ny_mn:ny_mx"),
         "dens_ptb_damp": ("nz_mn:nz_mx", "nx_mn:nx_mx", "ny_mn:ny_mx"),
         "dens_ptb_bnd": ("nz_mn:nz_mx", "nx_mn:nx_mx", "ny_mn:ny_mx", "2")},
        ["dens_ptb_damp", "dens_ref_f", "dens_ptb_bnd"],
        families=[("AT_TIGHT_STENCIL", "DOM_TIGHT_STENCIL"),
                  ("AT4_TIGHT_STENCIL", "DOM4_TIGHT_STENCIL")]),
    "bounded": App(
        "bounded", [("ref", "bounded/bounded.h90")], "b_state",
        {"a": ("nx", "ny"), "b": ("nx", "ny")}, ["a", "b"]),
    "surface_flux": App(
        "surface_flux",
        [("ref", "surface_flux/sf_state.h90"), ("ref", "surface_flux/surface_flux.h90"),
         ("ref", "surface_flux/driver.h90")], "sf_state",
        {"cover_frac": ("ntlm", "nx", "ny"), "wind_speed": ("nx", "ny"),
         "flx_sum_x": ("nx", "ny"), "flx_sum_y": ("nx", "ny")},
        ["cover_frac", "wind_speed", "flx_sum_x", "flx_sum_y"]),
    "reduction": App(
        "reduction", [("ref", "reduction/reduction.h90")], "red_state",
        {"y": ("nz", "nx", "ny")}, ["total", "y"], backend="acc"),
    "dycore": App(
        "dycore", [("own", "dycore/dyn_state.h90"), ("own", "dycore/dycore.h90")], "dyn_state",
        {n: ("nz", "nx", "ny") for n in ("rho", "th", "u", "v", "w", "p")},
        ["th", "u", "v", "w", "p", "rho"]),
    # the dynamics with Wicker-Skamarock RK3 (entry main_rk3)
    "dycore_rk3": App(
        "dycore_rk3", [("own", "dycore/dyn_state.h90"), ("own", "dycore/dycore.h90")],
        "dyn_state", {n: ("nz", "nx", "ny") for n in ("rho", "th", "u", "v", "w", "p")},
        ["th", "u", "v", "w", "p"], entry="main_rk3", program="dycore"),
    # the full timestep: dycore + column physics (entry main_full)
    "dycore_full": App(
        "dycore_full", [("own", "dycore/dyn_state.h90"), ("own", "dycore/dycore.h90")],
        "dyn_state",
        dict({n: ("nz", "nx", "ny") for n in ("rho", "th", "u", "v", "w", "p")},
             tsfc=("nx", "ny"), colm=("nx", "ny")),
        ["th", "u", "v", "w", "p", "colm"], entry="main_full", program="dycore"),
    # the ASUCA time scheme: RK3 long step, RK2 HE-VI acoustic short steps with damping,
    # limited advection of rho, theta and momentum (apps/dycore/asuca.h90, entry main_asuca)
    "asuca": App(
        "asuca", [("own", "dycore/dyn_state.h90"), ("own", "dycore/dycore.h90"),
                  ("own", "dycore/asuca.h90")],
        "dyn_state", {n: ("nz", "nx", "ny") for n in ("rho", "th", "u", "v", "w", "p")},
        ["rho", "th", "u", "v", "w", "p"], entry="main_asuca", program="dycore"),
    # feature coverage of the code generator (hfc); not a built-in program of the engine
    "kitchen": App(
        "kitchen", [("own", "kitchen/kit_state.h90"), ("own", "kitchen/kitchen.h90")],
        "kit_state",
        {"a": ("nz", "nx", "ny"), "b": ("nz", "nx", "ny"), "c": ("nx", "ny"),
         "halo": ("0:nz", "0:nx", "ny")},
        ["a", "b", "c", "halo", "alpha", "total_host"], program="kitchen_gen"),
}

# Synthetic-state conventions; seeds are fixed per field.
DYCORE_SCALARS = {"dt": 0.1, "rdx": 2.0, "rdy": 2.0, "rdz": 20.0, "cs2": 1.0,
                  "grav": 0.0327, "th0": 300.0}
DYCORE_FILLS = {  # name: (seed, offset, scale)
    "rho": (7, 1.0, 0.1), "th": (8, 300.0, 1.0), "u": (9, -0.01, 0.02),
    "v": (10, -0.01, 0.02), "w": (11, -0.002, 0.004), "p": (12, -0.005, 0.01)}
PHYS_SCALARS = {"ch": 0.05, "rrelax": 0.01}
PHYS_FILLS = {"tsfc": (13, 300.0, 2.0), "colm": (14, 300.0, 0.5)}
ASUCA_RDMP = 0.2  # maximum damping rate of the lateral band / upper sponge


def asuca_params(nz, nsound=6, nbnd=2, kdmp=None):
    """(ints, reals) of the ASUCA scheme: nsound short steps per long step, a lateral
    damping band of nbnd cells, the upper sponge above level kdmp (default: the top
    quarter of the column)."""
    kdmp = nz - max(1, nz // 4) if kdmp is None else kdmp
    return (dict(nsound=nsound, nbnd=nbnd, kdmp=kdmp),
            dict(rdmp=ASUCA_RDMP, rnbnd=1.0 / nbnd, rnzd=1.0 / (nz - kdmp)))


@dataclass
class Case:
    name: str
    app: str
    ints: dict
    reals: dict
    fills: dict            # name -> (seed, offset, scale)
    unset: list = field(default_factory=list)
    gpu_check: bool = True  # also run run_gpu_simulated and require equality
    order: str = "shuffled"


def _diff(name, nx, ny, nz, nsteps, seed=1, off=280.0, scale=10.0, coef=0.1):
    return Case(name, "diffusion", dict(nx=nx, ny=ny, nz=nz, nsteps=nsteps), dict(coef=coef),
                {"t_old": (seed, off, scale)}, unset=["t_new"])


def _dyc(name, nx, ny, nz, nsteps, gpu_check=True):
    return Case(name, "dycore", dict(nx=nx, ny=ny, nz=nz, nsteps=nsteps), dict(DYCORE_SCALARS),
                dict(DYCORE_FILLS), gpu_check=gpu_check)


def _full(name, nx, ny, nz, nsteps, gpu_check=True):
    return Case(name, "dycore_full", dict(nx=nx, ny=ny, nz=nz, nsteps=nsteps),
                dict(DYCORE_SCALARS, **PHYS_SCALARS), dict(DYCORE_FILLS, **PHYS_FILLS),
                gpu_check=gpu_check)


def _rk3(name, nx, ny, nz, nsteps, gpu_check=True):
    return Case(name, "dycore_rk3", dict(nx=nx, ny=ny, nz=nz, nsteps=nsteps),
                dict(DYCORE_SCALARS), dict(DYCORE_FILLS), gpu_check=gpu_check)


def _asu(name, nx, ny, nz, nsteps, gpu_check=True, **kw):
    ints, reals = asuca_params(nz, **kw)
    return Case(name, "asuca", dict(nx=nx, ny=ny, nz=nz, nsteps=nsteps, **ints),
                dict(DYCORE_SCALARS, **reals), dict(DYCORE_FILLS), gpu_check=gpu_check)


CASES = [
    # SURVEY §8(c) anchor: sum(t_old) after 10 steps == 2054.7107351501668
    _diff("diffusion_16x16x16_s10_anchor", 16, 16, 16, 10, seed=0, off=0.0, scale=1.0),
    _diff("diffusion_37x21x9_s3", 37, 21, 9, 3),
    _diff("diffusion_1x1x3_s2", 1, 1, 3, 2),
    _diff("diffusion_31x5x3_s2", 31, 5, 3, 2),
    _diff("diffusion_32x5x3_s2", 32, 5, 3, 2),
    _diff("diffusion_33x5x3_s2", 33, 5, 3, 2),
    _diff("diffusion_67x5x3_s2", 67, 5, 3, 2),
    _diff("diffusion_67x1x3_s2", 67, 1, 3, 2),
    _diff("diffusion_40x36x58_s1", 40, 36, 58, 1),
    Case("damping_37x21x9", "damping",
         dict(nx_mn=-1, nx_mx=35, ny_mn=0, ny_mx=20, nz_mn=1, nz_mx=9),
         dict(tratio_bnd=0.3, mtratio_bnd=0.7),
         {"dens_ref_f": (2, 1.0, 1.0), "dens_ptb_bnd": (3, -0.005, 0.01)}, unset=["dens_ptb_damp"]),
    Case("damping_1x1x1", "damping",
         dict(nx_mn=1, nx_mx=1, ny_mn=1, ny_mx=1, nz_mn=1, nz_mx=1),
         dict(tratio_bnd=0.3, mtratio_bnd=0.7),
         {"dens_ref_f": (2, 1.0, 1.0), "dens_ptb_bnd": (3, -0.005, 0.01)}, unset=["dens_ptb_damp"]),
    Case("damping_70x9x58_neg", "damping",
         dict(nx_mn=-3, nx_mx=66, ny_mn=-2, ny_mx=6, nz_mn=0, nz_mx=57),
         dict(tratio_bnd=0.3, mtratio_bnd=0.7),
         {"dens_ref_f": (2, 1.0, 1.0), "dens_ptb_bnd": (3, -0.005, 0.01)}, unset=["dens_ptb_damp"]),
    Case("bounded_37x21", "bounded", dict(nx=37, ny=21), {},
         {"a": (4, 0.0, 1.0), "b": (6, -1.0, 0.5)}),
    Case("bounded_3x3", "bounded", dict(nx=3, ny=3), {},
         {"a": (4, 0.0, 1.0), "b": (6, -1.0, 0.5)}),
    Case("bounded_67x34", "bounded", dict(nx=67, ny=34), {},
         {"a": (4, 0.0, 1.0), "b": (6, -1.0, 0.5)}),
    Case("surface_flux_37x21_t1", "surface_flux", dict(nx=37, ny=21, tile_land=1), {},
         {"cover_frac": (5, 0.0, 1.0)}, unset=["wind_speed", "flx_sum_x", "flx_sum_y"]),
    Case("surface_flux_33x7_t3", "surface_flux", dict(nx=33, ny=7, tile_land=3), {},
         {"cover_frac": (5, 0.0, 1.0)}, unset=["wind_speed", "flx_sum_x", "flx_sum_y"]),
    Case("reduction_37x21x9", "reduction", dict(nx=37, ny=21, nz=9), dict(total=0.0),
         {"y": (6, 0.0, 1.0)}),
    Case("reduction_67x5x58", "reduction", dict(nx=67, ny=5, nz=58), dict(total=0.0),
         {"y": (6, 0.0, 1.0)}),
    _dyc("dycore_13x7x10_s3", 13, 7, 10, 3),
    _dyc("dycore_24x20x12_s2", 24, 20, 12, 2),
    _dyc("dycore_1x5x2_s2", 1, 5, 2, 2),
    _dyc("dycore_33x3x58_s1", 33, 3, 58, 1),
    _dyc("dycore_13x7x10_s100", 13, 7, 10, 100, gpu_check=False),
    _full("full_13x7x10_s3", 13, 7, 10, 3),
    _full("full_24x20x12_s2", 24, 20, 12, 2),
    _full("full_1x5x2_s2", 1, 5, 2, 2),
    _full("full_33x3x58_s1", 33, 3, 58, 1),
    _rk3("rk3_13x7x10_s2", 13, 7, 10, 2),
    _rk3("rk3_24x20x12_s1", 24, 20, 12, 1),
    _rk3("rk3_1x5x2_s2", 1, 5, 2, 2),
    _rk3("rk3_33x3x58_s1", 33, 3, 58, 1),
    _asu("asuca_13x7x10_s2", 13, 7, 10, 2),
    _asu("asuca_24x20x12_s1", 24, 20, 12, 1, nbnd=3),
    _asu("asuca_1x5x3_s1", 1, 5, 3, 1, nsound=12, nbnd=1),
    _asu("asuca_33x3x58_s1", 33, 3, 58, 1, nbnd=4),
    _asu("asuca_13x7x10_s20", 13, 7, 10, 20, gpu_check=False),
]
CASE_BY_NAME = {c.name: c for c in CASES}


def _kit(name, nx, ny, nz, nsteps, shift):
    return Case(name, "kitchen", dict(nx=nx, ny=ny, nz=nz, nsteps=nsteps, shift=shift),
                dict(alpha=0.7, total_host=0.0),
                {"a": (21, -0.5, 1.0), "b": (22, 0.0, 2.0), "c": (23, 0.0, 1.0),
                 "halo": (24, 0.0, 1.0)})


# programs run only through generated code (hfc plugins); goldens by the reference itself
HFC_CASES = [
    _kit("kitchen_13x7x5_s2", 13, 7, 5, 2, 1),
    _kit("kitchen_37x21x9_s3", 37, 21, 9, 3, 4),
    _kit("kitchen_3x3x3_s1", 3, 3, 3, 1, 0),
    _kit("kitchen_33x4x12_s2", 33, 4, 12, 2, -2),
]
CASE_BY_NAME.update({c.name: c for c in HFC_CASES})
