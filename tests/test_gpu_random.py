"""Seeded random shapes and inputs (the reference's property-test style,
test_analysis.cpp:460-510 mt19937_64(2024)): every app through the C ABI equals the
oracle bit for bit, over sizes that cross tile edges, K phases and boundary cases."""
import numpy as np
import pytest

from cases import DYCORE_SCALARS, PHYS_SCALARS, Case
from golden_io import bits_equal, make_inputs, run_oracle
from test_gpu_parity import run_engine
from cases import APPS

pytestmark = pytest.mark.gpu
RNG = np.random.default_rng(2024)


def _draw(n):
    out = []
    for s in range(n):
        nx = int(RNG.integers(1, 100))
        ny = int(RNG.integers(1, 40))
        nz = int(RNG.integers(2, 66))
        steps = int(RNG.integers(1, 4))
        fills = {k: (int(RNG.integers(1, 1000)), float(RNG.uniform(-1, 1)),
                     float(RNG.uniform(0.001, 0.05))) for k in ("u", "v", "w", "p")}
        fills["rho"] = (int(RNG.integers(1, 1000)), 1.0, float(RNG.uniform(0.01, 0.2)))
        fills["th"] = (int(RNG.integers(1, 1000)), 300.0, float(RNG.uniform(0.1, 5.0)))
        out.append((nx, ny, nz, steps, fills))
    return out


@pytest.mark.parametrize("app", ["dycore", "dycore_rk3", "dycore_full"])
@pytest.mark.parametrize("draw", _draw(6), ids=lambda d: f"{d[0]}x{d[1]}x{d[2]}s{d[3]}")
def test_random_dycore_vs_oracle(app, draw):
    nx, ny, nz, steps, fills = draw
    reals = dict(DYCORE_SCALARS)
    f = dict(fills)
    if app == "dycore_full":
        reals.update(PHYS_SCALARS)
        f.update({"tsfc": (13, 300.0, 2.0), "colm": (14, 300.0, 0.5)})
    case = Case(f"r_{app}", app, dict(nx=nx, ny=ny, nz=nz, nsteps=steps), reals, f)
    a_gpu = make_inputs(case)
    a_ora = {k: v.copy() for k, v in a_gpu.items()}
    run_oracle(case, a_ora)
    run_engine(case, a_gpu)
    for k in APPS[app].outputs:
        assert bits_equal(a_gpu[k], a_ora[k]), k


@pytest.mark.parametrize("draw", _draw(6), ids=lambda d: f"{d[0]}x{d[1]}x{d[2]}s{d[3]}")
def test_random_diffusion_vs_oracle(draw):
    nx, ny, nz, steps, _ = draw
    case = Case("r_diff", "diffusion", dict(nx=nx, ny=ny, nz=nz, nsteps=steps), dict(coef=0.1),
                {"t_old": (int(RNG.integers(1, 99)), 280.0, 10.0)}, unset=["t_new"])
    a_gpu = make_inputs(case)
    a_ora = {k: v.copy() for k, v in a_gpu.items()}
    run_oracle(case, a_ora)
    run_engine(case, a_gpu)
    for k in ("t_old", "t_new"):
        assert bits_equal(a_gpu[k], a_ora[k]), k
