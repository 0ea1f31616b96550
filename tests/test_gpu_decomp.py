"""The 2-D horizontal decomposition on one GPU: every rank of a px x py
decomposition is its own context (tile-shaped state, global offsets), the ranks run in
lockstep in an in-process group and exchange their halo rings by device copies
(hfb_group_*). The assembled tiles must equal the undecomposed result BIT FOR BIT
(1e-12 for the reduction) — halo placement, global-index boundaries, face boxes and the
pack/unpack kernels are the same code the NCCL path uses."""
import numpy as np
import pytest

import paper_1710_08616_b200 as hfb
from cases import APPS, DYCORE_FILLS, DYCORE_SCALARS, PHYS_FILLS, PHYS_SCALARS, Case, _asu
from golden_io import bits_equal, decl, make_inputs, run_oracle

pytestmark = pytest.mark.gpu

# which declared dims are (i, j) for each array of an app
IJ_DIMS = {"diffusion": (1, 2), "dycore": (1, 2), "reduction": (1, 2), "bounded": (0, 1),
           "damping": (1, 2), "surface_flux": None, "dycore_full": (1, 2),
           "dycore_rk3": (1, 2), "asuca": (1, 2)}


def tile_slices(app, name, arr, d):
    if app == "surface_flux":
        ij = (1, 2) if name == "cover_frac" else (0, 1)
    elif arr.ndim == 2:
        ij = (0, 1)
    else:
        ij = IJ_DIMS[app]
    sl = [slice(None)] * arr.ndim
    sl[ij[0]] = slice(d.i0, d.i0 + d.nx)
    sl[ij[1]] = slice(d.j0, d.j0 + d.ny)
    return tuple(sl)


def tile_ints(case, d):
    i = dict(case.ints)
    if case.app == "damping":
        i["nx_mn"] = case.ints["nx_mn"] + d.i0
        i["nx_mx"] = i["nx_mn"] + d.nx - 1
        i["ny_mn"] = case.ints["ny_mn"] + d.j0
        i["ny_mx"] = i["ny_mn"] + d.ny - 1
    else:
        i["nx"], i["ny"] = int(d.nx), int(d.ny)
    return i


def global_extent(case):
    if case.app == "damping":
        return (case.ints["nx_mx"] - case.ints["nx_mn"] + 1,
                case.ints["ny_mx"] - case.ints["ny_mn"] + 1)
    return case.ints["nx"], case.ints["ny"]


def run_decomposed(case, px, py, entry=None, halo=2, ordered=False, options=None):
    entry = entry or APPS[case.app].entry
    garr = make_inputs(case)
    gnx, gny = global_extent(case)
    nz = case.ints.get("nz", 1)
    engines, tiles, decomps = [], [], []
    for r in range(px * py):
        d = hfb.decomp_init(gnx, gny, nz, px, py, r, halo=halo)
        eng = hfb.Engine(APPS[case.app].prog)
        eng.set_decomposition(d)
        for k, v in (options or {}).items():
            eng.set_option(k, v)
        if ordered:
            eng.set_reduction_order(True)
        ints = tile_ints(case, d)
        for k, v in ints.items():
            eng.set(k, int(v))
        for k, v in case.reals.items():
            eng.set(k, float(v))
        t = {}
        for name, a in garr.items():
            t[name] = np.ascontiguousarray(a[tile_slices(case.app, name, a, d)])
            _, lower = decl(case.app, name, ints)
            eng.bind(name, t[name], lower=lower)
        engines.append(eng)
        tiles.append(t)
        decomps.append(d)
    with hfb.Group(engines) as g:
        stats = g.run(entry)
    totals = [e.get("total") for e in engines] if case.app == "reduction" else None
    halo_bytes = sum(e.halo_bytes() for e in engines)
    out = {k: np.empty_like(v) for k, v in garr.items()}
    for t, d in zip(tiles, decomps):
        for name, a in t.items():
            out[name][tile_slices(case.app, name, out[name], d)] = a
    for e in engines:
        e.close()
    return garr, out, totals, stats, halo_bytes


def dyc(nx, ny, nz, nsteps):
    return Case(f"dycore_{nx}x{ny}x{nz}", "dycore", dict(nx=nx, ny=ny, nz=nz, nsteps=nsteps),
                dict(DYCORE_SCALARS), dict(DYCORE_FILLS))


@pytest.mark.parametrize("px,py", [(2, 1), (1, 2), (2, 2), (3, 2), (4, 2)])
def test_dycore_decomposed_equals_single(px, py):
    case = dyc(70, 45, 58, 3)
    garr, out, _, stats, halo_bytes = run_decomposed(case, px, py)
    ref = {k: v.copy() for k, v in garr.items()}
    run_oracle(case, ref)
    for k in ("th", "u", "v", "w", "p", "rho"):
        assert bits_equal(out[k], ref[k]), f"{px}x{py}: {k} differs"
    assert halo_bytes > 0
    # per rank and step: the interior launch while the halos travel + 4 boundary strips
    assert stats.native_launches == 3 * px * py * 5


def test_full_step_decomposed_equals_single():
    case = Case("f", "dycore_full", dict(nx=70, ny=45, nz=58, nsteps=3),
                dict(DYCORE_SCALARS, **PHYS_SCALARS), dict(DYCORE_FILLS, **PHYS_FILLS))
    garr, out, _, _, _ = run_decomposed(case, 2, 2)
    ref = {k: v.copy() for k, v in garr.items()}
    run_oracle(case, ref)
    for k in ("th", "u", "v", "w", "p", "colm"):
        assert bits_equal(out[k], ref[k]), k


def test_dycore_decomposed_ragged_tiles_generic_kernel():
    """Uneven tiles (remainders) and the portable kernel under decomposition."""
    case = dyc(37, 23, 80, 2)
    garr, out, _, _, _ = run_decomposed(case, 3, 3, options={"variant": "generic"})
    ref = {k: v.copy() for k, v in garr.items()}
    run_oracle(case, ref)
    for k in ("th", "u", "v", "w", "p"):
        assert bits_equal(out[k], ref[k]), k


@pytest.mark.parametrize("px,py", [(2, 2), (4, 1)])
def test_diffusion_decomposed_equals_single(px, py):
    case = Case("d", "diffusion", dict(nx=40, ny=36, nz=58, nsteps=3), dict(coef=0.1),
                {"t_old": (1, 280.0, 10.0)}, unset=["t_new"])
    garr, out, _, _, _ = run_decomposed(case, px, py, halo=1)
    ref = {k: v.copy() for k, v in garr.items()}
    run_oracle(case, ref)
    for k in ("t_old", "t_new"):
        assert bits_equal(out[k], ref[k]), k


def test_bounded_decomposed_equals_single():
    case = Case("b", "bounded", dict(nx=37, ny=21), {}, {"a": (4, 0.0, 1.0), "b": (6, -1.0, 0.5)})
    garr, out, _, _, _ = run_decomposed(case, 2, 3, halo=1)
    ref = {k: v.copy() for k, v in garr.items()}
    run_oracle(case, ref)
    assert bits_equal(out["b"], ref["b"]) and bits_equal(out["a"], ref["a"])


def test_damping_decomposed_equals_single():
    case = Case("dm", "damping", dict(nx_mn=-1, nx_mx=35, ny_mn=0, ny_mx=20, nz_mn=1, nz_mx=9),
                dict(tratio_bnd=0.3, mtratio_bnd=0.7),
                {"dens_ref_f": (2, 1.0, 1.0), "dens_ptb_bnd": (3, -0.005, 0.01)})
    garr, out, _, _, _ = run_decomposed(case, 2, 2, halo=0)
    ref = {k: v.copy() for k, v in garr.items()}
    run_oracle(case, ref)
    assert bits_equal(out["dens_ptb_damp"], ref["dens_ptb_damp"])


def test_reduction_decomposed_allreduce():
    case = Case("r", "reduction", dict(nx=67, ny=45, nz=58), dict(total=0.0), {"y": (6, 0.0, 1.0)})
    garr, out, totals, _, _ = run_decomposed(case, 2, 2, halo=0)
    ref = run_oracle(case, {k: v.copy() for k, v in garr.items()})["total"]
    assert len(set(totals)) == 1
    assert abs(totals[0] - ref) <= 1e-12 * abs(ref)


@pytest.mark.parametrize("px,py", [(2, 2), (3, 1), (1, 4)])
def test_reduction_decomposed_ordered_bit_exact(px, py):
    """Ordered reductions in a group: the tiles' column partials are assembled in global
    (j, i) order, so the total is bit-identical to the single-domain acc-simulated order."""
    case = Case("r", "reduction", dict(nx=67, ny=45, nz=58), dict(total=0.0), {"y": (6, 0.0, 1.0)})
    garr, out, totals, _, _ = run_decomposed(case, px, py, halo=0, ordered=True)
    accsim = run_oracle(case, {k: v.copy() for k, v in garr.items()})["total_accsim"]
    assert len(set(totals)) == 1
    assert np.float64(totals[0]).view(np.uint64) == np.float64(accsim).view(np.uint64)


@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("app", ["dycore", "dycore_full", "diffusion"])
def test_overlapped_exchange_equals_serial(app, overlap):
    """Decomposed stencil steps run the interior columns while the halos travel, then the
    boundary strips (option overlap=0: exchange first, one full launch). Both are
    bit-identical to the undecomposed oracle."""
    if app == "diffusion":
        case = Case("d", "diffusion", dict(nx=70, ny=45, nz=20, nsteps=3), dict(coef=0.1),
                    {"t_old": (1, 280.0, 10.0)}, unset=["t_new"])
        names = ("t_old", "t_new")
    else:
        reals = dict(DYCORE_SCALARS, **PHYS_SCALARS) if app == "dycore_full" else dict(DYCORE_SCALARS)
        fills = dict(DYCORE_FILLS, **PHYS_FILLS) if app == "dycore_full" else dict(DYCORE_FILLS)
        case = Case("x", app, dict(nx=70, ny=45, nz=20, nsteps=2), reals, fills)
        names = APPS[app].outputs
    garr, out, _, stats, _ = run_decomposed(case, 2, 2, options={"overlap": int(overlap)})
    ref = {k: v.copy() for k, v in garr.items()}
    run_oracle(case, ref)
    for k in names:
        assert bits_equal(out[k], ref[k]), k
    steps = case.ints["nsteps"]
    assert stats.native_launches == 4 * steps * (5 if overlap else 1)


@pytest.mark.parametrize("app", ["dycore_full", "diffusion"])
def test_overlapped_exchange_whole_tile_strips(app):
    """Tiles wide and tall enough for whole-tile boundary strips (32 columns, 4 rows): the
    interior is whole tiles too, and the split is still bit-identical to the oracle."""
    if app == "diffusion":
        case = Case("d", "diffusion", dict(nx=150, ny=30, nz=12, nsteps=3), dict(coef=0.1),
                    {"t_old": (1, 280.0, 10.0)}, unset=["t_new"])
        names = ("t_old", "t_new")
    else:
        case = Case("x", app, dict(nx=150, ny=30, nz=20, nsteps=2),
                    dict(DYCORE_SCALARS, **PHYS_SCALARS), dict(DYCORE_FILLS, **PHYS_FILLS))
        names = APPS[app].outputs
    garr, out, _, stats, _ = run_decomposed(case, 2, 2, options={"overlap": 1})
    ref = {k: v.copy() for k, v in garr.items()}
    run_oracle(case, ref)
    for k in names:
        assert bits_equal(out[k], ref[k]), k
    assert stats.native_launches == 4 * case.ints["nsteps"] * 5


def test_group_refuses_the_asuca_scheme():
    """The ASUCA scheme's exchanges include scratch arrays that in-process groups cannot
    pull by name: a decomposed asuca_step in a group fails with HFB_CONFIG (the peer and
    NCCL transports run it, tests/test_gpu_peer.py) instead of computing without halos."""
    case = _asu("g_asuca", 40, 30, 10, 1, nbnd=2)
    with pytest.raises(hfb.HfbError, match="peer or NCCL"):
        run_decomposed(case, 2, 1)
