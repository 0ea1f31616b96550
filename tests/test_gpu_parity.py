"""Parity of the B200 path (libhfb.so through the C ABI) with the reference.

* every golden case (fixtures produced by the reference interpreter itself): bit-exact
  outputs, and LaunchStats equal to the reference's simulated launches;
* larger seeded inputs against the CPU restatement (oracle/), bit-exact;
* full-size (BASELINE configs) single steps against the oracle, bit-exact;
* the drop-in surface: per-step entries, residency errors, the generated-kernel ABI,
  graph replay.
"""
import numpy as np
import pytest

import paper_1710_08616_b200 as hfb
from cases import (APPS, CASES, CASE_BY_NAME, DYCORE_FILLS, DYCORE_SCALARS, PHYS_FILLS,
                   PHYS_SCALARS, Case, _asu)
from golden_io import bits_equal, decl, load_golden, make_inputs, run_oracle

pytestmark = pytest.mark.gpu


def run_engine(case, arrs, entry=None, options=None):
    app = APPS[case.app]
    entry = entry or app.entry
    with hfb.Engine(app.prog) as eng:
        for k, v in (options or {}).items():
            eng.set_option(k, v)
        for k, v in case.ints.items():
            eng.set(k, int(v))
        for k, v in case.reals.items():
            eng.set(k, float(v))
        for name, a in arrs.items():
            _, lower = decl(case.app, name, case.ints)
            eng.bind(name, a, lower=lower)
        stats = eng.run(entry)
        scal = {}
        if case.app == "reduction":
            scal["total"] = eng.get("total")
    return stats, scal


@pytest.mark.parametrize("case", CASES, ids=lambda c: c.name)
@pytest.mark.parametrize("order", ["C", "F"])
def test_golden_case(case, order):
    meta, out, init, extra = load_golden(case.name)
    arrs = make_inputs(case, order=order)
    stats, scal = run_engine(case, arrs)
    for name in APPS[case.app].outputs:
        if name == "total":
            ref = float(out["total"].reshape(()))
            assert abs(scal["total"] - ref) <= 1e-12 * abs(ref), (scal["total"], ref)
        else:
            assert bits_equal(arrs[name], out[name]), f"{case.name}: {name} differs"
    if "gpu_launches" in meta and case.app != "reduction":
        assert stats.launches == meta["gpu_launches"]
        assert stats.threads == meta["gpu_threads"]
        assert stats.guard_returns == meta["gpu_guard_returns"]
    assert stats.native_launches > 0


def _oracle_vs_gpu(case, order="C", options=None):
    a_gpu = make_inputs(case, order=order)
    a_ora = {k: v.copy(order="A") for k, v in a_gpu.items()}
    run_oracle(case, a_ora)
    run_engine(case, a_gpu, options=options)
    for name in APPS[case.app].outputs:
        if name in a_gpu:
            assert bits_equal(a_gpu[name], a_ora[name]), f"{case.name}: {name} differs"


LARGE = [
    Case("diffusion_128x128x58_s10", "diffusion", dict(nx=128, ny=128, nz=58, nsteps=10),
         dict(coef=0.1), {"t_old": (1, 280.0, 10.0)}, unset=["t_new"]),
    Case("diffusion_333x77x58_s3", "diffusion", dict(nx=333, ny=77, nz=58, nsteps=3),
         dict(coef=0.1), {"t_old": (1, 280.0, 10.0)}, unset=["t_new"]),
    Case("damping_260x131x58", "damping",
         dict(nx_mn=-1, nx_mx=258, ny_mn=0, ny_mx=130, nz_mn=1, nz_mx=58),
         dict(tratio_bnd=0.3, mtratio_bnd=0.7),
         {"dens_ref_f": (2, 1.0, 1.0), "dens_ptb_bnd": (3, -0.005, 0.01)}),
    Case("bounded_1024x515", "bounded", dict(nx=1024, ny=515), {},
         {"a": (4, 0.0, 1.0), "b": (6, -1.0, 0.5)}),
    Case("surface_flux_1024x1024", "surface_flux", dict(nx=1024, ny=1024, tile_land=2), {},
         {"cover_frac": (5, 0.0, 1.0)}),
    Case("dycore_128x96x58_s5", "dycore", dict(nx=128, ny=96, nz=58, nsteps=5),
         dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
    Case("dycore_77x203x31_s3", "dycore", dict(nx=77, ny=203, nz=31, nsteps=3),
         dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
    # nz - 1 > 64: 512 TMEM columns per CTA (one CTA per SM) up to nz = 129; beyond that
    # the generic (L2 round-trip) kernels
    Case("dycore_40x30x80_s2", "dycore", dict(nx=40, ny=30, nz=80, nsteps=2),
         dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
    Case("dycore_37x21x129_s2", "dycore", dict(nx=37, ny=21, nz=129, nsteps=2),
         dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
    Case("dycore_35x9x140_s1", "dycore", dict(nx=35, ny=9, nz=140, nsteps=1),
         dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
    Case("rk3_40x30x100_s2", "dycore_rk3", dict(nx=40, ny=30, nz=100, nsteps=2),
         dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
    Case("dycore_33x9x65_s2", "dycore", dict(nx=33, ny=9, nz=65, nsteps=2),
         dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
    Case("dycore_31x7x2_s3", "dycore", dict(nx=31, ny=7, nz=2, nsteps=3),
         dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
    Case("rk3_128x96x58_s2", "dycore_rk3", dict(nx=128, ny=96, nz=58, nsteps=2),
         dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
    Case("rk3_77x41x31_s3", "dycore_rk3", dict(nx=77, ny=41, nz=31, nsteps=3),
         dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
    Case("full_128x96x58_s3", "dycore_full", dict(nx=128, ny=96, nz=58, nsteps=3),
         dict(DYCORE_SCALARS, **PHYS_SCALARS), dict(DYCORE_FILLS, **PHYS_FILLS)),
    Case("full_45x37x80_s2", "dycore_full", dict(nx=45, ny=37, nz=80, nsteps=2),
         dict(DYCORE_SCALARS, **PHYS_SCALARS), dict(DYCORE_FILLS, **PHYS_FILLS)),
    _asu("asuca_128x96x58_s1", 128, 96, 58, 1, nbnd=6),
    _asu("asuca_77x41x31_s2", 77, 41, 31, 2, nsound=12, nbnd=3),
    _asu("asuca_40x36x2_s2", 40, 36, 2, 2, kdmp=1),
    _asu("asuca_33x9x65_s1", 33, 9, 65, 1, nsound=6, nbnd=4),
    _asu("asuca_33x21x100_s1", 33, 21, 100, 1, nsound=6, nbnd=4),
    # the tendency pass tiles x by 31 columns (+ a ghost lane): exact multiples, one past,
    # and interior tiles of both box parities
    _asu("asuca_93x11x12_s1", 93, 11, 12, 1, nbnd=3),
    _asu("asuca_94x13x12_s1", 94, 13, 12, 1, nbnd=3),
    _asu("asuca_190x14x9_s1", 190, 14, 9, 1, nbnd=2),
]


@pytest.mark.parametrize("case", LARGE, ids=lambda c: c.name)
def test_large_vs_oracle(case):
    _oracle_vs_gpu(case)


@pytest.mark.parametrize("name", ["reduction_37x21x9", "reduction_67x5x58"])
def test_reduction_ordered_matches_reference_accsim(name):
    """hfb_set_reduction_order(1): bit-identical to the REFERENCE's run_gpu_simulated total
    on the OpenACC backend (golden out_accsim.total), not just within 1e-12."""
    case = CASE_BY_NAME[name]
    _, out, _, extra = load_golden(name)
    arrs = make_inputs(case)
    app = APPS[case.app]
    with hfb.Engine(app.prog) as eng:
        eng.set_reduction_order(True)
        for k, v in case.ints.items():
            eng.set(k, int(v))
        for k, v in case.reals.items():
            eng.set(k, float(v))
        eng.bind("y", arrs["y"])
        eng.run("main")
        total = eng.get("total")
    ref = float(extra["out_accsim.total"].reshape(()))
    assert np.float64(total).view(np.uint64) == np.float64(ref).view(np.uint64), (total, ref)


def test_reduction_ordered_full_size():
    """512 x 512 x 58 ordered total == the oracle's acc-simulated order, bit for bit."""
    case = Case("reduction_512x512x58", "reduction", dict(nx=512, ny=512, nz=58),
                dict(total=0.0), {"y": (6, 0.0, 1.0)})
    arrs = make_inputs(case)
    ref = run_oracle(case, {k: v.copy() for k, v in arrs.items()})["total_accsim"]
    with hfb.Engine("reduction") as eng:
        eng.set_reduction_order(True)
        for k, v in case.ints.items():
            eng.set(k, int(v))
        eng.set("total", 0.0)
        eng.bind("y", arrs["y"])
        eng.run("main")
        total = eng.get("total")
    assert np.float64(total).view(np.uint64) == np.float64(ref).view(np.uint64)


def test_reduction_large_tolerance():
    case = Case("reduction_512x512x58", "reduction", dict(nx=512, ny=512, nz=58),
                dict(total=0.0), {"y": (6, 0.0, 1.0)})
    arrs = make_inputs(case)
    ref = run_oracle(case, {k: v.copy() for k, v in arrs.items()})
    _, scal = run_engine(case, arrs)
    assert abs(scal["total"] - ref["total"]) <= 1e-12 * abs(ref["total"])


def test_split_step_matches():
    """The two-kernel step (advect + TMEM acoustic; variant split) gives the same bits."""
    _oracle_vs_gpu(Case("dycore_70x45x58_s2", "dycore", dict(nx=70, ny=45, nz=58, nsteps=2),
                        dict(DYCORE_SCALARS), dict(DYCORE_FILLS)), options={"variant": "split"})


def test_full_step_split_path_matches():
    """dycore kernels + the standalone column-physics kernel (variant split)."""
    _oracle_vs_gpu(Case("full_70x45x58_s2", "dycore_full", dict(nx=70, ny=45, nz=58, nsteps=2),
                        dict(DYCORE_SCALARS, **PHYS_SCALARS), dict(DYCORE_FILLS, **PHYS_FILLS)),
                   options={"variant": "split"})


def test_full_size_full_timestep_c3():
    """BASELINE configs[2]: full timestep with column physics, 1024 x 1024 x 58, one step."""
    _oracle_vs_gpu(Case("full_1024x1024x58_s1", "dycore_full",
                        dict(nx=1024, ny=1024, nz=58, nsteps=1),
                        dict(DYCORE_SCALARS, **PHYS_SCALARS), dict(DYCORE_FILLS, **PHYS_FILLS)))


def test_single_role_fused_matches():
    """The single-role fused kernel (variant single_role) gives the same bits."""
    _oracle_vs_gpu(Case("dycore_70x45x58_s2", "dycore", dict(nx=70, ny=45, nz=58, nsteps=2),
                        dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
                   options={"variant": "single_role"})


def test_ab_variants_not_in_product_library():
    """The measured-slower variants (tma, ws2) and the timing switches are compiled only
    into the A/B build; the product library refuses them (no hidden knobs)."""
    if hfb.variants_build():
        pytest.skip("running against the A/B build")
    with hfb.Engine("dycore") as eng:
        for k, v in (("variant", "tma"), ("variant", "ws2"), ("debug_skip", "1"),
                     ("variant", "nonsense"), ("no_such_option", "1")):
            with pytest.raises(hfb.HfbError) as e:
                eng.set_option(k, v)
            assert e.value.kind == "config"


@pytest.mark.parametrize("app", ["dycore", "dycore_full", "dycore_rk3"])
@pytest.mark.parametrize("variant", ["tma", "ws2"])
def test_step_variant_matches(app, variant):
    """The measured alternatives of the fused step give the same bits: the TMA-fed twin
    (tma) and the two-columns-per-thread kernel (ws2). They live in the A/B build
    (libhfb_variants.so), run here in a child process that loads it."""
    import subprocess
    import sys
    from pathlib import Path
    lib = hfb.runtime.VARIANTS_LIB
    if not lib.exists():
        pytest.skip("A/B build not present (make -C paper_1710_08616_b200/csrc variants)")
    here = Path(__file__).resolve().parent
    code = ("import sys; sys.path[:0] = [%r, %r, %r]\n"
            "import paper_1710_08616_b200 as hfb; assert hfb.variants_build()\n"
            "from test_gpu_parity import _variant_case, _oracle_vs_gpu\n"
            "_oracle_vs_gpu(_variant_case(%r), options={'variant': %r})\n"
            % (str(here.parent), str(here), str(here.parent / "oracle"), app, variant))
    r = subprocess.run([sys.executable, "-c", code], env=dict(__import__("os").environ,
                       HFB_LIB=str(lib)), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]


def _variant_case(app):
    reals = dict(DYCORE_SCALARS, **PHYS_SCALARS) if app == "dycore_full" else dict(DYCORE_SCALARS)
    fills = dict(DYCORE_FILLS, **PHYS_FILLS) if app == "dycore_full" else dict(DYCORE_FILLS)
    return Case(f"{app}_70x45x58_s2", app, dict(nx=70, ny=45, nz=58, nsteps=2), reals, fills)


@pytest.mark.parametrize("app", ["dycore", "dycore_rk3"])
@pytest.mark.parametrize("edge", ["th_eq_th0", "zero_w_p", "tiny"])
def test_division_fast_path_edges(app, edge):
    """HE-VI quotients share reciprocals (hfb_fp64.cuh) behind a range check; inputs that
    fail it (zero numerators: theta == th0 makes dt*grav*(theta-th0) exactly 0, a resting
    state makes the pressure-difference numerator 0; tiny magnitudes) take the dialect's
    divisions. Bit-exact either way."""
    fills = dict(DYCORE_FILLS)
    reals = dict(DYCORE_SCALARS)
    if edge == "th_eq_th0":
        fills["th"] = (8, 300.0, 0.0)
    elif edge == "zero_w_p":
        for k in ("u", "v", "w", "p"):
            fills[k] = (fills[k][0], 0.0, 0.0)
    else:  # tiny pressure perturbations at rest: tiny and subnormal quotients
        for k in ("u", "v", "w"):
            fills[k] = (fills[k][0], 0.0, 0.0)
        fills["p"] = (12, 0.0, 1e-300)
    _oracle_vs_gpu(Case(f"{app}_{edge}_40x36x20_s2", app, dict(nx=40, ny=36, nz=20, nsteps=2),
                        reals, fills))


def test_generic_diffusion_kernel_matches():
    """The L1-cached diffusion kernel (variant generic; the product kernel stages planes
    in shared memory, hfb_diffusion.cu) gives the same bits."""
    _oracle_vs_gpu(Case("diffusion_333x77x58_s3", "diffusion", dict(nx=333, ny=77, nz=58, nsteps=3),
                        dict(coef=0.1), {"t_old": (1, 280.0, 10.0)}, unset=["t_new"]),
                   options={"variant": "generic"})


def test_generic_kernels_match():
    """The portable acoustic kernel (variant generic) gives the same bits."""
    _oracle_vs_gpu(Case("dycore_70x45x58_s2", "dycore", dict(nx=70, ny=45, nz=58, nsteps=2),
                        dict(DYCORE_SCALARS), dict(DYCORE_FILLS)), options={"variant": "generic"})


@pytest.mark.parametrize("nx,ny", [(512, 512), (1581, 1301)])
def test_full_size_dycore_step(nx, ny):
    """BASELINE configs C2 / C4: one dycore step, bit-exact against the oracle."""
    case = Case(f"dycore_{nx}x{ny}x58_s1", "dycore", dict(nx=nx, ny=ny, nz=58, nsteps=1),
                dict(DYCORE_SCALARS), dict(DYCORE_FILLS))
    _oracle_vs_gpu(case)


def test_north_star_full_timestep_c4():
    """north_star: one full timestep (dycore + HE-VI + column physics, `full_step`) on the
    1581 x 1301 x 58 production grid — the bench's headline workload — bit-exact against
    the oracle in every prognostic field and the column means."""
    _oracle_vs_gpu(Case("full_1581x1301x58_s1", "dycore_full",
                        dict(nx=1581, ny=1301, nz=58, nsteps=1),
                        dict(DYCORE_SCALARS, **PHYS_SCALARS), dict(DYCORE_FILLS, **PHYS_FILLS)))


def test_asuca_step_c3():
    """The ASUCA time scheme (RK3 long step; 11 RK2 HE-VI acoustic short steps with
    lateral/upper damping; limited advection of rho, theta, u, v, w) on the BASELINE
    configs[2] grid, 1024 x 1024 x 58, one step, bit-exact against the oracle."""
    _oracle_vs_gpu(_asu("asuca_1024x1024x58_s1", 1024, 1024, 58, 1, nbnd=8))


def test_asuca_per_step_entry_and_graph_replay():
    """asuca_step as a per-step entry (device resident, enqueued) and replayed from a CUDA
    graph equals main_asuca (copy-in, nsteps, copy-out)."""
    case = _asu("asuca_70x45x20_s4", 70, 45, 20, 4, nbnd=3)
    ref = make_inputs(case)
    run_engine(case, ref)
    for mode in ("enqueue", "graph"):
        arrs = make_inputs(case)
        with hfb.Engine("dycore") as eng:
            for k, v in case.ints.items():
                eng.set(k, int(v))
            for k, v in case.reals.items():
                eng.set(k, float(v))
            for n, a in arrs.items():
                eng.bind(n, a)
                eng.copy_to_device(n)
            if mode == "enqueue":
                for _ in range(case.ints["nsteps"]):
                    eng.enqueue("asuca_step")
                eng.synchronize()
            else:
                eng.run_graph("asuca_step", 2)
                eng.run_graph("asuca_step", 2)
            for n in arrs:
                eng.copy_from_device(n)
        for n in ("rho", "th", "u", "v", "w", "p"):
            assert bits_equal(arrs[n], ref[n]), f"{mode}: {n} differs"


def test_full_size_rk3_step_c2():
    """BASELINE configs[1] grid with the Wicker-Skamarock RK3 long step (three fused
    stages), one step, bit-exact against the oracle."""
    _oracle_vs_gpu(Case("rk3_512x512x58_s1", "dycore_rk3", dict(nx=512, ny=512, nz=58, nsteps=1),
                        dict(DYCORE_SCALARS), dict(DYCORE_FILLS)))


def test_c2_dycore_100_steps():
    """BASELINE configs[1] as stated: dycore + HE-VI, 512 x 512 x 58 for 100 steps (one
    `main` call: copy-in, 100 fused steps, copy-out), bit-exact against the oracle after
    all 100 steps — no drift envelope is needed because every step is bit-identical."""
    _oracle_vs_gpu(Case("dycore_512x512x58_s100", "dycore", dict(nx=512, ny=512, nz=58, nsteps=100),
                        dict(DYCORE_SCALARS), dict(DYCORE_FILLS)))


def test_full_size_diffusion_step():
    case = Case("diffusion_1581x1301x58_s1", "diffusion", dict(nx=1581, ny=1301, nz=58, nsteps=1),
                dict(coef=0.1), {"t_old": (1, 280.0, 10.0)}, unset=["t_new"])
    _oracle_vs_gpu(case)


# ---------------------------------------------------------------------------
# drop-in surface: per-step entries, residency, generated-kernel ABI, graphs
# ---------------------------------------------------------------------------

def _diffusion_engine(nx=40, ny=36, nz=58, nsteps=3):
    case = Case("d", "diffusion", dict(nx=nx, ny=ny, nz=nz, nsteps=nsteps), dict(coef=0.1),
                {"t_old": (1, 280.0, 10.0)}, unset=["t_new"])
    arrs = make_inputs(case)
    eng = hfb.Engine("diffusion")
    for k, v in case.ints.items():
        eng.set(k, v)
    eng.set("coef", 0.1)
    for k, a in arrs.items():
        eng.bind(k, a)
    return case, arrs, eng


def test_missing_transfer_is_a_residency_error():
    # deleting transferHere -> "[residency] array 't_old' has no device copy"
    case, arrs, eng = _diffusion_engine()
    with pytest.raises(hfb.HfbError) as e:
        eng.run("hfd_diffuse_step")
    assert e.value.kind == "residency" and "t_old" in str(e.value)
    with pytest.raises(hfb.HfbError) as e:
        eng.copy_from_device("t_old")
    assert e.value.kind == "residency" and "never transferred" in str(e.value)
    eng.close()


def test_per_step_entry_matches_simulation_run():
    case, arrs, eng = _diffusion_engine(nsteps=3)
    ref = {k: v.copy() for k, v in arrs.items()}
    run_oracle(case, ref)
    eng.copy_to_device("t_old")
    eng.copy_to_device("t_new")
    for _ in range(3):
        st = eng.run("diffuse_step")
        assert st.launches == 2
    assert eng.residency("t_old") == ("device", True)
    with pytest.raises(hfb.HfbError) as e:  # device data is newer
        eng.copy_to_device("t_old")
    assert e.value.kind == "residency"
    eng.copy_from_device("t_old")
    eng.copy_from_device("t_new")
    assert bits_equal(arrs["t_old"], ref["t_old"]) and bits_equal(arrs["t_new"], ref["t_new"])
    eng.mark_host_modified("t_old")
    with pytest.raises(hfb.HfbError) as e:  # stale device copy
        eng.run("diffuse_step")
    assert e.value.kind == "residency"
    eng.close()


def test_graph_replay_matches_step_loop():
    case = Case("g", "dycore", dict(nx=96, ny=64, nz=58, nsteps=6), dict(DYCORE_SCALARS),
                dict(DYCORE_FILLS))
    arrs = make_inputs(case)
    ref = {k: v.copy() for k, v in arrs.items()}
    run_oracle(case, ref)
    with hfb.Engine("dycore") as eng:
        for k, v in case.ints.items():
            eng.set(k, v)
        for k, v in case.reals.items():
            eng.set(k, v)
        for k, a in arrs.items():
            eng.bind(k, a)
        for k in arrs:
            eng.copy_to_device(k)
        st = eng.run_graph("dycore_step", 2)
        assert st.native_launches == 2  # one fused kernel per timestep
        eng.run_graph("dycore_step", 2)
        eng.run_graph("dycore_step", 2)
        for k in arrs:
            eng.copy_from_device(k)
    for k in ("th", "u", "v", "w", "p"):
        assert bits_equal(arrs[k], ref[k]), k


def test_rk3_graph_replay_and_mixed_steps():
    """RK3 steps (3 buffers per field) in a CUDA graph, mixed with single-stage steps."""
    case = Case("g", "dycore", dict(nx=96, ny=64, nz=58, nsteps=1), dict(DYCORE_SCALARS),
                dict(DYCORE_FILLS))
    arrs = make_inputs(case)
    import oracle
    ref = {k: v.copy() for k, v in arrs.items()}
    oracle.rk3_run(2, DYCORE_SCALARS, *(ref[k] for k in ("rho", "th", "u", "v", "w", "p")))
    oracle.dycore_run(1, DYCORE_SCALARS, *(ref[k] for k in ("rho", "th", "u", "v", "w", "p")))
    oracle.rk3_run(3, DYCORE_SCALARS, *(ref[k] for k in ("rho", "th", "u", "v", "w", "p")))
    with hfb.Engine("dycore") as eng:
        for k, v in case.ints.items():
            eng.set(k, v)
        for k, v in case.reals.items():
            eng.set(k, v)
        for k, a in arrs.items():
            eng.bind(k, a)
            eng.copy_to_device(k)
        st = eng.run_graph("rk3_step", 2)
        assert st.launches == 50 and st.native_launches == 6
        eng.run("dycore_step")
        eng.run_graph("rk3_step", 3)
        for k in arrs:
            eng.copy_from_device(k)
    for k in ("th", "u", "v", "w", "p"):
        assert bits_equal(arrs[k], ref[k]), k


def test_errors_mirror_reference_kinds():
    with pytest.raises(hfb.HfbError) as e:
        hfb.Engine("no_such_app")
    assert e.value.kind == "config"
    case, arrs, eng = _diffusion_engine()
    with pytest.raises(hfb.HfbError) as e:
        eng.run("no_such_entry")
    assert e.value.kind == "config"
    eng.set("nx", 41)  # bound buffers no longer match the declaration
    with pytest.raises(hfb.HfbError) as e:
        eng.run("main")
    assert e.value.kind == "runtime"
    eng.close()
    # bounded with nx = 2: ceiling(0/32) = 0 blocks -> the reference rejects the launch
    with hfb.Engine("bounded") as eng:
        eng.set("nx", 2)
        eng.set("ny", 5)
        a = np.ones((2, 5))
        b = np.zeros((2, 5))
        eng.bind("a", a)
        eng.bind("b", b)
        with pytest.raises(hfb.HfbError) as e:
            eng.run("main")
        assert e.value.kind == "runtime"


def test_pinned_binding_and_fortran_order_equal():
    case = CASE_BY_NAME["dycore_24x20x12_s2"]
    meta, out, init, extra = load_golden(case.name)
    arrs = make_inputs(case, order="F")
    with hfb.Engine("dycore") as eng:
        for k, v in case.ints.items():
            eng.set(k, v)
        for k, v in case.reals.items():
            eng.set(k, v)
        for k, a in arrs.items():
            eng.bind(k, a, pin=True)
        eng.run("main")
    for k in ("th", "u", "v", "w", "p"):
        assert bits_equal(arrs[k], out[k])


@pytest.mark.parametrize("app", ["diffusion", "dycore", "damping"])
def test_layout_invariance_all_host_orders(app):
    """SPEC.md:549 "identical results under any configured storage-order permutation":
    the same logical arrays bound in every dim permutation of host memory order give
    bit-identical results (the device layout is fixed; only the relayout changes)."""
    import itertools
    case = {"diffusion": CASE_BY_NAME["diffusion_37x21x9_s3"],
            "dycore": CASE_BY_NAME["dycore_24x20x12_s2"],
            "damping": CASE_BY_NAME["damping_37x21x9"]}[app]
    base = make_inputs(case)
    results = []
    for perm in itertools.permutations(range(3)):
        arrs = {}
        for k, a in base.items():
            p = perm + tuple(range(3, a.ndim))
            inv = tuple(np.argsort(p))
            # a fresh copy in permuted memory order (ascontiguousarray would alias `base`
            # for the identity permutation and let the run overwrite the inputs)
            arrs[k] = np.array(a.transpose(p), order="C", copy=True).transpose(inv)
        run_engine(case, arrs)
        results.append({k: np.ascontiguousarray(v) for k, v in arrs.items()})
    for r in results[1:]:
        for k in results[0]:
            assert bits_equal(r[k], results[0][k]), k
    _, out, _, _ = load_golden(case.name)
    for k in APPS[case.app].outputs:
        assert bits_equal(results[0][k], out[k]), k


def test_transfer_state_machine_matches_reference():
    """hfrt_device_allocate / copy_to_device / copy_from_device against the reference's
    exec_transfer (interp.cpp:1369-1415): error kinds and texts, residency after each."""
    case, arrs, eng = _diffusion_engine(nsteps=1)
    with pytest.raises(hfb.HfbError) as e:
        eng.copy_from_device("t_new")
    assert e.value.kind == "residency" and "never transferred to the device" in str(e.value)
    eng.device_allocate("t_new")  # a device copy; residency unchanged (still host)
    assert eng.residency("t_new") == ("host", True)
    eng.device_allocate("t_new")  # idempotent
    with pytest.raises(hfb.HfbError) as e:
        eng.copy_from_device("t_new")
    assert e.value.kind == "residency" and "would overwrite newer host data" in str(e.value)
    eng.copy_to_device("t_old")
    assert eng.residency("t_old") == ("both", True)
    eng.run("diffuse_step")  # writes both on the device
    assert eng.residency("t_new") == ("device", True)
    with pytest.raises(hfb.HfbError) as e:
        eng.copy_to_device("t_new")
    assert e.value.kind == "residency" and "would overwrite newer device data" in str(e.value)
    eng.copy_from_device("t_new")
    assert eng.residency("t_new") == ("both", True)
    eng.copy_to_device("t_new")  # both -> both: allowed
    eng.close()


def test_entry_copy_out_skips_untouched_arrays():
    """`main` copies the six dycore fields in and, at the end, out — except rho, which no
    step writes: residency is still Both, the host already holds the device's bytes, so
    no D2H happens (and the result is unchanged)."""
    case = Case("x", "dycore", dict(nx=40, ny=24, nz=12, nsteps=2), dict(DYCORE_SCALARS),
                dict(DYCORE_FILLS))
    arrs = make_inputs(case)
    ref = {k: v.copy() for k, v in arrs.items()}
    run_oracle(case, ref)
    with hfb.Engine("dycore") as eng:
        for k, v in case.ints.items():
            eng.set(k, int(v))
        for k, v in case.reals.items():
            eng.set(k, float(v))
        for name, a in arrs.items():
            eng.bind(name, a)
        eng.run("main")
        h2d, d2h = eng.transfer_bytes()
        assert eng.residency("rho") == ("both", True)
    field = 12 * 40 * 24 * 8
    assert h2d == 6 * field and d2h == 5 * field
    for k in ("th", "u", "v", "w", "p", "rho"):
        assert bits_equal(arrs[k], ref[k]), k


@pytest.mark.parametrize("nz,fused", [(58, True), (100, True), (129, True), (140, False)])
def test_tall_columns_take_the_fused_kernel(nz, fused):
    """Columns of up to 128 faces run the fused step kernel (512 TMEM columns, one CTA per
    SM, above 64 faces): one native launch per step. Taller ones fall back to the portable
    kernels (advection + acoustic launches, the dialect's intermediates through L2)."""
    case = Case(f"tall_{nz}", "dycore", dict(nx=40, ny=12, nz=nz, nsteps=2),
                dict(DYCORE_SCALARS), dict(DYCORE_FILLS))
    stats, _ = run_engine(case, make_inputs(case))
    assert (stats.native_launches == 2) == fused, stats
