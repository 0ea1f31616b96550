"""Programs generated from Hybrid-Fortran sources (paper_1710_08616_b200/hfc: .h90 ->
CUDA C++ for sm_100a -> program plugin) run through the same C ABI and reproduce the
REFERENCE INTERPRETER's outputs bit for bit (tests/golden, produced by oracle/_ref from
the same sources), with the generated code's launch accounting equal to the reference's
simulated launches (interp.cpp:1417-1475)."""
import numpy as np
import pytest

import paper_1710_08616_b200 as hfb
from paper_1710_08616_b200 import hfc
from cases import APPS, CASES, HFC_CASES
from golden_io import bits_equal, decl, load_golden, make_inputs

pytestmark = pytest.mark.gpu
GEN = hfc.GEN_DIR / "dycore_gen.so"
DYCORE_CASES = [c for c in CASES if c.app in ("dycore", "dycore_rk3", "dycore_full", "asuca")]


def run_generated(case, arrs):
    app = APPS[case.app]
    with hfb.Engine(str(GEN)) as eng:
        assert eng.module == "dyn_state"
        for k, v in case.ints.items():
            eng.set(k, int(v))
        for k, v in case.reals.items():
            eng.set(k, float(v))
        for name, a in arrs.items():
            eng.bind(name, a)
        return eng.run(app.entry)


@pytest.mark.parametrize("case", DYCORE_CASES, ids=lambda c: c.name)
def test_generated_dycore_matches_reference(case):
    meta, out, _, _ = load_golden(case.name)
    arrs = make_inputs(case)
    stats = run_generated(case, arrs)
    for name in APPS[case.app].outputs:
        assert bits_equal(arrs[name], out[name]), f"{case.name}: {name} differs"
    if "gpu_launches" in meta:  # the reference's run_gpu_simulated accounting
        assert stats.launches == meta["gpu_launches"]
        assert stats.threads == meta["gpu_threads"]
        assert stats.guard_returns == meta["gpu_guard_returns"]
    assert stats.native_launches == stats.launches


def test_generated_program_per_step_entries_and_residency():
    """per-step entries (no transfers) work on device-resident state; a step without the
    copy-in is the reference's residency error"""
    case = [c for c in DYCORE_CASES if c.name == "dycore_24x20x12_s2"][0]
    with hfb.Engine(str(GEN)) as eng:
        for k, v in case.ints.items():
            eng.set(k, int(v))
        for k, v in case.reals.items():
            eng.set(k, float(v))
        arrs = make_inputs(case)
        for name, a in arrs.items():
            eng.bind(name, a)
        with pytest.raises(hfb.HfbError) as ei:
            eng.run("dycore_step")
        assert ei.value.kind == "residency"
        for name in arrs:
            eng.copy_to_device(name)
        eng.enqueue("dycore_step")
        eng.enqueue("dycore_step")
        eng.synchronize()
        for name in arrs:
            eng.copy_from_device(name)
    _, out, _, _ = load_golden(case.name)
    for name in ("th", "u", "v", "w", "p"):
        assert bits_equal(arrs[name], out[name]), name


@pytest.mark.parametrize("case", HFC_CASES, ids=lambda c: c.name)
def test_generated_feature_program_matches_reference(case):
    """apps/kitchen: intrinsics with mixed kinds, integer arithmetic, if/else if/else,
    privatised and routine-local device arrays, lower bounds 0, startAt/endAt regions,
    nested device routines with intent(inout), module scalars updated on the host."""
    meta, out, _, _ = load_golden(case.name)
    app = APPS[case.app]
    arrs = make_inputs(case)
    with hfb.Engine(str(hfc.GEN_DIR / "kitchen_gen.so")) as eng:
        for k, v in case.ints.items():
            eng.set(k, int(v))
        for k, v in case.reals.items():
            eng.set(k, float(v))
        for name, a in arrs.items():
            _, lower = decl(case.app, name, case.ints)
            eng.bind(name, a, lower=lower)
        stats = eng.run(app.entry)
        scal = {k: eng.get(k) for k in ("alpha", "total_host")}
    for name in app.outputs:
        if name in scal:
            got = np.float64(scal[name]).view(np.uint64)
            assert got == np.float64(out[name].reshape(())).view(np.uint64), name
        else:
            assert bits_equal(arrs[name], out[name]), f"{case.name}: {name} differs"
    assert stats.launches == meta["gpu_launches"]
    assert stats.threads == meta["gpu_threads"]
    assert stats.guard_returns == meta["gpu_guard_returns"]


CORPUS = [c for c in CASES if f"{c.app}_gen" in hfc.CORPUS_SOURCES]


@pytest.mark.parametrize("case", CORPUS, ids=lambda c: c.name)
def test_generated_reference_corpus_matches_reference(case):
    """The reference's own application corpus compiled by hfc (the plugins are built from
    /root/reference by build(); they travel prebuilt): appliesTo(CPU) wrappers over GPU
    kernels, array dummy arguments, element-wise intent(out) device arguments, host array
    updates between transfers, module parameters, damping's template families, and the
    OpenACC-style reduce(+:total) in the simulated order (interp.cpp:1114-1173)."""
    so = hfc.GEN_DIR / f"{case.app}_gen.so"
    if not so.exists():
        pytest.skip(f"{so.name} not built (the reference corpus was absent at build time)")
    meta, out, _, extra = load_golden(case.name)
    app = APPS[case.app]
    arrs = make_inputs(case)
    with hfb.Engine(str(so)) as eng:
        assert eng.module == app.module
        for k, v in case.ints.items():
            eng.set(k, int(v))
        for k, v in case.reals.items():
            eng.set(k, float(v))
        for name, a in arrs.items():
            _, lower = decl(case.app, name, case.ints)
            eng.bind(name, a, lower=lower)
        stats = eng.run(app.entry)
        scal = {k: eng.get(k) for k in app.outputs if k not in arrs}
    for name in app.outputs:
        if name in scal:  # the GPU-mode (acc-simulated) value where it differs
            want = extra.get(f"out_accsim.{name}", out[name])
            assert np.float64(scal[name]).view(np.uint64) == \
                np.float64(want.reshape(())).view(np.uint64), name
        else:
            assert bits_equal(arrs[name], out[name]), f"{case.name}: {name} differs"
    assert stats.launches == meta["gpu_launches"]
    assert stats.threads == meta["gpu_threads"]
    assert stats.guard_returns == meta["gpu_guard_returns"]
    assert stats.native_launches >= 1


def test_generated_program_graph_replay():
    """hfb_run_graph captures the generated host driver's launches (after one warm step has
    materialised the scratch arrays) and replays them: 1 enqueued + 2 replayed steps equal
    the reference's 3 steps, with the same launch accounting per step."""
    case = [c for c in DYCORE_CASES if c.name == "dycore_13x7x10_s3"][0]
    arrs = make_inputs(case)
    with hfb.Engine(str(GEN)) as eng:
        for k, v in case.ints.items():
            eng.set(k, int(v))
        for k, v in case.reals.items():
            eng.set(k, float(v))
        for name, a in arrs.items():
            eng.bind(name, a)
        for name in arrs:
            eng.copy_to_device(name)
        one = eng.enqueue("dycore_step")
        eng.synchronize()
        two = eng.run_graph("dycore_step", 2)
        for name in arrs:
            eng.copy_from_device(name)
    assert two.launches == 2 * one.launches and two.threads == 2 * one.threads
    _, out, _, _ = load_golden(case.name)
    for name in APPS[case.app].outputs:
        assert bits_equal(arrs[name], out[name]), name


def test_generated_reduction_refuses_graph_capture():
    so = hfc.GEN_DIR / "reduction_gen.so"
    if not so.exists():
        pytest.skip("reduction_gen.so not built")
    case = [c for c in CORPUS if c.app == "reduction"][0]
    arrs = make_inputs(case)
    with hfb.Engine(str(so)) as eng:
        for k, v in case.ints.items():
            eng.set(k, int(v))
        for k, v in case.reals.items():
            eng.set(k, float(v))
        for name, a in arrs.items():
            eng.bind(name, a)
        eng.copy_to_device("y")
        eng.run("grid_total")  # warm (allocates the partials)
        with pytest.raises(hfb.HfbError):
            eng.run_graph("grid_total", 1)


def test_generated_host_update_marks_host_copy_newer():
    """surface_flux's setup() updates cover_frac on the host (driver.h90:9-16); after a
    copy-in that makes the device copy stale, so a kernel reading it is the reference's
    residency error (interp.cpp:402-403); copying in again repairs it."""
    so = hfc.GEN_DIR / "surface_flux_gen.so"
    if not so.exists():
        pytest.skip("surface_flux_gen.so not built")
    case = [c for c in CORPUS if c.app == "surface_flux"][0]
    arrs = make_inputs(case)
    with hfb.Engine(str(so)) as eng:
        for k, v in case.ints.items():
            eng.set(k, int(v))
        for name, a in arrs.items():
            eng.bind(name, a)
        for name in arrs:
            eng.copy_to_device(name)
        eng.run("setup")
        with pytest.raises(hfb.HfbError) as ei:
            eng.run("physics_run")
        assert ei.value.kind == "residency" and "cover_frac" in str(ei.value)
        eng.copy_to_device("cover_frac")
        eng.run("physics_run")
