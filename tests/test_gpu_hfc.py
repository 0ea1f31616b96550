"""Programs generated from Hybrid-Fortran sources (paper_1710_08616_b200/hfc: .h90 ->
CUDA C++ for sm_100a -> program plugin) run through the same C ABI and reproduce the
REFERENCE INTERPRETER's outputs bit for bit (tests/golden, produced by oracle/_ref from
the same sources), with the generated code's launch accounting equal to the reference's
simulated launches (interp.cpp:1417-1475)."""
import numpy as np
import pytest

import paper_1710_08616_b200 as hfb
from paper_1710_08616_b200 import hfc
from cases import APPS, CASES
from golden_io import bits_equal, load_golden, make_inputs

pytestmark = pytest.mark.gpu
GEN = hfc.GEN_DIR / "dycore_gen.so"
DYCORE_CASES = [c for c in CASES if c.app in ("dycore", "dycore_rk3", "dycore_full")]


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
