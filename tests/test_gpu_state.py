"""Scenario files and state images through the C ABI on the GPU: every scenario (the
reference interpreter's golden checksums) passes hfb_run_scenario; a failing expectation is
HFB_VALIDATION; save -> load is a bit-exact checkpoint/resume; device-newer arrays are
saved from the device without changing residency."""
from pathlib import Path

import numpy as np
import pytest

import paper_1710_08616_b200 as hfb
from paper_1710_08616_b200 import state
from cases import DYCORE_FILLS, DYCORE_SCALARS
from golden_io import bits_equal
import oracle

pytestmark = pytest.mark.gpu
SCN = Path(__file__).resolve().parent / "scenarios"


@pytest.mark.parametrize("path", sorted(SCN.glob("*.scn")), ids=lambda p: p.stem)
def test_scenario_on_gpu(path):
    eng, stats, report = hfb.Engine.scenario(path)
    try:
        lines = [l for l in report.splitlines() if l]
        assert lines and all(l.endswith(" ok") for l in lines), report
        assert stats.native_launches > 0
    finally:
        eng.close()


def test_scenario_failure_is_validation(tmp_path):
    src = (SCN / "bounded_37x21.scn").read_text().splitlines()
    bad = [l if not l.startswith("expect b bits") else "expect b bits 0x1234" for l in src]
    p = tmp_path / "bad.scn"
    p.write_text("\n".join(bad) + "\n")
    with pytest.raises(hfb.HfbError) as ei:
        hfb.Engine.scenario(p)
    assert ei.value.kind == "validation" and "b bits" in str(ei.value)


def _dycore_engine(nx, ny, nz, nsteps):
    eng = hfb.Engine("dycore")
    for k, v in dict(nx=nx, ny=ny, nz=nz, nsteps=nsteps).items():
        eng.set(k, v)
    for k, v in DYCORE_SCALARS.items():
        eng.set(k, v)
    arrs = {k: oracle.fill((nz, nx, ny), *DYCORE_FILLS[k]) for k in DYCORE_FILLS}
    for k, a in arrs.items():
        eng.bind(k, a)
    return eng, arrs


def test_checkpoint_resume_bit_exact(tmp_path):
    nx, ny, nz = 40, 36, 20
    eng, arrs = _dycore_engine(nx, ny, nz, 2)
    eng.run("main")
    ck = tmp_path / "step2.hfbstate"
    eng.save_state(ck)
    img = state.read_state(ck)
    assert img.program == "dycore" and img.scalars["nsteps"] == ("int", True, 2)
    for k in DYCORE_FILLS:
        assert bits_equal(img.arrays[k][1], arrs[k])
    eng.set("nsteps", 1)
    eng.run("main")  # 3 steps in total on the original context
    res = hfb.Engine.from_state(ck)
    try:
        res.set("nsteps", 1)
        res.run("main")  # resumed: 2 + 1 steps
        ref = {k: oracle.fill((nz, nx, ny), *DYCORE_FILLS[k]) for k in DYCORE_FILLS}
        oracle.dycore_run(3, DYCORE_SCALARS, *(ref[k] for k in ("rho", "th", "u", "v", "w", "p")))
        for k in DYCORE_FILLS:
            assert bits_equal(res.array(k), arrs[k]), k
            assert bits_equal(res.array(k), ref[k]), k
            s, b = res.checksum(k)
            assert (s, b) == state.checksums(ref[k])
    finally:
        res.close()
        eng.close()


def test_save_reads_device_newer_copy(tmp_path):
    nx, ny, nz = 33, 20, 12
    eng, arrs = _dycore_engine(nx, ny, nz, 1)
    for k in arrs:
        eng.copy_to_device(k)
    eng.enqueue("dycore_step")
    eng.enqueue("dycore_step")
    eng.synchronize()
    assert eng.residency("th") == ("device", True)
    p = tmp_path / "dev.hfbstate"
    eng.save_state(p)
    assert eng.residency("th") == ("device", True)  # saving does not transfer
    ref = {k: oracle.fill((nz, nx, ny), *DYCORE_FILLS[k]) for k in DYCORE_FILLS}
    oracle.dycore_run(2, DYCORE_SCALARS, *(ref[k] for k in ("rho", "th", "u", "v", "w", "p")))
    img = state.read_state(p)
    for k in DYCORE_FILLS:
        assert bits_equal(img.arrays[k][1], ref[k]), k
    # the host buffers were not touched
    assert bits_equal(arrs["th"], oracle.fill((nz, nx, ny), *DYCORE_FILLS["th"]))
    eng.close()


def test_python_written_image_loads(tmp_path):
    """The oracle side writes an image with state.py; the engine loads it and runs."""
    nx, ny, nz = 24, 20, 12
    a = {k: oracle.fill((nz, nx, ny), *DYCORE_FILLS[k]) for k in DYCORE_FILLS}
    scal = {"nx": ("int", True, nx), "ny": ("int", True, ny), "nz": ("int", True, nz),
            "nsteps": ("int", True, 2)}
    scal.update({k: ("real", True, v) for k, v in DYCORE_SCALARS.items()})
    p = tmp_path / "py.hfbstate"
    state.write_state(p, state.State("dycore", "dyn_state", scal,
                                     {k: ((1, 1, 1), v) for k, v in a.items()}))
    eng = hfb.Engine.from_state(p)
    try:
        eng.run("main")
        oracle.dycore_run(2, DYCORE_SCALARS, *(a[k] for k in ("rho", "th", "u", "v", "w", "p")))
        for k in DYCORE_FILLS:
            assert bits_equal(eng.array(k), a[k]), k
    finally:
        eng.close()


def test_corrupt_image_is_io_error(tmp_path):
    eng, _ = _dycore_engine(8, 8, 4, 1)
    p = tmp_path / "x.hfbstate"
    eng.save_state(p)
    raw = bytearray(p.read_bytes())
    raw[len(raw) // 2] ^= 0xFF
    p.write_bytes(bytes(raw))
    with pytest.raises(hfb.HfbError) as ei:
        eng.load_state(p)
    assert ei.value.kind == "io"
    eng.close()
