"""State images (HFBSTAT1) and scenario files on the host side (no GPU): the wire format
round-trips, corruption is detected, and every scenario file reproduces the reference
interpreter's golden outputs through the oracle (fills, ArrayValue order, checksums)."""
from pathlib import Path

import numpy as np
import pytest

from cases import APPS, CASE_BY_NAME
from golden_io import bits_equal, decl, make_inputs, run_oracle
from paper_1710_08616_b200 import state

SCN = Path(__file__).resolve().parent / "scenarios"
SCENARIOS = sorted(SCN.glob("*.scn"))


def test_image_roundtrip(tmp_path):
    rng = np.random.default_rng(3)
    st = state.State("damping", "svar",
                     {"nx_mn": ("int", True, -1), "tratio_bnd": ("real", True, 0.3),
                      "mtratio_bnd": ("real", False, 0.0)},
                     {"dens_ref_f": ((1, -1, 0), rng.random((3, 4, 5))),
                      "dens_ptb_bnd": ((1, -1, 0, 1), rng.random((3, 4, 5, 2)))})
    p = tmp_path / "s.hfbstate"
    state.write_state(p, st)
    back = state.read_state(p)
    assert back.program == "damping" and back.module == "svar"
    assert back.scalars == st.scalars
    for k, (lo, a) in st.arrays.items():
        assert back.arrays[k][0] == lo and bits_equal(back.arrays[k][1], a)
    assert state.read_header(p)["program"] == "damping"


def test_image_corruption_detected(tmp_path):
    st = state.State("bounded", "b_state", {"nx": ("int", True, 3)},
                     {"a": ((1, 1), np.arange(9.0).reshape(3, 3))})
    p = tmp_path / "s.hfbstate"
    state.write_state(p, st)
    raw = bytearray(p.read_bytes())
    raw[-20] ^= 1
    p.write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="checksum"):
        state.read_state(p)
    p.write_bytes(bytes(raw[:40]))
    with pytest.raises(ValueError):
        state.read_state(p)


def test_fnv_and_sum_conventions():
    a = np.array([[1.0, 2.0], [3.0, 4.5]])
    s, b = state.checksums(np.asfortranarray(a))  # declared index order, any memory order
    assert s == 10.5
    assert b == state.fnv1a64(np.ascontiguousarray(a).tobytes())
    assert state.fnv1a64(b"") == 0xCBF29CE484222325


def test_anchor_scenario():
    """sum(t_old) after 10 steps of diffusion 16^3 == 2054.7107351501668."""
    sc = state.Scenario.parse(SCN / "diffusion_16x16x16_s10_anchor.scn")
    sums = [float(e.value) for e in sc.expects if e.name == "t_old" and e.kind == "sum"]
    assert sums == [2054.7107351501668]


@pytest.mark.parametrize("path", SCENARIOS, ids=lambda p: p.stem)
def test_scenario_reproduces_reference_through_oracle(path):
    case = CASE_BY_NAME[path.stem.removesuffix("_ordered")]
    sc = state.Scenario.parse(path)
    assert sc.program == APPS[case.app].prog and sc.entry == APPS[case.app].entry

    def declared(name, sets):
        shape, lower = decl(case.app, name, {k: int(v) for k, v in sets.items()
                                             if k in case.ints})
        return [(lo, lo + n - 1) for lo, n in zip(lower, shape)]

    inputs = sc.inputs(declared)
    ref_inputs = make_inputs(case)
    assert set(inputs) == set(ref_inputs)
    for k, (lower, a) in inputs.items():
        assert bits_equal(a, ref_inputs[k]), f"{path.stem}: fill of {k} differs"
    arrs = {k: a.copy() for k, (_, a) in inputs.items()}
    scal = run_oracle(case, arrs)
    if sc.options.get("reduction") == "ordered":  # the acc-simulated order
        scal = {"total": scal["total_accsim"]}
    res = sc.check(arrs, scal)
    bad = [(e.name, e.kind, m) for e, m, ok in res if not ok]
    assert not bad, f"{path.stem}: {bad}"
