"""The CPU restatement (oracle/) against fixtures produced by the reference itself.

Every case in tests/cases.py: the reference interpreter's output
(tests/golden/<case>.npz, made by tests/golden/make_golden.py from
/root/reference/proj/src/interp.cpp) must equal the C restatement bit for bit,
in both the reference's ArrayValue order and the Fortran KIJ order.
"""
import numpy as np
import pytest

from cases import APPS, CASES
from golden_io import bits_equal, load_golden, make_inputs, run_oracle


@pytest.mark.parametrize("case", CASES, ids=lambda c: c.name)
@pytest.mark.parametrize("order", ["C", "F"])
def test_oracle_matches_reference(case, order):
    meta, out, init, extra = load_golden(case.name)
    arrs = make_inputs(case, order=order)
    scalars = run_oracle(case, arrs)
    for name in APPS[case.app].outputs:
        if name in scalars:
            got = np.float64(scalars[name])
            assert bits_equal(got.reshape(1), out[name].reshape(1)), (name, got, out[name])
        else:
            assert bits_equal(arrs[name], out[name]), f"{case.name}: {name} differs"
    if "out_accsim.total" in extra:
        # the OpenACC-simulated combine order (interp.cpp:1163-1173) is restated exactly
        assert bits_equal(np.float64(scalars["total_accsim"]).reshape(1),
                          extra["out_accsim.total"].reshape(1))


def test_diffusion_anchor_checksum():
    # sum(t_old) after 10 steps of 16^3 from splitmix64 seed 0
    meta, out, init, extra = load_golden("diffusion_16x16x16_s10_anchor")
    assert out["t_old"].sum() == pytest.approx(2054.7107351501668, rel=0, abs=1e-9)


def test_dycore_drift_envelope_100_steps():
    """100-step run stays bounded and the oracle tracks the reference exactly."""
    meta, out, init, extra = load_golden("dycore_13x7x10_s100")
    th = out["th"]
    assert np.isfinite(th).all() and 299.0 < th.min() and th.max() < 302.0
    assert np.abs(out["w"]).max() < 0.05
