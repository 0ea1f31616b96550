"""The reference-side C++ binding (integration/hfb_adapter.hpp), compiled against the
reference's own headers and library (oracle/_ref/hft_ref_b200, oracle/Makefile `b200`):
`mode b200` of the reference harness runs each golden case's entry on the B200 through
hfb_adapter::run_gpu — the drop-in for run_gpu_simulated(program, state, entry) — on an
hft::interp::MachineState, and must reproduce the reference interpreter's outputs bit for
bit (1e-12 for the tree-summed reduction) with the same LaunchStats."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from cases import APPS, CASES
from golden_io import bits_equal, decl, load_golden
from hfb_dump import read_dump

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "oracle" / "_ref" / "hft_ref_b200"


def scenario(case, out):
    app = APPS[case.app]
    lines = ["mode b200", f"app {app.prog}", f"entry {app.entry}"]
    for k, v in case.ints.items():
        lines.append(f"int {app.module} {k} {v}")
    for k, v in case.reals.items():
        lines.append(f"real {app.module} {k} {float(v).hex()}")
    for name in app.arrays:
        shape, lower = decl(case.app, name, case.ints)
        bounds = " ".join(f"{lo} {lo + n - 1}" for lo, n in zip(lower, shape))
        lines.append(f"array {app.module} {name} {bounds}")
    for k, (seed, off, scale) in case.fills.items():
        lines.append(f"fill {app.module} {k} {seed} {float(off).hex()} {float(scale).hex()}")
    for k in app.outputs:
        lines.append(f"dump {app.module} {k}")
    lines.append(f"out {out}")
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("case", [c for c in CASES if c.gpu_check], ids=lambda c: c.name)
def test_reference_harness_through_adapter(case, tmp_path):
    if not EXE.exists():
        pytest.skip("hft_ref_b200 not built (needs the reference sources at build time)")
    out = tmp_path / "out.bin"
    sc = tmp_path / "case.sc"
    sc.write_text(scenario(case, out))
    r = subprocess.run([str(EXE), str(sc)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    meta, golden, _, extra = load_golden(case.name)
    dump = read_dump(out)
    app = APPS[case.app]
    for k in app.outputs:
        got = dump.arrays[f"{app.module}.{k}"].data
        if app.backend == "acc" and k == "total":
            want = float(np.asarray(golden[k]).reshape(()))
            assert abs(float(got) - want) <= 1e-12 * abs(want), k
        else:
            assert bits_equal(np.asarray(got).reshape(golden[k].shape), golden[k]), k
    assert (dump.launches, dump.threads, dump.guard_returns) == \
        (meta["gpu_launches"], meta["gpu_threads"], meta["gpu_guard_returns"])


def test_adapter_maps_engine_errors_to_reference_error_kinds(tmp_path):
    """A residency violation inside the engine comes back as hft::Error[residency]."""
    if not EXE.exists():
        pytest.skip("hft_ref_b200 not built")
    case = [c for c in CASES if c.app == "dycore"][0]
    sc = tmp_path / "case.sc"
    text = scenario(case, tmp_path / "o.bin").replace(f"entry {APPS['dycore'].entry}",
                                                      "entry dycore_step")
    sc.write_text(text)
    r = subprocess.run([str(EXE), str(sc)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 10 + 6, (r.returncode, r.stderr)  # ErrKind::Residency
    assert "hft::Error[residency]" in r.stderr
