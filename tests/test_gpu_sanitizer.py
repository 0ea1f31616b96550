"""compute-sanitizer over the native kernels (the reference simulates races
and residency; on the B200 the hardware-level checks are memcheck and racecheck):
small runs of every app under the sanitizer report no errors."""
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

SCRIPT = r"""
import sys
sys.path[:0] = [{root!r}, {root!r} + "/tests", {root!r} + "/oracle"]
import paper_1710_08616_b200 as hfb
from pathlib import Path
for scn in ["diffusion_37x21x9_s3", "damping_37x21x9", "bounded_37x21",
            "surface_flux_37x21_t1", "reduction_37x21x9", "reduction_37x21x9_ordered",
            "dycore_24x20x12_s2", "full_24x20x12_s2", "rk3_24x20x12_s1"]:
    eng, st, rep = hfb.Engine.scenario(Path({root!r}) / "tests/scenarios" / (scn + ".scn"))
    eng.close()
print("sanitized ok")
"""


@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_apps_clean_under_compute_sanitizer(tool):
    if not Path(SAN).exists():
        pytest.skip("compute-sanitizer not installed")
    code = SCRIPT.format(root=str(ROOT))
    r = subprocess.run([SAN, "--tool", tool, "--error-exitcode", "9", sys.executable, "-c", code],
                       capture_output=True, text=True, timeout=900)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0 and "sanitized ok" in r.stdout, tail
    out = r.stdout + r.stderr
    assert "ERROR SUMMARY: 0 errors" in out or "0 hazards displayed (0 errors, 0 warnings)" in out, tail
