"""bench.py's reference arm runs on the host alone (the reference interpreter, one per
core): its JSON line must carry the contract keys the driver reads."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(not (ROOT / "oracle" / "_ref" / "hft_ref").exists(),
                    reason="oracle/_ref/hft_ref not built")
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == "grid-point updates/sec per timestep"
    assert d["unit"] == "grid-point updates/s" and d["value"] > 0
    assert d["higher_is_better"] is True and d["steps"] == 1 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert "workload" in d["config"]


@pytest.mark.skipif(not (ROOT / "oracle" / "_ref" / "hft_ref").exists(),
                    reason="oracle/_ref/hft_ref not built")
def test_reference_arm_asuca_entry():
    """--entry asuca_step: the reference interpreter runs main_asuca (apps/dycore/asuca.h90)
    on its sample blocks; same contract keys."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--entry", "asuca_step", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["config"]["entry"] == "asuca_step"
    assert d["value"] > 0 and "ASUCA" in d["config"]["workload"]
    assert d["cpu_baseline"]["kind"] == "reference"
