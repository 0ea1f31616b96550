#!/usr/bin/env python3
"""Generate the golden fixtures from the REFERENCE ITSELF (run here, in the build
container, where /root/reference exists). Test infrastructure only.

For every case in tests/cases.py this writes a scenario file, runs the
reference's own interpreter (oracle/_ref/hft_ref = /root/reference/proj/src/*.cpp
+ oracle/ref_driver.cpp, built by `make -C oracle ref`) under run_reference, and —
unless the case opts out — under run_gpu_simulated (shuffled thread order) and
run_cpu_generated too, requiring the three oracle modes to agree bit-for-bit
(1e-12 relative for the acc-simulated reduction). The reference-mode
outputs are stored as tests/golden/<case>.npz with a JSON header.

Usage: python tests/golden/make_golden.py [case-name ...]
"""
import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from cases import APPS, CASES, HFC_CASES, OWN_APPS, REF_APPS, REPO  # noqa: E402
from hfb_dump import read_dump  # noqa: E402

HFT_REF = REPO / "oracle" / "_ref" / "hft_ref"


def scenario_text(case, mode, out):
    app = APPS[case.app]
    lines = []
    for root, rel in app.sources:
        lines.append(f"source {(REF_APPS if root == 'ref' else OWN_APPS) / rel}")
    lines.append(f"mode {mode}")
    if mode == "gpu":
        lines.append("entry hfd_" + app.entry)
        lines.append(f"backend {app.backend}")
        lines.append(f"order {case.order}")
    else:
        lines.append(f"entry {app.entry}")
    lines.append("max_steps 2000000000")
    for a, d in app.families:
        lines.append(f"family {a} {d}")
    for k, v in case.ints.items():
        lines.append(f"int {app.module} {k} {v}")
    for k, v in case.reals.items():
        lines.append(f"real {app.module} {k} {float(v).hex()}")
    for k, (seed, off, scale) in case.fills.items():
        lines.append(f"fill {app.module} {k} {seed} {float(off).hex()} {float(scale).hex()}")
    for k in case.unset:
        lines.append(f"unset {app.module} {k}")
    for k in app.outputs:
        lines.append(f"dump {app.module} {k}")
    lines.append(f"out {out}")
    return "\n".join(lines) + "\n"


def run_mode(case, mode, tmp):
    out = Path(tmp) / f"{case.name}.{mode}.bin"
    sc = Path(tmp) / f"{case.name}.{mode}.sc"
    sc.write_text(scenario_text(case, mode, out))
    r = subprocess.run([str(HFT_REF), str(sc)], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"{case.name} [{mode}] failed rc={r.returncode}: {r.stderr.strip()}")
    return read_dump(out)


def same_bits(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint64),
                          np.ascontiguousarray(b).view(np.uint64))


def main(names):
    if not HFT_REF.exists():
        subprocess.run(["make", "-C", str(REPO / "oracle"), "ref"], check=True)
    cases = [c for c in CASES + HFC_CASES if not names or c.name in names]
    with tempfile.TemporaryDirectory() as tmp:
        for case in cases:
            app = APPS[case.app]
            ref = run_mode(case, "ref", tmp)
            modes_checked = ["ref"]
            if case.gpu_check:
                for mode in ("gpu", "cpu"):
                    if mode == "cpu" and app.backend == "acc":
                        continue  # the CPU backend emits an OMP reduction the interpreter runs sequentially
                    other = run_mode(case, mode, tmp)
                    for k in app.outputs:
                        key = f"{app.module}.{k}"
                        a, b = ref.arrays[key].data, other.arrays[key].data
                        if app.backend == "acc" and k == "total":
                            rel = abs(float(a) - float(b)) / max(abs(float(a)), 1e-300)
                            assert rel <= 1e-12, (case.name, mode, rel)
                        else:
                            assert same_bits(a, b), f"{case.name}: {mode} differs from ref in {k}"
                    modes_checked.append(mode)
                    if mode == "gpu":
                        gpu = other
            payload = {}
            meta = {"case": case.name, "app": case.app, "ints": case.ints, "reals": case.reals,
                    "fills": {k: list(v) for k, v in case.fills.items()}, "unset": case.unset,
                    "modes_checked": modes_checked, "ref_seconds": ref.seconds, "arrays": {}}
            for k in app.outputs:
                arr = ref.arrays[f"{app.module}.{k}"]
                payload[f"out.{k}"] = arr.data
                payload[f"init.{k}"] = arr.init
                meta["arrays"][k] = {"lower": list(arr.lower), "upper": list(arr.upper)}
            if case.gpu_check:
                meta["gpu_launches"] = gpu.launches
                meta["gpu_threads"] = gpu.threads
                meta["gpu_guard_returns"] = gpu.guard_returns
                if app.backend == "acc":
                    payload["out_accsim.total"] = gpu.arrays[f"{app.module}.total"].data
            payload["meta"] = np.frombuffer(json.dumps(meta, sort_keys=True).encode(), np.uint8)
            np.savez_compressed(HERE / f"{case.name}.npz", **payload)
            print(f"{case.name}: modes {modes_checked}, ref {ref.seconds:.2f}s")


if __name__ == "__main__":
    main(sys.argv[1:])
