"""CPU-side checks of the C ABI: the library builds for sm_100a, loads, exports every
symbol include/hfb.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import re
from pathlib import Path

import pytest

import paper_1710_08616_b200 as hfb
from paper_1710_08616_b200.runtime import EXPORTS

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    """functions libhfb.so exports: include/hfb.h and the services of include/hfb_plugin.h
    (minus `hfb_plugin`, the one symbol a generated program exports)"""
    text = "".join((ROOT / "include" / h).read_text() for h in ("hfb.h", "hfb_plugin.h"))
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"\b((?:hfb|hfrt|hfk\d+)_\w+)\s*\(", text))
    names.discard("hfb_plugin")
    return sorted(names)


def test_every_declared_symbol_is_exported():
    L = hfb.lib()
    decl = declared_symbols()
    assert decl, "no declarations found"
    for name in decl:
        assert hasattr(L, name), f"libhfb.so does not export {name}"
    assert sorted(EXPORTS) == decl


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          str(ROOT / "paper_1710_08616_b200" / "libhfb.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(hfb.HfbError) as e:
        hfb.Engine("diffusion")
    assert e.value.kind == "cuda"


def test_decomposition_host_logic():
    # 1581 x 1301 on 4 x 2 ranks: tiles cover the grid exactly once
    tiles = [hfb.decomp_init(1581, 1301, 58, 4, 2, r, halo=2) for r in range(8)]
    covered = set()
    for d in tiles:
        for i in range(d.i0, d.i0 + d.nx):
            covered.add(("i", d.ry, i))
        assert d.nx in (395, 396) and d.ny in (650, 651)
    assert tiles[0].west == -1 and tiles[0].east == 1 and tiles[0].north == 4
    assert tiles[7].east == -1 and tiles[7].south == 3
    # send box of one side is the neighbour's receive box shifted by the tile extent
    d0, d1 = tiles[0], tiles[1]
    s_east, _ = hfb.decomp_faces(d0, 1)
    _, r_west = hfb.decomp_faces(d1, 0)
    assert (s_east[0] - d0.nx, s_east[1] - d0.nx) == (r_west[0], r_west[1])
    assert s_east[2:] == r_west[2:]
    with pytest.raises(hfb.HfbError):
        hfb.decomp_init(3, 3, 58, 4, 1, 0)


def test_reference_adapter_builds_and_maps_errors(tmp_path):
    """integration/hfb_adapter.hpp compiles against the reference's headers (the `b200`
    oracle target); without a GPU its run_gpu surfaces the engine's HFB_CUDA status as the
    reference's own hft::Error[runtime] (exit code 10 + ErrKind::Runtime)."""
    import subprocess
    exe = ROOT / "oracle" / "_ref" / "hft_ref_b200"
    if not exe.exists():
        pytest.skip("hft_ref_b200 not built (needs /root/reference at build time)")
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present: tests/test_gpu_adapter.py covers the adapter")
    sc = tmp_path / "s.sc"
    sc.write_text("mode b200\napp dycore\nentry main\nint dyn_state nx 4\n")
    r = subprocess.run([str(exe), str(sc)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 15, (r.returncode, r.stderr)
    assert "hft::Error[runtime] no CUDA device" in r.stderr
