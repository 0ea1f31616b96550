"""hfc — Hybrid-Fortran (.h90) to CUDA C++ for sm_100a.

    from paper_1710_08616_b200 import hfc
    so = hfc.build(["apps/dycore/dyn_state.h90", "apps/dycore/dycore.h90"], "dycore_gen",
                   "build/dycore_gen.so")
    eng = Engine(so)          # hfb_load_program(ctx, "<path>.so")

The generated translation unit (gen.py) is compiled by nvcc for sm_100a with the same
bit-exactness flags as libhfb.so (-fmad=false, IEEE division and square root) into a
program plugin (include/hfb_plugin.h) linked against libhfb.so.
"""
import os
import subprocess
from pathlib import Path

from .gen import GenError, generate  # noqa: F401
from .parse import ParseError  # noqa: F401

PKG = Path(__file__).resolve().parents[1]
GEN_DIR = PKG / "gen"  # generated plugins (built by __graft_entry__.build, git-ignored)
# programs of this repository generated at build time: name -> sources (repo-relative)
BUILTIN_SOURCES = {
    "dycore_gen": ["apps/dycore/dyn_state.h90", "apps/dycore/dycore.h90",
                   "apps/dycore/asuca.h90"],
    "kitchen_gen": ["apps/kitchen/kit_state.h90", "apps/kitchen/kitchen.h90"],
}
# the reference's own application corpus (proj/tests/data/apps), compiled when the reference
# tree is present (this container); the sources are never copied into the repository
REFERENCE_APPS = Path(os.environ.get("HFB_REFERENCE_APPS", "/root/reference/proj/tests/data/apps"))
CORPUS_SOURCES = {
    "diffusion_gen": ["diffusion/diffusion.h90"],
    "damping_gen": ["damping/damping.h90"],
    "bounded_gen": ["bounded/bounded.h90"],
    "surface_flux_gen": ["surface_flux/sf_state.h90", "surface_flux/surface_flux.h90",
                         "surface_flux/driver.h90"],
    "reduction_gen": ["reduction/reduction.h90"],
}
INCLUDE = PKG.parent / "include"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-fmad=false",
         "-prec-div=true", "-prec-sqrt=true", "-lineinfo", "-shared", "-Xcompiler", "-fPIC"]


def translate(paths, name):
    """CUDA C++ source of the program made of the given .h90 files."""
    return generate([(str(p), Path(p).read_text()) for p in paths], name)


def build(paths, name, out, keep_source=True, checked=False):
    """Translate and compile into the plugin `out` (.so); returns its absolute path.
    checked=True builds the debug variant: every array access is checked against the
    declared bounds and the element init flags (the reference's runtime errors,
    interp.cpp:487-507), reported after each launch as HFB_RUNTIME."""
    out = Path(out).resolve()
    out.parent.mkdir(parents=True, exist_ok=True)
    src = out.with_suffix(".cu")
    src.write_text(translate(paths, name))
    cmd = [NVCC, *FLAGS, *(["-DHFC_CHECKED"] if checked else []), "-I", str(INCLUDE), str(src),
           "-o", str(out), "-L", str(PKG), "-lhfb", "-Xlinker", f"-rpath={PKG}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
    if not keep_source:
        src.unlink()
    return str(out)
