"""python -m paper_1710_08616_b200.hfc -o prog.so --name prog a.h90 b.h90 [--emit-only] [--checked]"""
import argparse

from . import build, translate

ap = argparse.ArgumentParser(prog="hfc")
ap.add_argument("sources", nargs="+")
ap.add_argument("-o", "--out", required=True)
ap.add_argument("--name", required=True)
ap.add_argument("--emit-only", action="store_true", help="write the .cu only")
ap.add_argument("--checked", action="store_true",
                help="debug build: bounds and unset-element checks on every array access")
a = ap.parse_args()
if a.emit_only:
    open(a.out, "w").write(translate(a.sources, a.name))
else:
    print(build(a.sources, a.name, a.out, checked=a.checked))
