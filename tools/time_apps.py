#!/usr/bin/env python3
"""Device-resident timings of the reference corpus kernels at production size (CUDA events
on the engine stream, per-step entries), with their algorithmic bytes."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1710_08616_b200 as hfb  # noqa: E402
from paper_1710_08616_b200 import synthetic  # noqa: E402

NX, NY, NZ = 1581, 1301, 58


def timed(eng, entry, n=20):
    s = torch.cuda.ExternalStream(eng.stream)
    for _ in range(3):
        eng.enqueue(entry)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n):
        eng.enqueue(entry)
    e1.record(s)
    eng.synchronize()
    return e0.elapsed_time(e1) / n


def report(name, ms, nbytes, units):
    print(f"{name}: {ms:.4f} ms  {units / ms * 1e3:.3e} units/s  {nbytes / ms / 1e6:.0f} GB/s(alg)")


def damping():
    eng = hfb.Engine("damping")
    for k, v in dict(nx_mn=1, nx_mx=NX, ny_mn=1, ny_mx=NY, nz_mn=1, nz_mx=NZ).items():
        eng.set(k, v)
    eng.set("tratio_bnd", 0.3)
    eng.set("mtratio_bnd", 0.7)
    a = {"dens_ref_f": synthetic.field((NZ, NX, NY), 2, 1.0, 1.0, order="F"),
         "dens_ptb_damp": np.zeros((NZ, NX, NY), order="F"),
         "dens_ptb_bnd": synthetic.field((NZ, NX, NY, 2), 3, -0.005, 0.01, order="F")}
    for k, v in a.items():
        eng.bind(k, v)
        eng.copy_to_device(k)
    report("damping", timed(eng, "lateral_and_upper_damping"), 32 * NX * NY * NZ, NX * NY * NZ)
    eng.close()


def reduction(ordered):
    eng = hfb.Engine("reduction")
    eng.set_reduction_order(ordered)
    for k, v in dict(nx=NX, ny=NY, nz=NZ).items():
        eng.set(k, v)
    eng.set("total", 0.0)
    y = synthetic.field((NZ, NX, NY), 6, 0.0, 1.0, order="F")
    eng.bind("y", y)
    eng.copy_to_device("y")
    import time
    for _ in range(3):
        eng.run("grid_total")
    t0 = time.perf_counter()
    n = 20
    for _ in range(n):
        eng.run("grid_total")  # synchronous: returns the total to the host
    ms = (time.perf_counter() - t0) / n * 1e3
    report(f"reduction ({'ordered' if ordered else 'tree'}, incl. host readback)", ms,
           8 * NX * NY * NZ, NX * NY * NZ)
    eng.close()


def bounded():
    eng = hfb.Engine("bounded")
    eng.set("nx", NX * 4)
    eng.set("ny", NY * 4)
    a = {"a": synthetic.field((NX * 4, NY * 4), 4, 0.0, 1.0, order="F"),
         "b": np.zeros((NX * 4, NY * 4), order="F")}
    for k, v in a.items():
        eng.bind(k, v)
        eng.copy_to_device(k)
    report("bounded (6324x5204)", timed(eng, "interior_update"), 16 * 16 * NX * NY, 16 * NX * NY)
    eng.close()


if __name__ == "__main__":
    damping()
    bounded()
    reduction(False)
    reduction(True)
