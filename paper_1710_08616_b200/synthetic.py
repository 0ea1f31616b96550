"""Synthetic initial states: value = offset + scale * u(seed, flat).

u(seed, flat) = (splitmix64((seed << 40) + flat) >> 11) * 2**-53 with the reference's
SplitMix64 (/root/reference/proj/src/interp.cpp:22-28); `flat` is the logical
row-major index over the GLOBAL declared dims (interp.cpp:485-494), so every tile of
a decomposition sees exactly the values of the undecomposed field.
"""
import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def uniform(seed, flat):
    return (splitmix64((np.uint64(seed) << np.uint64(40)) + flat) >> np.uint64(11)).astype(
        np.float64) * 2.0 ** -53


def field(gshape, seed, offset, scale, box=None, order="C"):
    """Field over global declared shape `gshape`; `box` = per-dim (start, stop) 0-based
    slice of the global index space (a tile), default the whole field."""
    box = box or [(0, n) for n in gshape]
    idx = [np.arange(a, b, dtype=np.uint64) for a, b in box]
    flat = np.zeros([b - a for a, b in box], dtype=np.uint64)
    stride = np.uint64(1)
    for d in range(len(gshape) - 1, -1, -1):
        shape = [1] * len(gshape)
        shape[d] = -1
        flat += idx[d].reshape(shape) * stride
        stride *= np.uint64(gshape[d])
    out = offset + scale * uniform(seed, flat)
    return np.asfortranarray(out) if order == "F" else np.ascontiguousarray(out)


# dycore synthetic state (same conventions as tests/cases.py)
DYCORE_SCALARS = {"dt": 0.1, "rdx": 2.0, "rdy": 2.0, "rdz": 20.0, "cs2": 1.0,
                  "grav": 0.0327, "th0": 300.0}
DYCORE_FILLS = {"rho": (7, 1.0, 0.1), "th": (8, 300.0, 1.0), "u": (9, -0.01, 0.02),
                "v": (10, -0.01, 0.02), "w": (11, -0.002, 0.004), "p": (12, -0.005, 0.01)}
# column physics of the full timestep (dyn_state.tsfc / colm, dycore.h90 column_physics)
PHYS_SCALARS = {"ch": 0.05, "rrelax": 0.01}
PHYS_FILLS = {"tsfc": (13, 300.0, 2.0), "colm": (14, 300.0, 0.5)}


def asuca_params(nz, nsound=6, nbnd=8, kdmp=None, rdmp=0.2):
    """dyn_state scalars of the ASUCA scheme (asuca.h90): nsound short steps per long step,
    lateral damping band of nbnd cells, upper sponge above kdmp (default: the top quarter)."""
    kdmp = nz - max(1, nz // 4) if kdmp is None else kdmp
    return {"nsound": nsound, "nbnd": nbnd, "kdmp": kdmp, "rdmp": rdmp, "rnbnd": 1.0 / nbnd,
            "rnzd": 1.0 / (nz - kdmp)}
