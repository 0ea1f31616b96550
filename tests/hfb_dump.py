"""Reader for the HFTD dump files written by oracle/ref_driver.cpp (test infrastructure).

Each array comes back in the reference's ArrayValue order: row-major over the
declared dims, last subscript fastest (/root/reference/proj/src/interp.cpp:485-494),
together with its inclusive lower/upper bounds and per-element init flags.
"""
import struct
from dataclasses import dataclass

import numpy as np


@dataclass
class DumpArray:
    name: str
    lower: tuple
    upper: tuple
    data: np.ndarray   # shaped by the declared dims (row-major, last fastest)
    init: np.ndarray   # uint8, same shape


@dataclass
class Dump:
    launches: int
    threads: int
    guard_returns: int
    seconds: float
    arrays: dict


def read_dump(path) -> Dump:
    b = open(path, "rb").read()
    if b[:4] != b"HFTD":
        raise ValueError(f"{path}: not an HFTD dump")
    o = 8
    launches, threads, guards, secs = struct.unpack_from("<qqqd", b, o)
    o += 32
    (n,) = struct.unpack_from("<I", b, o)
    o += 4
    arrays = {}
    for _ in range(n):
        (ln,) = struct.unpack_from("<I", b, o)
        o += 4
        name = b[o:o + ln].decode()
        o += ln
        (rank,) = struct.unpack_from("<I", b, o)
        o += 4
        lo = struct.unpack_from("<%dq" % rank, b, o)
        o += 8 * rank
        hi = struct.unpack_from("<%dq" % rank, b, o)
        o += 8 * rank
        (cnt,) = struct.unpack_from("<q", b, o)
        o += 8
        data = np.frombuffer(b, dtype="<f8", count=cnt, offset=o).copy()
        o += 8 * cnt
        init = np.frombuffer(b, dtype=np.uint8, count=cnt, offset=o).copy()
        o += cnt
        shape = tuple(h - l + 1 for l, h in zip(lo, hi)) or ()
        arrays[name] = DumpArray(name, lo, hi, data.reshape(shape), init.reshape(shape))
    return Dump(launches, threads, guards, secs, arrays)
