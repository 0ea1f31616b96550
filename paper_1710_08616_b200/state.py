"""HFBSTAT1 state images and scenario files, host side (mirror of csrc/hfb_runtime.cu).

The reference specifies a harness input "scenario file naming the program, array shapes,
fill patterns (constant, linear ramp, seeded pseudo-random with stated algorithm and
seed), and expected-checksum entries" and never implemented it
(proj/src/scenario.cpp:1 is a placeholder). This module reads and writes the same two
formats the C ABI does (hfb_run_scenario, hfb_save_state / hfb_load_state), so the
oracle (tests/, oracle/), the CPU baseline and the B200 engine share one wire format.

Arrays are stored and filled in the reference's ArrayValue order: row-major, last
subscript fastest (interp.cpp:485-494). Pure numpy: no device, no engine.
"""
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .synthetic import uniform

MAGIC = b"HFBSTAT1"
_FNV_BASIS = 0xCBF29CE484222325
_FNV_PRIME = 0x100000001B3
_MASK = (1 << 64) - 1


def fnv1a64(data, h=_FNV_BASIS):
    """FNV-1a 64 of a bytes-like object (the image trailer and the `bits` checksum)."""
    for b in bytes(data):
        h = ((h ^ b) * _FNV_PRIME) & _MASK
    return h


def checksums(a):
    """(sum in ArrayValue order, FNV-1a 64 of the bits) of an array given in its declared
    index order (any memory order)."""
    flat = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    s = 0.0
    for v in flat.tolist():  # sequential, in order: the engine's fp64 sum
        s += v
    return s, fnv1a64(flat.tobytes())


# ---- HFBSTAT1 images --------------------------------------------------------------------
@dataclass
class State:
    program: str
    module: str
    scalars: dict = field(default_factory=dict)  # name -> (kind 'int'|'real', set, value)
    arrays: dict = field(default_factory=dict)   # name -> (lower tuple, ndarray C-order)


def _str(b):
    return struct.pack("<I", len(b)) + b


def write_state(path, st):
    body = bytearray(MAGIC)
    body += struct.pack("<I", 1)
    body += _str(st.program.encode()) + _str(st.module.encode())
    body += struct.pack("<I", len(st.scalars))
    for name in sorted(st.scalars):  # the engine writes its std::map order
        kind, is_set, v = st.scalars[name]
        body += _str(name.encode())
        body += struct.pack("<BB", 0 if kind == "int" else 1, 1 if is_set else 0)
        body += struct.pack("<q", int(v)) if kind == "int" else struct.pack("<d", float(v))
    body += struct.pack("<I", len(st.arrays))
    for name in sorted(st.arrays):
        lower, a = st.arrays[name]
        a = np.ascontiguousarray(a, dtype=np.float64)
        upper = tuple(lo + n - 1 for lo, n in zip(lower, a.shape))
        body += _str(name.encode()) + struct.pack("<I", a.ndim)
        body += struct.pack(f"<{a.ndim}q", *lower) + struct.pack(f"<{a.ndim}q", *upper)
        body += a.astype("<f8").tobytes()
    body += struct.pack("<Q", fnv1a64(body))
    Path(path).write_bytes(bytes(body))


class _Rd:
    def __init__(self, data):
        self.d, self.o = data, 0

    def take(self, n):
        if self.o + n > len(self.d):
            raise ValueError("truncated state image")
        b = self.d[self.o:self.o + n]
        self.o += n
        return b

    def u(self, fmt):
        return struct.unpack("<" + fmt, self.take(struct.calcsize("<" + fmt)))

    def s(self):
        (n,) = self.u("I")
        return self.take(n).decode()


def read_header(path):
    r = _Rd(Path(path).read_bytes())
    if r.take(8) != MAGIC:
        raise ValueError(f"{path}: not an HFBSTAT1 image")
    (ver,) = r.u("I")
    return {"version": ver, "program": r.s(), "module": r.s()}


def read_state(path, verify=True):
    data = Path(path).read_bytes()
    r = _Rd(data)
    if r.take(8) != MAGIC:
        raise ValueError(f"{path}: not an HFBSTAT1 image")
    (ver,) = r.u("I")
    if ver != 1:
        raise ValueError(f"{path}: unsupported version {ver}")
    st = State(r.s(), r.s())
    (ns,) = r.u("I")
    for _ in range(ns):
        name = r.s()
        kind, is_set = r.u("BB")
        (v,) = r.u("q") if kind == 0 else r.u("d")
        st.scalars[name] = ("int" if kind == 0 else "real", bool(is_set), v)
    (na,) = r.u("I")
    for _ in range(na):
        name = r.s()
        (rank,) = r.u("I")
        lo = r.u(f"{rank}q")
        hi = r.u(f"{rank}q")
        shape = tuple(h - l + 1 for l, h in zip(lo, hi))
        n = int(np.prod(shape))
        a = np.frombuffer(r.take(8 * n), dtype="<f8").astype(np.float64).reshape(shape)
        st.arrays[name] = (tuple(lo), a)
    end = r.o
    (stored,) = r.u("Q")
    if verify and stored != fnv1a64(data[:end]):
        raise ValueError(f"{path}: checksum mismatch")
    return st


# ---- scenario files -----------------------------------------------------------------------
@dataclass
class Expect:
    line: int
    name: str
    kind: str      # sum | bits | value
    value: str
    tol: float = 0.0


@dataclass
class Scenario:
    program: str = ""
    entry: str = "main"
    options: dict = field(default_factory=dict)  # e.g. {"reduction": "ordered"}
    sets: dict = field(default_factory=dict)     # scalar -> float (as written)
    shapes: dict = field(default_factory=dict)   # array -> [(lo, hi), ...]
    fills: list = field(default_factory=list)    # (array, kind, params)
    expects: list = field(default_factory=list)

    @classmethod
    def parse(cls, path_or_text):
        text = path_or_text
        if isinstance(path_or_text, Path) or "\n" not in str(path_or_text):
            text = Path(path_or_text).read_text()
        sc = cls()
        for ln, raw in enumerate(text.splitlines(), 1):
            t = raw.split("#", 1)[0].split()
            if not t:
                continue
            k = t[0]
            if k == "program":
                sc.program = t[1].lower()
            elif k == "entry":
                sc.entry = t[1]
            elif k == "option":
                sc.options[t[1]] = t[2]
            elif k == "set":
                sc.sets[t[1].lower()] = float(t[2])
            elif k == "array":
                dims = []
                for d in t[2:]:
                    if ":" in d:
                        a, b = d.split(":")
                        dims.append((int(float(a)), int(float(b))))
                    else:
                        dims.append((1, int(float(d))))
                sc.shapes[t[1].lower()] = dims
            elif k == "fill":
                kind = t[2]
                if kind == "splitmix":
                    params = (int(t[3], 0), float(t[4]), float(t[5]))
                else:
                    params = tuple(float(x) for x in t[3:])
                sc.fills.append((t[1].lower(), kind, params))
            elif k == "expect":
                sc.expects.append(Expect(ln, t[1].lower(), t[2], t[3],
                                         float(t[4]) if len(t) > 4 else 0.0))
            else:
                raise ValueError(f"scenario line {ln}: unknown keyword {k!r}")
        return sc

    def fill_array(self, kind, params, shape):
        n = int(np.prod(shape))
        flat = np.arange(n, dtype=np.uint64)
        if kind == "const":
            out = np.full(n, params[0])
        elif kind == "ramp":
            out = params[0] + params[1] * flat.astype(np.float64)
        elif kind == "splitmix":
            seed, off, scale = params
            out = off + scale * uniform(seed, flat)
        else:
            raise ValueError(f"unknown fill {kind!r}")
        return out.reshape(shape)

    def inputs(self, declared_shape):
        """{array: (lower, C-order ndarray)} of every filled array; `declared_shape(name,
        sets)` gives [(lo, hi), ...] for arrays without an `array` line."""
        out = {}
        for name, kind, params in self.fills:
            dims = self.shapes.get(name) or declared_shape(name, self.sets)
            shape = tuple(h - l + 1 for l, h in dims)
            out[name] = (tuple(l for l, _ in dims), self.fill_array(kind, params, shape))
        return out

    def check(self, arrays, scalars=None):
        """Evaluate the expectations on result arrays (declared index order) and scalars:
        [(expect, measured, ok)]."""
        res = []
        for e in self.expects:
            if e.kind in ("sum", "bits"):
                s, b = checksums(arrays[e.name])
                if e.kind == "sum":
                    want = float(e.value)
                    ok = s == want if e.tol == 0 else abs(s - want) <= e.tol * abs(want)
                    res.append((e, s, ok))
                else:
                    res.append((e, b, b == int(e.value, 0)))
            elif e.kind == "value":
                v, want = float(scalars[e.name]), float(e.value)
                ok = v == want if e.tol == 0 else abs(v - want) <= e.tol * abs(want)
                res.append((e, v, ok))
            else:
                raise ValueError(f"unknown expectation {e.kind!r}")
        return res
