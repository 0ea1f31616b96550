"""Python host mirror of the reference's executor interface, over the C ABI (include/hfb.h).

The reference runs a Hybrid-Fortran program with

    Program p(units); MachineState st = p.prepare_state(); ...
    LaunchStats s = run_gpu_simulated(p, st, "hfd_main");      # interp.hpp:113-122

Here the same shape of call runs the program's kernels natively on a B200:

    eng = Engine("diffusion")                     # Program + MachineState (+ device)
    eng.set("nx", 128); ...; eng.bind("t_old", a)  # module scalars / ObjectSlot host buffers
    stats = eng.run("main")                        # LaunchStats (launches/threads/guard_returns)

Errors are raised as HfbError with the reference's ErrKind name (diagnostics.hpp:21-32).
There is no fallback: if libhfb.so or a CUDA device is missing, Engine() raises.
"""
import ctypes
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
# HFB_LIB: another build of the library — the A/B build libhfb_variants.so (make -C csrc
# variants), which adds the measured-slower kernel variants; bench.py refuses it
LIB_PATH = Path(os.environ["HFB_LIB"]) if os.environ.get("HFB_LIB") else PKG / "libhfb.so"
VARIANTS_LIB = PKG / "libhfb_variants.so"
CSRC = PKG / "csrc"

KINDS = {0: "ok", 10: "config", 15: "runtime", 16: "residency", 17: "race", 18: "validation",
         19: "io", 30: "cuda"}

# exported C-ABI symbols (include/hfb.h); the CPU test checks each one resolves
EXPORTS = [
    "hfb_last_error", "hfb_abi_version", "hfb_create", "hfb_destroy", "hfb_load_program",
    "hfb_set_scalar_i64", "hfb_set_scalar_f64", "hfb_get_scalar_i64", "hfb_get_scalar_f64",
    "hfb_bind_array", "hfb_residency", "hfrt_device_allocate", "hfrt_copy_to_device",
    "hfrt_copy_from_device", "hfb_mark_host_modified", "hfb_run", "hfb_enqueue",
    "hfb_synchronize", "hfb_stream", "hfb_run_graph", "hfb_device_array", "hfk0_diffuse_step",
    "hfk1_diffuse_step", "hfk0_lateral_and_upper_damping", "hfk0_interior_update",
    "hfk0_sf_slab_flx_tile_run", "hfb_decomp_init", "hfb_decomp_faces", "hfb_set_decomposition",
    "hfb_halo_bytes", "hfb_nccl_unique_id", "hfb_profile", "hfb_kernel_time",
    "hfb_group_create", "hfb_group_destroy", "hfb_group_run", "hfb_save_state",
    "hfb_load_state", "hfb_host_array", "hfb_array_checksum", "hfb_run_scenario",
    "hfb_set_reduction_order", "hfb_program_name", "hfb_program_module", "hfb_plugin_prepare",
    "hfb_plugin_written", "hfb_plugin_view", "hfb_plugin_scratch", "hfb_plugin_host", "hfb_plugin_host_ref",
    "hfb_peer_export", "hfb_peer_attach", "hfb_peer_stats", "hfb_transfer_bytes",
    "hfb_set_option", "hfb_variants_build", "hfb_enqueue_graph", "hfb_bind_init",
    "hfb_plugin_array_info", "hfb_plugin_scratch_clear_init", "hfb_plugin_error",
    "hfb_layout_of", "hfb_pack_box_host", "hfb_unpack_box_host",
]

# module of each built-in program (the apps' state modules)
MODULES = {"diffusion": "diff_state", "damping": "svar", "bounded": "b_state",
           "surface_flux": "sf_state", "reduction": "red_state", "dycore": "dyn_state"}


class HfbError(RuntimeError):
    def __init__(self, code, msg):
        self.code = code
        self.kind = KINDS.get(code, "unknown")
        super().__init__(f"[{self.kind}] {msg}")


@dataclass
class LaunchStats:
    launches: int
    threads: int
    guard_returns: int
    native_launches: int


class _Stats(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("threads", ctypes.c_int64),
                ("guard_returns", ctypes.c_int64), ("native_launches", ctypes.c_int64)]


class Decomp(ctypes.Structure):
    _fields_ = [("global_nx", ctypes.c_int64), ("global_ny", ctypes.c_int64),
                ("nz", ctypes.c_int64), ("px", ctypes.c_int32), ("py", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("halo", ctypes.c_int32), ("rx", ctypes.c_int32),
                ("ry", ctypes.c_int32), ("i0", ctypes.c_int64), ("j0", ctypes.c_int64),
                ("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("west", ctypes.c_int32),
                ("east", ctypes.c_int32), ("south", ctypes.c_int32), ("north", ctypes.c_int32)]


_lib = None


def build(verbose=False):
    """Compile the sm_100a kernels + C ABI into paper_1710_08616_b200/libhfb.so."""
    subprocess.run(["make", "-s", "-C", str(CSRC), "-j4"], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        c = ctypes
        P, S, i64, dbl = c.c_void_p, c.c_char_p, c.c_int64, c.c_double
        L.hfb_last_error.restype = S
        L.hfb_create.argtypes = [c.c_int, c.POINTER(P)]
        L.hfb_destroy.argtypes = [P]
        L.hfb_destroy.restype = None
        L.hfb_load_program.argtypes = [P, S]
        L.hfb_set_scalar_i64.argtypes = [P, S, S, i64]
        L.hfb_set_scalar_f64.argtypes = [P, S, S, dbl]
        L.hfb_get_scalar_i64.argtypes = [P, S, S, c.POINTER(i64)]
        L.hfb_get_scalar_f64.argtypes = [P, S, S, c.POINTER(dbl)]
        L.hfb_bind_array.argtypes = [P, S, S, c.c_int, c.POINTER(i64), c.POINTER(i64), P,
                                     c.POINTER(i64), c.c_uint]
        L.hfb_residency.argtypes = [P, S, S, c.POINTER(c.c_int), c.POINTER(c.c_int)]
        for n in ("hfrt_device_allocate", "hfrt_copy_to_device", "hfrt_copy_from_device",
                  "hfb_mark_host_modified"):
            getattr(L, n).argtypes = [P, S, S]
        L.hfb_run.argtypes = [P, S, c.POINTER(_Stats)]
        L.hfb_enqueue.argtypes = [P, S, c.POINTER(_Stats)]
        L.hfb_synchronize.argtypes = [P]
        L.hfb_stream.argtypes = [P]
        L.hfb_stream.restype = P
        L.hfb_run_graph.argtypes = [P, S, i64, c.POINTER(_Stats)]
        L.hfb_enqueue_graph.argtypes = [P, S, i64, c.POINTER(_Stats)]
        L.hfb_decomp_init.argtypes = [c.POINTER(Decomp)]
        L.hfb_decomp_faces.argtypes = [c.POINTER(Decomp), c.c_int32, c.POINTER(i64),
                                       c.POINTER(i64)]
        L.hfb_set_decomposition.argtypes = [P, c.POINTER(Decomp), P]
        L.hfb_halo_bytes.argtypes = [P]
        L.hfb_halo_bytes.restype = i64
        L.hfb_nccl_unique_id.argtypes = [P]
        L.hfb_profile.argtypes = [P, c.c_int]
        L.hfb_kernel_time.argtypes = [P, S, c.POINTER(dbl), c.POINTER(i64)]
        L.hfb_group_create.argtypes = [c.POINTER(P), c.c_int, c.POINTER(P)]
        L.hfb_group_destroy.argtypes = [P]
        L.hfb_group_destroy.restype = None
        L.hfb_group_run.argtypes = [P, S, c.POINTER(_Stats)]
        L.hfb_set_reduction_order.argtypes = [P, c.c_int]
        L.hfb_program_name.argtypes = [P]
        L.hfb_program_name.restype = S
        L.hfb_program_module.argtypes = [P]
        L.hfb_program_module.restype = S
        L.hfb_save_state.argtypes = [P, S]
        L.hfb_load_state.argtypes = [P, S]
        L.hfb_host_array.argtypes = [P, S, S, c.POINTER(c.POINTER(dbl)), c.POINTER(c.c_int),
                                     c.POINTER(i64), c.POINTER(i64), c.POINTER(i64)]
        L.hfb_array_checksum.argtypes = [P, S, S, c.POINTER(dbl), c.POINTER(c.c_uint64)]
        L.hfb_run_scenario.argtypes = [P, S, c.POINTER(_Stats), c.c_char_p, c.c_size_t]
        L.hfb_peer_export.argtypes = [P, P, c.c_size_t, c.POINTER(c.c_size_t)]
        L.hfb_peer_attach.argtypes = [P, c.c_int, c.POINTER(P), c.POINTER(c.c_size_t)]
        L.hfb_peer_stats.argtypes = [P, c.POINTER(i64), c.POINTER(i64)]
        L.hfb_transfer_bytes.argtypes = [P, c.POINTER(i64), c.POINTER(i64)]
        L.hfb_set_option.argtypes = [P, S, S]
        L.hfb_bind_init.argtypes = [P, S, S, P]
        L.hfb_layout_of.argtypes = [i64] * 4 + [c.POINTER(i64)] * 4
        L.hfb_pack_box_host.argtypes = [P, i64, i64, i64, c.POINTER(i64), P]
        L.hfb_unpack_box_host.argtypes = [P, i64, i64, i64, c.POINTER(i64), P]
        L.hfb_variants_build.restype = c.c_int
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise HfbError(rc, lib().hfb_last_error().decode())


def _b(s):
    return s.encode() if isinstance(s, str) else s


def decomp_init(global_nx, global_ny, nz, px, py, rank, halo=2):
    d = Decomp(global_nx, global_ny, nz, px, py, rank, halo)
    _check(lib().hfb_decomp_init(ctypes.byref(d)))
    return d


def decomp_faces(d, side):
    sb = (ctypes.c_int64 * 4)()
    rb = (ctypes.c_int64 * 4)()
    _check(lib().hfb_decomp_faces(ctypes.byref(d), side, sb, rb))
    return tuple(sb), tuple(rb)


class Engine:
    """One context = the reference's (Program, MachineState) pair on one GPU."""

    def __init__(self, app, device=0):
        self.app = app
        self.module = MODULES.get(app, app)
        h = ctypes.c_void_p()
        _check(lib().hfb_create(device, ctypes.byref(h)))
        self._h = h
        self._bound = {}
        if app is not None:
            _check(lib().hfb_load_program(h, _b(str(app))))
            if str(app).endswith(".so"):  # a program generated from .h90 sources (hfc)
                self.app = lib().hfb_program_name(h).decode()
                self.module = lib().hfb_program_module(h).decode()

    @classmethod
    def from_state(cls, path, device=0):
        """A context restored from an HFBSTAT1 image (hfb_load_state): program, scalars
        and arrays (in context-owned host buffers, see array())."""
        eng = cls(None, device)
        try:
            _check(lib().hfb_load_state(eng._h, _b(str(path))))
        except Exception:
            eng.close()
            raise
        from .state import read_header
        eng.app = read_header(path)["program"]
        eng.module = MODULES.get(eng.app, eng.app)
        return eng

    @classmethod
    def scenario(cls, path, device=0):
        """Run a scenario file (hfb_run_scenario): returns (engine, LaunchStats, report);
        a failed expectation raises HfbError('validation')."""
        from .state import Scenario
        sc = Scenario.parse(path)
        eng = cls(None, device)
        st = _Stats()
        buf = ctypes.create_string_buffer(1 << 16)
        rc = lib().hfb_run_scenario(eng._h, _b(str(path)), ctypes.byref(st), buf, len(buf))
        eng.app = sc.program
        eng.module = MODULES.get(sc.program, sc.program)
        if rc != 0:
            msg = lib().hfb_last_error().decode()
            eng.close()
            raise HfbError(rc, msg)
        return eng, LaunchStats(st.launches, st.threads, st.guard_returns,
                                st.native_launches), buf.value.decode()

    def close(self):
        if getattr(self, "_h", None):
            lib().hfb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # --- MachineState --------------------------------------------------------------
    def set(self, name, value):
        if isinstance(value, (int, np.integer)) and not isinstance(value, bool):
            _check(lib().hfb_set_scalar_i64(self._h, _b(self.module), _b(name), int(value)))
        else:
            _check(lib().hfb_set_scalar_f64(self._h, _b(self.module), _b(name), float(value)))

    def get(self, name, integer=False):
        if integer:
            v = ctypes.c_int64()
            _check(lib().hfb_get_scalar_i64(self._h, _b(self.module), _b(name), ctypes.byref(v)))
        else:
            v = ctypes.c_double()
            _check(lib().hfb_get_scalar_f64(self._h, _b(self.module), _b(name), ctypes.byref(v)))
        return v.value

    def bind(self, name, array, lower=None, pin=False):
        """Bind a float64 host array shaped by the declared dims (any dense order)."""
        a = array
        if a.dtype != np.float64:
            raise TypeError("module arrays are real(r_size) = float64")
        rank = a.ndim
        lower = tuple(lower) if lower is not None else (1,) * rank
        upper = tuple(l + n - 1 for l, n in zip(lower, a.shape))
        strides = (ctypes.c_int64 * rank)(*[s // 8 for s in a.strides])
        lo = (ctypes.c_int64 * rank)(*lower)
        hi = (ctypes.c_int64 * rank)(*upper)
        _check(lib().hfb_bind_array(self._h, _b(self.module), _b(name), rank, lo, hi,
                                    a.ctypes.data, strides, 1 if pin else 0))
        self._bound[name] = a  # keep the buffer alive

    def bind_init(self, name, init):
        """Element init flags (uint8, the array's shape and element order) for a bound array
        (hfb_bind_init); kept alive by the engine, written back by copy-outs."""
        if init is None:
            _check(lib().hfb_bind_init(self._h, _b(self.module), _b(name), None))
            self._bound.pop("@init:" + name, None)
            return
        a = self._bound[name]
        if init.dtype != np.uint8 or init.shape != a.shape or init.strides != tuple(
                s // 8 for s in a.strides):
            raise TypeError("init flags must be uint8 with the data array's shape and order")
        _check(lib().hfb_bind_init(self._h, _b(self.module), _b(name), init.ctypes.data))
        self._bound["@init:" + name] = init

    def array(self, name):
        """numpy view (declared bounds' shape, host order) of an array's bound host buffer:
        the caller's, or the context-owned one of a restored state / scenario."""
        p = ctypes.POINTER(ctypes.c_double)()
        rank = ctypes.c_int()
        lo, hi, st = (ctypes.c_int64 * 4)(), (ctypes.c_int64 * 4)(), (ctypes.c_int64 * 4)()
        _check(lib().hfb_host_array(self._h, _b(self.module), _b(name), ctypes.byref(p),
                                    ctypes.byref(rank), lo, hi, st))
        shape = tuple(hi[d] - lo[d] + 1 for d in range(rank.value))
        count = int(np.prod(shape))
        flat = np.ctypeslib.as_array(p, shape=(count,))
        strides = tuple(8 * (st[d] if shape[d] > 1 else 1) for d in range(rank.value))
        return np.lib.stride_tricks.as_strided(flat, shape=shape, strides=strides)

    def set_option(self, key, value):
        """Per-context option (hfb_set_option): "variant" (product | generic | split |
        single_role; tma | ws2 in the A/B build), "overlap" ("0" | "1")."""
        _check(lib().hfb_set_option(self._h, _b(key), _b(str(value))))

    def set_reduction_order(self, ordered=True):
        """Ordered reductions: bit-identical to the reference's acc-simulated order
        (hfb_set_reduction_order); default is the fast tree (1e-12 relative)."""
        _check(lib().hfb_set_reduction_order(self._h, 1 if ordered else 0))

    def save_state(self, path):
        """HFBSTAT1 image of the MachineState (hfb_save_state); newest copies, residency
        unchanged."""
        _check(lib().hfb_save_state(self._h, _b(str(path))))

    def load_state(self, path):
        _check(lib().hfb_load_state(self._h, _b(str(path))))

    def checksum(self, name):
        """(fp64 sum, FNV-1a 64 of the bits) of an array's newest copy, ArrayValue order."""
        s, b = ctypes.c_double(), ctypes.c_uint64()
        _check(lib().hfb_array_checksum(self._h, _b(self.module), _b(name), ctypes.byref(s),
                                        ctypes.byref(b)))
        return s.value, b.value

    # --- transfers (hfrt_*) -----------------------------------------------------------
    def device_allocate(self, name):
        _check(lib().hfrt_device_allocate(self._h, _b(self.module), _b(name)))

    def copy_to_device(self, name):
        _check(lib().hfrt_copy_to_device(self._h, _b(self.module), _b(name)))

    def copy_from_device(self, name):
        _check(lib().hfrt_copy_from_device(self._h, _b(self.module), _b(name)))

    def mark_host_modified(self, name):
        _check(lib().hfb_mark_host_modified(self._h, _b(self.module), _b(name)))

    def residency(self, name):
        r, d = ctypes.c_int(), ctypes.c_int()
        _check(lib().hfb_residency(self._h, _b(self.module), _b(name), ctypes.byref(r),
                                   ctypes.byref(d)))
        return ("host", "device", "both")[r.value], bool(d.value)

    # --- entries ------------------------------------------------------------------
    def run(self, entry="main"):
        st = _Stats()
        _check(lib().hfb_run(self._h, _b(entry), ctypes.byref(st)))
        return LaunchStats(st.launches, st.threads, st.guard_returns, st.native_launches)

    def enqueue(self, entry):
        st = _Stats()
        _check(lib().hfb_enqueue(self._h, _b(entry), ctypes.byref(st)))
        return LaunchStats(st.launches, st.threads, st.guard_returns, st.native_launches)

    def run_graph(self, entry, steps):
        st = _Stats()
        _check(lib().hfb_run_graph(self._h, _b(entry), int(steps), ctypes.byref(st)))
        return LaunchStats(st.launches, st.threads, st.guard_returns, st.native_launches)

    def enqueue_graph(self, entry, steps):
        """Launch (without synchronising) the cached CUDA graph of `steps` steps."""
        st = _Stats()
        _check(lib().hfb_enqueue_graph(self._h, _b(entry), int(steps), ctypes.byref(st)))
        return LaunchStats(st.launches, st.threads, st.guard_returns, st.native_launches)

    def synchronize(self):
        _check(lib().hfb_synchronize(self._h))

    @property
    def stream(self):
        return lib().hfb_stream(self._h)

    def set_decomposition(self, d, nccl_id=None):
        buf = None
        if nccl_id is not None:
            buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        _check(lib().hfb_set_decomposition(self._h, ctypes.byref(d), buf))

    def peer_export(self):
        """This rank's peer-transport blob (CUDA IPC handles of its device buffers)."""
        n = ctypes.c_size_t()
        _check(lib().hfb_peer_export(self._h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        _check(lib().hfb_peer_export(self._h, buf, n.value, ctypes.byref(n)))
        return buf.raw[:n.value]

    def peer_attach(self, blobs):
        """Map every rank's blob (all ranks, in any order) and switch to the peer transport."""
        keep = [ctypes.create_string_buffer(bytes(b), len(b)) for b in blobs]
        ptrs = (ctypes.c_void_p * len(keep))(*[ctypes.addressof(k) for k in keep])
        lens = (ctypes.c_size_t * len(keep))(*[len(b) for b in blobs])
        _check(lib().hfb_peer_attach(self._h, len(keep), ptrs, lens))

    def attach_peers(self, group=None):
        """Collective over torch.distributed: export, all-gather, attach, barrier."""
        import torch.distributed as dist
        mine = self.peer_export()
        blobs = [None] * dist.get_world_size(group)
        dist.all_gather_object(blobs, mine, group=group)
        self.peer_attach(blobs)
        dist.barrier(group)

    def transfer_bytes(self):
        """(host->device, device->host) bytes this context transferred so far"""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().hfb_transfer_bytes(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def peer_stats(self):
        """(halo updates by push kernel, halo updates handed off by the step epilogue)"""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().hfb_peer_stats(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def halo_bytes(self):
        return lib().hfb_halo_bytes(self._h)

    def profile(self, enable=True, clear=False):
        """CUDA-event timing of every native launch (on the context stream)."""
        _check(lib().hfb_profile(self._h, -1 if clear else (1 if enable else 0)))

    def kernel_time(self, kernel):
        """(total device ms, launches) accumulated for one native kernel."""
        ms, n = ctypes.c_double(), ctypes.c_int64()
        _check(lib().hfb_kernel_time(self._h, _b(kernel), ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value


class Group:
    """In-process rank group (hfb_group_*): every rank's Engine on this host thread, halos
    exchanged by device copies. Engines must carry decomposition ranks 0..n-1."""

    def __init__(self, engines):
        self.engines = list(engines)
        arr = (ctypes.c_void_p * len(self.engines))(*[e._h.value for e in self.engines])
        h = ctypes.c_void_p()
        _check(lib().hfb_group_create(arr, len(self.engines), ctypes.byref(h)))
        self._h = h

    def run(self, entry="main"):
        st = _Stats()
        _check(lib().hfb_group_run(self._h, _b(entry), ctypes.byref(st)))
        return LaunchStats(st.launches, st.threads, st.guard_returns, st.native_launches)

    def close(self):
        if getattr(self, "_h", None):
            lib().hfb_group_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class TileLayout:
    """The device layout of an (nk, nj, ni) array (hfb_layout_of) on a host buffer, with the
    library's host twins of the halo pack / unpack kernels."""

    def __init__(self, ni, nj, nk, nl=1):
        v = [ctypes.c_int64() for _ in range(4)]
        _check(lib().hfb_layout_of(ni, nj, nk, nl, *[ctypes.byref(x) for x in v]))
        self.ni, self.nj, self.nk = ni, nj, nk
        self.pitch, self.plane, self.alloc, self.origin = (x.value for x in v)
        self.buf = np.zeros(self.alloc)

    def interior(self):
        """(nk, nj, ni) view of the logical elements (i fastest)."""
        v = self.buf[self.origin:self.origin + self.nk * self.plane]
        return np.lib.stride_tricks.as_strided(
            v, shape=(self.nk, self.nj, self.ni), strides=(8 * self.plane, 8 * self.pitch, 8))

    def padded(self, h):
        """(nk, nj + 2h, ni + 2h) view including h cells of the halo ring (h <= 2)."""
        start = self.origin - h * self.pitch - h
        v = self.buf[start:]
        return np.lib.stride_tricks.as_strided(
            v, shape=(self.nk, self.nj + 2 * h, self.ni + 2 * h),
            strides=(8 * self.plane, 8 * self.pitch, 8))

    def _ptr(self):
        return self.buf.ctypes.data + 8 * self.origin

    def pack(self, box):
        n = (box[1] - box[0] + 1) * (box[3] - box[2] + 1) * self.nk
        out = np.empty(max(n, 0))
        b = (ctypes.c_int64 * 4)(*box)
        _check(lib().hfb_pack_box_host(self._ptr(), self.pitch, self.plane, self.nk, b,
                                       out.ctypes.data))
        return out

    def unpack(self, box, data):
        data = np.ascontiguousarray(data, dtype=np.float64)
        b = (ctypes.c_int64 * 4)(*box)
        _check(lib().hfb_unpack_box_host(self._ptr(), self.pitch, self.plane, self.nk, b,
                                         data.ctypes.data))


def variants_build():
    """True when the loaded library is the A/B build (libhfb_variants.so)."""
    return bool(lib().hfb_variants_build())


def nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    _check(lib().hfb_nccl_unique_id(buf))
    return buf.raw


def run_gpu(app, scalars, arrays, entry="main", device=0, lower=None):
    """run_gpu_simulated(program, state, entry) analogue: runs `entry` of `app` with the
    given module scalars and host arrays (updated in place); returns (LaunchStats, scalars)."""
    with Engine(app, device) as eng:
        for k, v in scalars.items():
            eng.set(k, v)
        for k, a in arrays.items():
            eng.bind(k, a, lower=(lower or {}).get(k))
        stats = eng.run(entry)
        out = {}
        for k, v in scalars.items():
            out[k] = eng.get(k, integer=isinstance(v, (int, np.integer)))
        return stats, out
