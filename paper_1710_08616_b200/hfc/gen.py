"""sm_100a CUDA C++ generator for Hybrid-Fortran programs.

The reference's backend emits CUDA-Fortran text (codegen.cpp:397-519) that nothing here
can compile; this one emits a CUDA C++ translation unit for B200 that libhfb.so loads as
a *program plugin* (include/hfb_plugin.h): every `@parallelRegion` becomes a `__global__`
kernel with the reference's launch contract (one thread per (i,j) point of the region,
block 32 x 4, guard `it > end`, codegen.cpp:421-512), called subroutines become
`__device__` functions, routines become host drivers (sequential statements, loops,
calls, `transferHere` copy-in/out, codegen.cpp:570-600), and module arrays live in the
engine's I-fastest device layout. Dimension extension follows analysis.cpp:439-527:
routine-local arrays bound to the region domain (`domName`) get the domain dims
prepended and, like the reference's generated code, are materialised as device arrays.

Arithmetic is emitted in the reference interpreter's semantics (interp.cpp:617-770):
int64 integers, binary64 reals, one rounding per operation in the parsed
(left-associative) order, no FMA (compiled with -fmad=false), integer exponents by
repeated multiplication from 1.0, `min`/`max` as the interpreter's left fold, real
literals as exact hex floats. Reductions (`reduce`) are not generated (the CUDA-style
backend of the reference rejects them too, codegen.cpp:399-403).
"""
import hashlib
from dataclasses import dataclass, field

from .parse import (Assign, Bin, Call, Decl, Do, If, Logical, Name, Num, ParseError, Ref,
                    Return, Stop,
                    Region, Un, parse_expr, parse_program)

ROLE_I, ROLE_J, ROLE_K, ROLE_L = 0, 1, 2, 3
INTRINSICS = {"sqrt", "abs", "min", "max", "real", "ceiling"}


class GenError(ValueError):
    pass


def lit_real(text):
    return float(text).hex()


@dataclass
class ArrInfo:
    name: str
    decl: Decl
    scope: str            # 'module' | 'local' | 'extended'
    roles: list = field(default_factory=list)
    dims: list = field(default_factory=list)   # [(lo_expr, hi_expr)] after extension
    key: str = ""


class Program:
    def __init__(self, sources, name):
        self.name = name
        self.mods = parse_program(sources)
        state = [m for m in self.mods.values() if m.decls]
        if len(state) != 1:
            raise GenError("exactly one module with declarations (the state module) is "
                           f"supported, found {[m.name for m in state]}")
        self.state = state[0]
        # module parameters are constants (inlined, not part of the MachineState)
        self.params = {n: d for n, d in self.state.decls.items() if d.param is not None}
        for n in self.params:
            del self.state.decls[n]
        self.routines = {}
        for m in self.mods.values():
            for r in m.routines.values():
                if r.name in self.routines:
                    raise GenError(f"routine {r.name} defined twice")
                self.routines[r.name] = r
        # target selection (SPEC §3.1 appliesTo): regions that do not apply to the GPU are
        # not parallel regions of this target; their bodies run as ordinary statements
        gpu = _gpu_routines(self.routines)
        for r in self.routines.values():
            r.body = _gpu_target(r.body, self.routines, gpu)
        for n, d in self.state.decls.items():
            if d.type == "dim3":
                raise GenError("type(dim3) module objects are not supported")
            if d.dims and d.type != "real":
                raise GenError(f"module array {n}: only real(r_size) arrays are supported")
            for lo, hi in d.dims:
                for e in (lo, hi):
                    if isinstance(e, Name) and e.name in self.params:
                        continue
                    if not isinstance(e, (Num, Name)):
                        raise GenError(f"module array {n}: dims must be literals or scalar "
                                       "names (the engine evaluates them)")
        self.device_routines = set()
        self._classify()
        self.module_roles = self._module_roles()

    # -- which routines run inside kernels (called from a region) ----------------------
    def _classify(self):
        def calls_in(stmts, acc):
            for s in stmts:
                if isinstance(s, Call):
                    acc.add(s.name)
                elif isinstance(s, Do):
                    calls_in(s.body, acc)
                elif isinstance(s, If):
                    for _, b in s.branches:
                        calls_in(b, acc)
                elif isinstance(s, Region):
                    calls_in(s.body, acc)
            return acc

        def regions_calls(stmts, acc):
            for s in stmts:
                if isinstance(s, Region):
                    calls_in(s.body, acc)
                elif isinstance(s, Do):
                    regions_calls(s.body, acc)
                elif isinstance(s, If):
                    for _, b in s.branches:
                        regions_calls(b, acc)
            return acc

        dev = set()
        for r in self.routines.values():
            regions_calls(r.body, dev)
        frontier = list(dev)
        while frontier:
            n = frontier.pop()
            if n not in self.routines:
                raise GenError(f"call of unknown routine {n}")
            for c in calls_in(self.routines[n].body, set()):
                if c not in dev:
                    dev.add(c)
                    frontier.append(c)
        self.device_routines = dev

    # -- I/J/K/L roles of module arrays from region subscripts -------------------------
    def _module_roles(self):
        found = {}

        def visit_expr(e, it):
            if isinstance(e, Ref):
                if e.name in self.state.decls and self.state.decls[e.name].dims:
                    roles = []
                    for a in e.args:
                        v = _iter_of(a, it)
                        roles.append(v)
                    found.setdefault(e.name, []).append(roles)
                for a in e.args:
                    visit_expr(a, it)
            elif isinstance(e, Bin):
                visit_expr(e.a, it)
                visit_expr(e.b, it)
            elif isinstance(e, Un):
                visit_expr(e.x, it)

        def visit(stmts, it):
            for s in stmts:
                if isinstance(s, Assign):
                    visit_expr(s.lhs, it)
                    visit_expr(s.rhs, it)
                elif isinstance(s, Do):
                    visit(s.body, it)
                elif isinstance(s, If):
                    for c, b in s.branches:
                        if c is not None:
                            visit_expr(c, it)
                        visit(b, it)
                elif isinstance(s, Region):
                    names = [n.lower() for n in s.attrs.get("domname", [])]
                    visit(s.body, names)
                elif isinstance(s, Call):
                    for a in s.args:
                        visit_expr(a, it)

        for r in self.routines.values():
            visit(r.body, [])
        roles = {}
        for n, d in self.state.decls.items():
            if not d.dims:
                continue
            rank = len(d.dims)
            rl = None
            for acc in found.get(n, []):
                cand = [None] * rank
                for pos, v in enumerate(acc):
                    if v == 0:
                        cand[pos] = ROLE_I
                    elif v == 1:
                        cand[pos] = ROLE_J
                if ROLE_I in cand or ROLE_J in cand:
                    rl = cand
                    break
            if rl is None:  # never indexed by a domain iterator: last two dims are (i, j)
                rl = [None] * rank
                if rank >= 2:
                    rl[rank - 2], rl[rank - 1] = ROLE_I, ROLE_J
                else:
                    rl[0] = ROLE_I
            rest = [ROLE_K, ROLE_L]
            for p in range(rank):
                if rl[p] is None:
                    if not rest:
                        raise GenError(f"array {n}: too many non-domain dims")
                    rl[p] = rest.pop(0)
            roles[n] = rl
        return roles


def _applies_gpu(s):
    applies = [x.lower() for x in s.attrs.get("appliesto", [])]
    return not applies or "gpu" in applies


def region_bounds(s):
    """(lower, upper) expressions per domain dimension (codegen.cpp:38-63)."""
    lo, hi = [], []
    for sz in s.attrs.get("domsize", []):
        if ":" in sz:
            a, b = sz.split(":")
            lo.append(parse_expr(a, s.line))
            hi.append(parse_expr(b, s.line))
        else:
            lo.append(Num("1", False))
            hi.append(parse_expr(sz, s.line))
    if "startat" in s.attrs:
        lo = [parse_expr(x, s.line) for x in s.attrs["startat"]]
    if "endat" in s.attrs:
        hi = [parse_expr(x, s.line) for x in s.attrs["endat"]]
    return lo, hi


def _walk(stmts):
    for s in stmts:
        yield s
        if isinstance(s, (Region, Do)):
            yield from _walk(s.body)
        elif isinstance(s, If):
            for _, b in s.branches:
                yield from _walk(b)


def _gpu_routines(routines):
    """Routines with GPU regions in scope: their own, or through the routines they call."""
    gpu = {n for n, r in routines.items()
           if any(isinstance(s, Region) and _applies_gpu(s) for s in _walk(r.body))}
    changed = True
    while changed:
        changed = False
        for n, r in routines.items():
            if n not in gpu and any(isinstance(s, Call) and s.name in gpu for s in _walk(r.body)):
                gpu.add(n)
                changed = True
    return gpu


def _gpu_target(stmts, routines, gpu):
    """GPU-target lowering of regions that do not apply to the GPU (codegen.cpp:297-312): a
    CPU-only region over code that launches its own kernels runs its body once with the
    iterators pinned to the region start; any other becomes plain host loops, the last
    domain outermost (codegen.cpp:335-359)."""
    out = []
    for s in stmts:
        if isinstance(s, Region):
            s.body = _gpu_target(s.body, routines, gpu)
            if not _applies_gpu(s):
                names = [n.lower() for n in s.attrs.get("domname", [])]
                lo, hi = region_bounds(s)
                covers = any((isinstance(t, Region) and _applies_gpu(t)) or
                             (isinstance(t, Call) and t.name in gpu) for t in _walk(s.body))
                if covers:
                    out += [Assign(Name(n), e, s.line) for n, e in zip(names, lo)]
                    out += s.body
                else:
                    body = s.body
                    for n, a, b in zip(names, lo, hi):  # innermost first
                        body = [Do(n, a, b, body, s.line)]
                    out += body
                continue
        elif isinstance(s, Do):
            s.body = _gpu_target(s.body, routines, gpu)
        elif isinstance(s, If):
            s.branches = [(c, _gpu_target(b, routines, gpu)) for c, b in s.branches]
        out.append(s)
    return out


def _iter_of(e, iters):
    """index of the domain iterator an index expression is (iterator +- constant)"""
    if isinstance(e, Name) and e.name in iters:
        return iters.index(e.name)
    if isinstance(e, Bin) and e.op in ("+", "-") and isinstance(e.a, Name) and e.a.name in iters \
            and isinstance(e.b, Num):
        return iters.index(e.a.name)
    return None


# ---- expression emitter ----------------------------------------------------------------
class Scope:
    """names visible to generated code: each maps to (kind, type, c_expr)"""

    def __init__(self, parent=None):
        self.names = {}
        self.parent = parent

    def get(self, n):
        s = self
        while s is not None:
            if n in s.names:
                return s.names[n]
            s = s.parent
        return None

    def set(self, n, kind, typ, cexpr):
        self.names[n] = (kind, typ, cexpr)


class Emitter:
    def __init__(self, prog):
        self.p = prog
        self.nids = {}  # array name -> id in kNames (checked accessors)
        self.used_idiv = False

    def nid(self, name):
        return self.nids.setdefault(name, len(self.nids))

    def etype(self, e, sc):
        if isinstance(e, Num):
            return "real" if e.is_real else "int"
        if isinstance(e, Logical):
            return "logical"
        if isinstance(e, Name):
            v = sc.get(e.name)
            if v is None:
                raise GenError(f"unknown name {e.name}")
            return v[1]
        if isinstance(e, Ref):
            v = sc.get(e.name)
            if v is not None and v[0] in ("array", "xarray", "harray"):
                return "real"
            if e.name in ("sqrt", "real"):
                return "real"
            if e.name == "ceiling":
                return "int"
            if e.name == "abs":
                return self.etype(e.args[0], sc)
            if e.name in ("min", "max"):
                return "int" if all(self.etype(a, sc) == "int" for a in e.args) else "real"
            raise GenError(f"unknown function or undeclared array {e.name}")
        if isinstance(e, Un):
            return "logical" if e.op == ".not." else self.etype(e.x, sc)
        if isinstance(e, Bin):
            if e.op in (".and.", ".or.", ".eq.", ".ne.", ".lt.", ".le.", ".gt.", ".ge."):
                return "logical"
            ta, tb = self.etype(e.a, sc), self.etype(e.b, sc)
            if e.op == "**":
                if tb == "int":
                    return ta
                return "real"
            return "int" if ta == "int" and tb == "int" else "real"
        raise GenError(f"unsupported expression {e}")

    def real(self, e, sc):
        c = self.expr(e, sc)
        return c if self.etype(e, sc) == "real" else f"static_cast<double>({c})"

    def expr(self, e, sc):
        if isinstance(e, Num):
            return f"{lit_real(e.text)}" if e.is_real else f"INT64_C({int(e.text)})"
        if isinstance(e, Logical):
            return "true" if e.value else "false"
        if isinstance(e, Name):
            v = sc.get(e.name)
            if v is None:
                raise GenError(f"unknown name {e.name}")
            if v[0] in ("array", "xarray", "harray"):
                raise GenError(f"array {e.name} used without subscripts")
            return v[2]
        if isinstance(e, Ref):
            v = sc.get(e.name)
            if v is not None and v[0] in ("array", "xarray", "harray"):
                write = bool(sc.get("@write"))
                if write:  # subscripts are reads
                    sc.names.pop("@write")
                idx = [self.expr(a, sc) if self.etype(a, sc) == "int"
                       else f"static_cast<int64_t>({self.expr(a, sc)})" for a in e.args]
                if write:
                    sc.set("@write", "meta", "", True)
                if v[0] == "xarray":  # extended local: domain iterators prepended
                    idx = list(sc.get("@iters")[2]) + idx
                acc = "HFC_WR" if write else "HFC_RD"
                nm = self.nid(e.name)
                if v[0] == "harray":  # host code: the bound host buffer (cached reference)
                    fn = "hfc_wr" if write else "hfc_rd"
                    view = f"{fn}(R, {sc.get('@href:' + e.name)[2]}, {v[2]})"
                    return f"{acc}({view}, {nm}, {', '.join(idx)})"
                return f"{acc}({v[2]}, {nm}, {', '.join(idx)})"
            return self.intrinsic(e, sc)
        if isinstance(e, Un):
            if e.op == ".not.":
                return f"(!{self.expr(e.x, sc)})"
            if e.op == "+":
                return self.expr(e.x, sc)
            return f"(-{self.expr(e.x, sc)})"
        if isinstance(e, Bin):
            op = e.op
            if op in (".and.", ".or."):
                c = "&&" if op == ".and." else "||"
                return f"({self.expr(e.a, sc)} {c} {self.expr(e.b, sc)})"
            ta, tb = self.etype(e.a, sc), self.etype(e.b, sc)
            if op in (".eq.", ".ne.", ".lt.", ".le.", ".gt.", ".ge."):
                c = {".eq.": "==", ".ne.": "!=", ".lt.": "<", ".le.": "<=", ".gt.": ">",
                     ".ge.": ">="}[op]
                if ta == "int" and tb == "int":
                    return f"({self.expr(e.a, sc)} {c} {self.expr(e.b, sc)})"
                return f"({self.real(e.a, sc)} {c} {self.real(e.b, sc)})"
            if op == "**":
                if tb == "int":
                    if ta == "int":
                        return f"hfc_ipowi({self.expr(e.a, sc)}, {self.expr(e.b, sc)})"
                    return f"hfc_powi({self.real(e.a, sc)}, {self.expr(e.b, sc)})"
                # the reference evaluates real exponents with the host's std::pow
                # (interp.cpp:745), which device pow() matches only to 2 ulp: refused
                # rather than silently breaking bit-exactness
                raise GenError("real exponent in '**': only integer exponents are supported "
                               "(device pow differs from the reference's std::pow)")
            if ta == "int" and tb == "int":
                if op == "/":
                    self.used_idiv = True
                    return f"hfc_idiv({self.expr(e.a, sc)}, {self.expr(e.b, sc)})"
                return f"({self.expr(e.a, sc)} {op} {self.expr(e.b, sc)})"
            return f"({self.real(e.a, sc)} {op} {self.real(e.b, sc)})"
        raise GenError(f"unsupported expression {e}")

    def intrinsic(self, e, sc):
        n, a = e.name, e.args
        if n == "sqrt":
            return f"sqrt({self.real(a[0], sc)})"
        if n == "real":
            return self.real(a[0], sc)
        if n == "ceiling":
            return f"static_cast<int64_t>(ceil({self.real(a[0], sc)}))"
        if n == "abs":
            if self.etype(a[0], sc) == "int":
                return f"hfc_iabs({self.expr(a[0], sc)})"
            return f"fabs({self.real(a[0], sc)})"
        if n in ("min", "max"):
            if len(a) < 2:
                raise GenError("min/max need at least two arguments")
            cmp = "<" if n == "min" else ">"
            if all(self.etype(x, sc) == "int" for x in a):
                acc = self.expr(a[0], sc)
                for x in a[1:]:
                    acc = f"hfc_fold_i({acc}, {self.expr(x, sc)}, {int(n == 'min')})"
                return acc
            acc = self.real(a[0], sc)  # interp.cpp:630-645: compare as reals, keep first
            for x in a[1:]:
                acc = f"hfc_fold_r({acc}, {self.real(x, sc)}, {int(n == 'min')})"
            return acc
        raise GenError(f"unknown function or undeclared array {n}")


# ---- code generation -------------------------------------------------------------------
PRELUDE = r"""
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <cuda_runtime.h>
#include "hfb.h"
#include "hfb_plugin.h"

namespace {

// Runtime errors of the program (the reference's rt_fail, interp.cpp:68-70): device code
// records the first one here, the host driver turns it into HFB_RUNTIME with the
// reference's text after the launch (checked builds) or at the end of the run.
struct HfcErr {
  int code;  // 1 index out of bounds, 2 read of an unset element, 3 integer division by 0
  int name, dim;
  long long idx, lo, hi;
};
__device__ HfcErr hfc_err;
__device__ double hfc_trash;  // target of out-of-bounds writes (the error is recorded)
__device__ __forceinline__ void hfc_report(int code, int name, int dim, long long idx,
                                           long long lo, long long hi) {
  if (atomicCAS(&hfc_err.code, 0, code) == 0) {
    hfc_err.name = name;
    hfc_err.dim = dim;
    hfc_err.idx = idx;
    hfc_err.lo = lo;
    hfc_err.hi = hi;
  }
}
struct HfcFail {  // a host-side runtime error: the run ends with this status and text
  int status;
  char msg[256];
};
extern const char* const kNames[];  // array names by id (checked accessors)
inline HfcFail hfc_fail_msg(int code, int name, int dim, long long idx, long long lo,
                            long long hi) {
  HfcFail f{HFB_RUNTIME, {0}};
  if (code == 1)
    std::snprintf(f.msg, sizeof f.msg, "index %lld out of bounds [%lld, %lld] in dimension %d of '%s'",
                  idx, lo, hi, dim, kNames[name]);
  else if (code == 2)
    std::snprintf(f.msg, sizeof f.msg, "read of unset element of '%s'", kNames[name]);
  else
    std::snprintf(f.msg, sizeof f.msg, "integer division by zero");
  return f;
}
__host__ __device__ inline void hfc_fail(int code, int name, int dim, long long idx, long long lo,
                                         long long hi) {
#ifdef __CUDA_ARCH__
  hfc_report(code, name, dim, idx, lo, hi);
#else
  throw hfc_fail_msg(code, name, dim, idx, lo, hi);
#endif
}

struct HArr {  // device view: element(d0..d3) = o[sum (d - lo) * s]
  double* o;
  int64_t s[4];
  int64_t lo[4];
#ifdef HFC_CHECKED
  // checked build (hfc --checked): declared upper bounds and the element init flags (device
  // views: the device copy's; host views: the caller's, or none)
  int64_t hi[4];
  uint8_t* init;
  __host__ __device__ int64_t off(int nm, int n, const int64_t* x) const {
    int64_t f = 0;
    for (int d = 0; d < n; ++d) {
      if (x[d] < lo[d] || x[d] > hi[d]) {  // interp.cpp:487-492
        hfc_fail(1, nm, d + 1, x[d], lo[d], hi[d]);
        return -1;
      }
      f += (x[d] - lo[d]) * s[d];
    }
    return f;
  }
  template <class... I>
  __host__ __device__ double rd(int nm, I... i) const {
    const int64_t x[] = {static_cast<int64_t>(i)...};
    const int64_t f = off(nm, static_cast<int>(sizeof...(I)), x);
    if (f < 0) return 0.0;
    if (init && !init[f]) {  // interp.cpp:505-507
      hfc_fail(2, nm, 0, 0, 0, 0);
      return 0.0;
    }
    return o[f];
  }
  template <class... I>
  __host__ __device__ double& wr(int nm, I... i) const {
    const int64_t x[] = {static_cast<int64_t>(i)...};
    const int64_t f = off(nm, static_cast<int>(sizeof...(I)), x);
#ifdef __CUDA_ARCH__
    if (f < 0) return hfc_trash;
#endif
    if (init) init[f] = 1;  // write_element sets the flag (interp.cpp:534)
    return o[f];
  }
#endif
  __host__ __device__ __forceinline__ double& at(int64_t a) const { return o[(a - lo[0]) * s[0]]; }
  __host__ __device__ __forceinline__ double& at(int64_t a, int64_t b) const {
    return o[(a - lo[0]) * s[0] + (b - lo[1]) * s[1]];
  }
  __host__ __device__ __forceinline__ double& at(int64_t a, int64_t b, int64_t c) const {
    return o[(a - lo[0]) * s[0] + (b - lo[1]) * s[1] + (c - lo[2]) * s[2]];
  }
  __host__ __device__ __forceinline__ double& at(int64_t a, int64_t b, int64_t c, int64_t d) const {
    return o[(a - lo[0]) * s[0] + (b - lo[1]) * s[1] + (c - lo[2]) * s[2] + (d - lo[3]) * s[3]];
  }
};

// interp.cpp:732-745: integer exponent by repeated multiplication from 1.0
__host__ __device__ __forceinline__ double hfc_powi(double b, int64_t n) {
  double acc = 1.0;
  const int64_t m = n < 0 ? -n : n;
  for (int64_t k = 0; k < m; ++k) acc *= b;
  return n < 0 ? 1.0 / acc : acc;
}
__host__ __device__ __forceinline__ int64_t hfc_ipowi(int64_t b, int64_t n) {
  int64_t acc = 1;
  for (int64_t k = 0; k < n; ++k) acc *= b;
  return acc;
}
// integer division; by zero: the reference's runtime error (interp.cpp:754)
__host__ __device__ __forceinline__ int64_t hfc_idiv(int64_t a, int64_t b) {
  if (b == 0) {
    hfc_fail(3, 0, 0, 0, 0, 0);
    return 0;
  }
  return a / b;
}
#ifdef HFC_CHECKED
#define HFC_RD(v, nm, ...) (v).rd(nm, __VA_ARGS__)
#define HFC_WR(v, nm, ...) (v).wr(nm, __VA_ARGS__)
#else
#define HFC_RD(v, nm, ...) (v).at(__VA_ARGS__)
#define HFC_WR(v, nm, ...) (v).at(__VA_ARGS__)
#endif
__host__ __device__ __forceinline__ int64_t hfc_iabs(int64_t a) { return a < 0 ? -a : a; }
// interp.cpp:630-645: min/max fold, the later value replaces only on strict improvement
__host__ __device__ __forceinline__ double hfc_fold_r(double best, double d, int is_min) {
  return (is_min ? d < best : d > best) ? d : best;
}
__host__ __device__ __forceinline__ int64_t hfc_fold_i(int64_t best, int64_t d, int is_min) {
  return (is_min ? d < best : d > best) ? d : best;
}

struct Run {
  hfb_ctx* ctx;
  hfb_launch_stats* st;
  cudaStream_t stream;
  int allow_transfers;
  int rc = HFB_OK;
  unsigned long long* ret = nullptr;  // kernel threads that left through a `return`
};
struct HfcStop {  // `stop`: the run ends normally (interp.cpp StopSignal)
  int code;
};

#define HFC_CHECK(call)                       \
  do {                                        \
    int rc_ = (call);                         \
    if (rc_ != HFB_OK) throw rc_;             \
  } while (0)

// reduce(...) regions: the partials in linear-id order combined from the initial value, one
// at a time (interp.cpp:1163-1173), by one thread
__global__ void hfc_ordered(const double* __restrict__ p, int64_t n, double init, int is_mul,
                            double* __restrict__ out) {
  double acc = init;
  for (int64_t t = 0; t < n; ++t) acc = is_mul ? acc * p[t] : acc + p[t];
  *out = acc;
}

HArr hfc_view(const hfb_view& v) {
  HArr a;
  a.o = v.origin;
  for (int d = 0; d < 4; ++d) {
    a.s[d] = v.stride[d];
    a.lo[d] = v.lower[d];
  }
#ifdef HFC_CHECKED
  for (int d = 0; d < 4; ++d) a.hi[d] = INT64_MAX;
  a.init = nullptr;
#endif
  return a;
}

}  // namespace
"""


def _names_in(stmts, acc, calls):
    def ex(e):
        if isinstance(e, Name):
            acc.add(e.name)
        elif isinstance(e, Ref):
            acc.add(e.name)
            for a in e.args:
                ex(a)
        elif isinstance(e, Bin):
            ex(e.a)
            ex(e.b)
        elif isinstance(e, Un):
            ex(e.x)

    for s in stmts:
        if isinstance(s, Assign):
            ex(s.lhs)
            ex(s.rhs)
        elif isinstance(s, Do):
            ex(s.lo)
            ex(s.hi)
            _names_in(s.body, acc, calls)
        elif isinstance(s, If):
            for c, b in s.branches:
                if c is not None:
                    ex(c)
                _names_in(b, acc, calls)
        elif isinstance(s, Call):
            calls.add(s.name)
            for a in s.args:
                ex(a)
        elif isinstance(s, Region):
            _names_in(s.body, acc, calls)
    return acc


class Gen:
    def mod_scalars_of(self, stmts, extra_exprs=(), local_names=()):
        """module scalars a region / device routine reads, through its device calls"""
        names, calls = set(), set()
        _names_in(stmts, names, calls)
        for e in extra_exprs:
            _names_in([Assign(Name("@"), e, 0)], names, calls)
        seen = set()
        while calls:
            c = calls.pop()
            if c in seen or c not in self.p.routines:
                continue
            seen.add(c)
            r = self.p.routines[c]
            sub = set()
            _names_in(r.body, sub, calls)
            names |= {n for n in sub if n not in r.decls and n not in r.args}
        mods = [n for n, d in self.p.state.decls.items() if not d.dims]
        return [n for n in mods if n in names and n not in local_names]

    def __init__(self, prog):
        self.p = prog
        self.em = Emitter(prog)
        self.kernels = []
        self.devfns = []
        self.hostfns = []
        self.kcount = {}
        self.routine_transfers = {}
        self.extended = set()
        self.rt_names = {}
        self.dev_mod_sc = {}

    # -- scopes ----------------------------------------------------------------------------
    def module_scope(self, sc, host):
        for n, d in self.p.params.items():
            sc.set(n, "const", d.type, self.em.expr(d.param, Scope()))
        for n, d in self.p.state.decls.items():
            if d.dims:
                continue
            t = d.type
            if host:
                getter = "hfc_geti" if t == "int" else "hfc_getr" if t == "real" else "hfc_getl"
                sc.set(n, "mscalar", t, f"{getter}(R, \"{n}\")")
            else:
                sc.set(n, "mscalar", t, f"m_{n}")

    def local_arrays(self, r):
        """routine-local arrays: (name -> (decl, extended_dims or None))"""
        ext = {}
        for dd in r.domdeps:
            dn = dd.attrs.get("domname")
            ds = dd.attrs.get("domsize")
            for n in dd.names:
                ext[n] = (dn, ds)
        out = {}
        for n, d in r.decls.items():
            if not d.dims or n in r.args:
                continue
            if d.type != "real":
                raise GenError(f"{r.name}: local array {n} must be real(r_size)")
            if n in ext and ext[n][0]:
                dn, ds = ext[n]
                pre = []
                for s in ds:
                    if ":" in s:
                        lo, hi = s.split(":")
                        pre.append((parse_expr(lo, 0), parse_expr(hi, 0)))
                    else:
                        pre.append((Num("1", False), parse_expr(s, 0)))
                out[n] = (d, pre + list(d.dims), True, [x.lower() for x in dn])
            else:
                out[n] = (d, list(d.dims), False, None)
        return out

    # -- device routines (called inside regions) --------------------------------------------
    def gen_devfn(self, r):
        sc = Scope()
        self.module_scope(sc, host=False)
        params = []
        for a in r.args:
            d = r.decls.get(a)
            if d is None or d.dims:
                raise GenError(f"{r.name}: argument {a} must be a declared scalar")
            ct = {"int": "int64_t", "real": "double", "logical": "bool"}[d.type]
            if d.intent in ("out", "inout"):
                params.append(f"{ct}& {a}")
            else:
                params.append(f"{ct} {a}")
            sc.set(a, "scalar", d.type, a)
        mod_sc = self.mod_scalars_of(r.body, local_names=set(r.decls) | set(r.args))
        self.dev_mod_sc[r.name] = mod_sc
        params += [f"{self.ctype(self.p.state.decls[n].type)} m_{n}" for n in mod_sc]
        body = []
        locals_ = []
        for n, d in r.decls.items():
            if n in r.args:
                continue
            if d.dims:
                raise GenError(f"{r.name}: local arrays in device routines are not supported")
            sc.set(n, "scalar", d.type, n)
            locals_.append(f"  {self.ctype(d.type)} {n} = {self.zero(d.type)};")
        body += locals_
        body += self.stmts(r.body, sc, "  ", kernel=True)
        sig = f"__device__ void dev_{r.name}({', '.join(params)})"
        self.devfns.append((sig, body))

    def ctype(self, t):
        return {"int": "int64_t", "real": "double", "logical": "bool"}[t]

    def zero(self, t):
        return {"int": "0", "real": "0.0", "logical": "false"}[t]

    # -- statements -------------------------------------------------------------------------
    def stmts(self, ss, sc, ind, kernel, R=None, region_ctx=None):
        out = []
        for s in ss:
            out += self.stmt(s, sc, ind, kernel, R, region_ctx)
        return out

    def stmt(self, s, sc, ind, kernel, R, region_ctx):
        em = self.em
        if isinstance(s, Return):
            if kernel and region_ctx is not None:  # a kernel thread leaves: a guard return
                region_ctx["ret"] = True
                return [f"{ind}{{ atomicAdd(hfc_ret, 1ULL); return; }}"]
            return [f"{ind}return;"]
        if isinstance(s, Stop):
            if kernel:
                raise GenError(f"line {s.line}: stop inside device code is not supported")
            return [f"{ind}throw HfcStop{{{s.code}}};"]
        if isinstance(s, Assign):
            rhs_t = em.etype(s.rhs, sc)
            if isinstance(s.lhs, Ref):
                v = sc.get(s.lhs.name)
                if v is None or v[0] not in ("array", "xarray", "harray"):
                    raise GenError(f"line {s.line}: assignment to non-array {s.lhs.name}(...)")
                if region_ctx is not None:
                    region_ctx["written"].add(s.lhs.name)
                rhs = em.real(s.rhs, sc)
                sc.set("@write", "meta", "", True)
                lhs = em.expr(s.lhs, sc)
                sc.names.pop("@write")
                if v[0] == "harray":  # host element write (marks the host copy newer)
                    return [f"{ind}{{ const double hfc_v = {rhs}; {lhs} = hfc_v; }}"]
                return [f"{ind}{lhs} = {rhs};"]
            n = s.lhs.name
            v = sc.get(n)
            if v is None:
                raise GenError(f"line {s.line}: assignment to unknown {n}")
            kind, t, c = v
            val = em.expr(s.rhs, sc)
            if t == "real" and rhs_t != "real":
                val = f"static_cast<double>({val})"
            elif t == "int" and rhs_t == "real":
                val = f"static_cast<int64_t>({val})"
            if kind == "const":
                raise GenError(f"line {s.line}: assignment to the parameter {n}")
            if kind == "mscalar":
                if kernel:
                    raise GenError(f"line {s.line}: module scalar {n} written inside a kernel "
                                   "outside a reduce(...) region")
                setter = "hfc_seti" if t == "int" else "hfc_setr" if t == "real" else "hfc_setl"
                return [f"{ind}{setter}(R, \"{n}\", {val});"]
            return [f"{ind}{c} = {val};"]
        if isinstance(s, Do):
            v = sc.get(s.var)
            if v is None or v[1] != "int":
                raise GenError(f"line {s.line}: loop variable {s.var} must be an integer")
            lo, hi = em.expr(s.lo, sc), em.expr(s.hi, sc)
            c = v[2]
            out = [f"{ind}{{", f"{ind}  const int64_t hfc_end_{s.line} = {hi};",
                   f"{ind}  for ({c} = {lo}; {c} <= hfc_end_{s.line}; ++{c}) {{"]
            out += self.stmts(s.body, sc, ind + "    ", kernel, R, region_ctx)
            out += [f"{ind}  }}", f"{ind}}}"]
            return out
        if isinstance(s, If):
            out = []
            for k, (cond, body) in enumerate(s.branches):
                if cond is not None:
                    kw = "if" if k == 0 else "} else if"
                    out.append(f"{ind}{kw} ({em.expr(cond, sc)}) {{")
                else:
                    out.append(f"{ind}}} else {{")
                out += self.stmts(body, sc, ind + "  ", kernel, R, region_ctx)
            out.append(f"{ind}}}")
            return out
        if isinstance(s, Call):
            if kernel:
                callee = self.p.routines.get(s.name)
                if callee is None:
                    raise GenError(f"line {s.line}: call of unknown routine {s.name}")
                args = []
                for a, formal in zip(s.args, callee.args):
                    d = callee.decls[formal]
                    if d.intent in ("out", "inout"):
                        if isinstance(a, Ref) and sc.get(a.name) is not None and \
                                sc.get(a.name)[0] in ("array", "xarray"):
                            if region_ctx is not None:
                                region_ctx["written"].add(a.name)
                            sc.set("@write", "meta", "", True)
                            elem = em.expr(a, sc)  # the element, by reference
                            sc.names.pop("@write")
                            if d.intent == "inout":  # copy-in reads it first
                                elem = f"((void){em.expr(a, sc)}, {elem})"
                            args.append(elem)
                            continue
                        if not isinstance(a, Name):
                            raise GenError(f"line {s.line}: intent(out) argument must be a "
                                           "variable or an array element")
                        args.append(sc.get(a.name)[2])
                    else:
                        args.append(em.real(a, sc) if d.type == "real" else em.expr(a, sc))
                args += [sc.get(n)[2] for n in self.dev_mod_sc[s.name]]
                return [f"{ind}dev_{s.name}({', '.join(args)});"]
            callee = self.p.routines.get(s.name)
            if callee is None:
                raise GenError(f"line {s.line}: call of unknown routine {s.name}")
            if len(s.args) != len(callee.args):
                raise GenError(f"line {s.line}: {s.name} takes {len(callee.args)} arguments")
            args = ["R"]
            for a, formal in zip(s.args, callee.args):
                d = callee.decls.get(formal)
                if d is None:
                    raise GenError(f"{s.name}: undeclared argument {formal}")
                if d.dims:  # array dummy: the actual array's runtime name
                    if not isinstance(a, Name) or sc.get(a.name) is None or \
                            sc.get(a.name)[0] != "harray":
                        raise GenError(f"line {s.line}: array argument {formal} needs an array")
                    args.append(sc.get(a.name)[2])
                elif d.intent in ("out", "inout"):
                    v = sc.get(a.name) if isinstance(a, Name) else None
                    if v is None or v[0] != "scalar":
                        raise GenError(f"line {s.line}: intent(out) argument must be a local "
                                       "variable")
                    args.append(v[2])
                else:
                    args.append(em.real(a, sc) if d.type == "real" else em.expr(a, sc))
            return [f"{ind}host_{s.name}({', '.join(args)});"]
        if isinstance(s, Region):
            if kernel:
                raise GenError(f"line {s.line}: nested parallel regions")
            return self.region(s, sc, ind, R)
        raise GenError(f"unsupported statement {s}")

    # -- a parallel region: kernel + launch -------------------------------------------------
    def region(self, s, hsc, ind, R):
        r = R["routine"]
        red = None  # (op, module scalar): the OpenACC-style reduction, acc-simulated order
        if "reduce" in s.attrs:
            if len(s.attrs["reduce"]) != 1 or ":" not in s.attrs["reduce"][0]:
                raise GenError(f"{r.name}:{s.line}: one reduce(op:var) is supported")
            op, var = [x.strip().lower() for x in s.attrs["reduce"][0].split(":")]
            v = hsc.get(var)
            if op not in ("+", "*") or v is None or v[0] != "mscalar" or v[1] != "real":
                raise GenError(f"{r.name}:{s.line}: reduce needs + or * on a real module scalar")
            red = (op, var)
        names = [n.lower() for n in s.attrs.get("domname", [])]
        sizes = s.attrs.get("domsize", [])
        if len(names) not in (1, 2) or len(names) != len(sizes):
            raise GenError(f"{r.name}:{s.line}: domName/domSize must name 1 or 2 dims")
        lo, hi = region_bounds(s)
        idx = self.kcount.get(r.name, 0)
        self.kcount[r.name] = idx + 1
        kname = f"hfk{idx}_{r.name}"
        # kernel scope: iterators, region-written scalars (kernel locals), arrays, values
        ksc = Scope()
        self.module_scope(ksc, host=False)
        used_arrays, read_scalars, written = [], [], set()

        def scan(stmts):
            for st in stmts:
                if isinstance(st, Assign):
                    if isinstance(st.lhs, Name):
                        written.add(st.lhs.name)
                    scan_e(st.lhs)
                    scan_e(st.rhs)
                elif isinstance(st, Do):
                    written.add(st.var)
                    scan_e(st.lo)
                    scan_e(st.hi)
                    scan(st.body)
                elif isinstance(st, If):
                    for c, b in st.branches:
                        if c is not None:
                            scan_e(c)
                        scan(b)
                elif isinstance(st, Call):
                    callee = self.p.routines.get(st.name)
                    for a, formal in zip(st.args, callee.args if callee else []):
                        if callee.decls[formal].intent in ("out", "inout") and isinstance(a, Name):
                            written.add(a.name)
                        scan_e(a)

        def scan_e(e):
            if isinstance(e, Name):
                if e.name not in read_scalars:
                    read_scalars.append(e.name)
            elif isinstance(e, Ref):
                v = hsc.get(e.name)
                if v is not None and v[0] == "harray" and e.name not in used_arrays:
                    used_arrays.append(e.name)
                # real(x, kind): the kind argument is not a value
                for a in (e.args[:1] if e.name == "real" and v is None else e.args):
                    scan_e(a)
            elif isinstance(e, Bin):
                scan_e(e.a)
                scan_e(e.b)
            elif isinstance(e, Un):
                scan_e(e.x)

        scan(s.body)
        for e in lo + hi:
            scan_e(e)
        params, args = [], []
        for a in used_arrays:
            params.append(f"HArr {a}")
            args.append(f"hfc_array(R, {hsc.get(a)[2]})")
            ksc.set(a, "xarray" if a in self.extended else "array", "real", a)
        for k, n in enumerate(names):
            ksc.set(n, "scalar", "int", n)
        ksc.set("@iters", "meta", "", tuple(names))
        values = []
        for n in read_scalars:
            if n in names or n in written:
                continue
            v = hsc.get(n)
            if v is None:
                raise GenError(f"{r.name}:{s.line}: unknown name {n} in a parallel region")
            if v[0] in ("harray", "const"):
                continue
            if v[0] == "mscalar":
                continue  # module scalars travel as m_<name>
            values.append(n)
            params.append(f"{self.ctype(v[1])} {n}")
            args.append(v[2])
            ksc.set(n, "scalar", v[1], n)
        mod_sc = self.mod_scalars_of(s.body, lo + hi, local_names=set(r.decls) | set(names))
        if red:
            mod_sc = [n for n in mod_sc if n != red[1]]
            params += ["double* hfc_red", "int64_t hfc_ex"]
            args += ["hfc_red_buf", "ex"]
        for n in mod_sc:
            t = self.p.state.decls[n].type
            params.append(f"{self.ctype(t)} m_{n}")
            args.append(hsc.get(n)[2])
        kloc = []
        for n in sorted(written):
            if n in names:
                continue
            v = hsc.get(n)
            if v is None:
                raise GenError(f"{r.name}:{s.line}: unknown name {n}")
            if red and n == red[1]:  # the thread's private accumulator from the identity
                ksc.set(n, "scalar", "real", n)
                kloc.append(f"  double {n} = {'1.0' if red[0] == '*' else '0.0'};")
                continue
            if v[0] == "mscalar":
                raise GenError(f"{r.name}:{s.line}: module scalar {n} written in a region "
                               "outside a reduce(...) clause")
            ksc.set(n, "scalar", v[1], n)
            kloc.append(f"  {self.ctype(v[1])} {n} = {self.zero(v[1])};")
        lo_c = [self.em.expr(e, ksc) for e in lo]
        hi_c = [self.em.expr(e, ksc) for e in hi]
        body = []
        body.append(f"  const int64_t {names[0]} = static_cast<int64_t>(blockIdx.x) * blockDim.x + "
                    f"threadIdx.x + ({lo_c[0]});")
        if len(names) == 2:
            body.append(f"  const int64_t {names[1]} = static_cast<int64_t>(blockIdx.y) * "
                        f"blockDim.y + threadIdx.y + ({lo_c[1]});")
            body.append(f"  if ({names[0]} > ({hi_c[0]}) || {names[1]} > ({hi_c[1]})) return;")
        else:
            body.append(f"  if ({names[0]} > ({hi_c[0]})) return;")
        body += kloc
        rctx = {"written": set()}
        body += self.stmts(s.body, ksc, "  ", kernel=True, region_ctx=rctx)
        if red:  # partial of iteration (i, j) at its linear id, i fastest (interp.cpp:1127)
            lin = f"({names[0]} - ({lo_c[0]}))"
            if len(names) == 2:
                lin = f"({names[1]} - ({lo_c[1]})) * hfc_ex + {lin}"
            body.append(f"  hfc_red[{lin}] = {red[1]};")
        if rctx.get("ret"):  # user returns counted on the device (exec_launch guard_returns)
            params.append("unsigned long long* hfc_ret")
            args.append("hfc_ret_counter(R)")
        sig = f"__global__ void __launch_bounds__(128) {kname}({', '.join(params)})"
        self.kernels.append((sig, body))
        # host launch (grid ceiling(extent / B), block (32, 4, 1): codegen.cpp:421-434)
        hlo = [self.em.expr(e, hsc) for e in lo]
        hhi = [self.em.expr(e, hsc) for e in hi]
        out = [f"{ind}{{  // {kname}: region at line {s.line}"]
        for a in used_arrays:
            mode = 2 if a in rctx["written"] else 0
            out.append(f"{ind}  hfc_prepare(R, {hsc.get(a)[2]}, {mode});")
        out.append(f"{ind}  const int64_t ex = ({hhi[0]}) - ({hlo[0]}) + 1;")
        out.append(f"{ind}  const int64_t ey = " + (f"({hhi[1]}) - ({hlo[1]}) + 1;" if len(names) == 2
                                                     else "1;"))
        if red:  # acc kernels: one virtual launch over the iteration space (interp.cpp:1114)
            out.append(f"{ind}  double* hfc_red_buf = hfc_red_alloc(R, \"{r.name}.@red{s.line}\", "
                       "ex * ey);")
            out.append(f"{ind}  R.st->launches += 1;")
            out.append(f"{ind}  R.st->threads += ex * ey;")
        else:
            out.append(f"{ind}  hfc_count(R, ex, ey);")
        out.append(f"{ind}  if (ex > 0 && ey > 0) {{")
        out.append(f"{ind}    dim3 grid(static_cast<unsigned>((ex + 31) / 32), "
                   f"static_cast<unsigned>((ey + 3) / 4), 1), block(32, 4, 1);")
        out.append(f"{ind}    {kname}<<<grid, block, 0, R.stream>>>({', '.join(args)});")
        out.append(f"{ind}    HFC_CHECK(hfc_launched(R));")
        out.append(f"{ind}  }}")
        if red:  # partials combined in linear-id order from the initial value (:1163-1173)
            out.append(f"{ind}  hfc_setr(R, \"{red[1]}\", hfc_red_finish(R, hfc_red_buf, ex * ey, "
                       f"hfc_getr(R, \"{red[1]}\"), {int(red[0] == '*')}));")
        for a in sorted(rctx["written"]):
            out.append(f"{ind}  hfc_written(R, {hsc.get(a)[2]});")
        out.append(f"{ind}}}")
        return out

    # -- host routines ------------------------------------------------------------------------
    def host_signature(self, r):
        params = ["Run& R"]
        for a in r.args:
            d = r.decls.get(a)
            if d is None:
                raise GenError(f"{r.name}: undeclared argument {a}")
            if d.dims:
                params.append(f"const char* a_{a}")
            elif d.intent in ("out", "inout"):
                params.append(f"{self.ctype(d.type)}& a_{a}")
            else:
                params.append(f"{self.ctype(d.type)} a_{a}")
        return f"void host_{r.name}({', '.join(params)})"

    def gen_host(self, r):
        sc = Scope()
        self.module_scope(sc, host=True)
        body = []
        locs = self.local_arrays(r)
        for n, d in self.p.state.decls.items():
            if d.dims:
                sc.set(n, "harray", "real", f"\"{n}\"")
                sc.set("@href:" + n, "meta", "", f"h_{n}")
                body.append(f"  HRef h_{n};")
        for n, d in r.decls.items():
            if n in r.args:
                if d.dims:
                    sc.set(n, "harray", "real", f"a_{n}")
                    sc.set("@href:" + n, "meta", "", f"ha_{n}")
                    body.append(f"  HRef ha_{n};")
                else:
                    sc.set(n, "scalar", d.type, f"a_{n}")
                continue
            if d.dims:
                continue
            sc.set(n, "scalar", d.type, f"l_{n}")
            body.append(f"  {self.ctype(d.type)} l_{n} = {self.zero(d.type)};")
        self.extended = {n for n, v in locs.items() if v[2]}
        self.rt_names = {n: f"{r.name}.{n}" for n in locs}
        for n, (d, dims, extended, dn) in locs.items():
            key = f"{r.name}.{n}"
            roles = self.local_roles(r, n, dims, extended)
            lo = ", ".join(self.em.expr(a, sc) for a, _ in dims)
            hi = ", ".join(self.em.expr(b, sc) for _, b in dims)
            rl = ", ".join(str(x) for x in roles)
            body.append(f"  {{ const int64_t lo[] = {{{lo}}}, hi[] = {{{hi}}}; "
                        f"const int roles[] = {{{rl}}};")
            body.append(f"    hfc_scratch(R, \"{key}\", {len(dims)}, lo, hi, roles); }}")
            sc.set(n, "harray", "real", f"\"{key}\"")
            sc.set("@href:" + n, "meta", "", f"hl_{n}")
            body.append(f"  HRef hl_{n};")
        transfers = []
        for dd in r.domdeps:
            if "transferhere" in dd.attrs.get("attribute", []):
                for n in dd.names:
                    if n in self.p.state.decls and self.p.state.decls[n].dims:
                        transfers.append(n)
        self.routine_transfers[r.name] = transfers
        for n in transfers:
            body.append(f"  HFC_CHECK(hfc_copy_in(R, \"{n}\"));")
        R = {"routine": r}
        body += self.stmts(r.body, sc, "  ", kernel=False, R=R)
        for n in transfers:
            body.append(f"  HFC_CHECK(hfc_copy_out(R, \"{n}\"));")
        self.hostfns.append((self.host_signature(r), body))

    def local_roles(self, r, n, dims, extended):
        rank = len(dims)
        if extended:  # domain dims prepended: (i, j, declared...)
            roles = [ROLE_I, ROLE_J][:min(2, rank)]
            rest = [ROLE_K, ROLE_L]
            roles += [rest.pop(0) for _ in range(rank - len(roles))]
            return roles
        # from region accesses of this routine
        iters_roles = None

        def visit_e(e, it):
            nonlocal iters_roles
            if isinstance(e, Ref):
                if e.name == n and it and iters_roles is None:
                    cand = [_iter_of(a, it) for a in e.args]
                    if any(c is not None for c in cand):
                        iters_roles = cand
                for a in e.args:
                    visit_e(a, it)
            elif isinstance(e, Bin):
                visit_e(e.a, it)
                visit_e(e.b, it)
            elif isinstance(e, Un):
                visit_e(e.x, it)

        def visit(ss, it):
            for s in ss:
                if isinstance(s, Assign):
                    visit_e(s.lhs, it)
                    visit_e(s.rhs, it)
                elif isinstance(s, Do):
                    visit(s.body, it)
                elif isinstance(s, If):
                    for c, b in s.branches:
                        if c is not None:
                            visit_e(c, it)
                        visit(b, it)
                elif isinstance(s, Region):
                    visit(s.body, [x.lower() for x in s.attrs.get("domname", [])])

        visit(r.body, [])
        roles = [None] * rank
        if iters_roles:
            for p, v in enumerate(iters_roles):
                if v is not None:
                    roles[p] = [ROLE_I, ROLE_J][v]
        rest = [ROLE_K, ROLE_L]
        for p in range(rank):
            if roles[p] is None:
                roles[p] = rest.pop(0) if rest else ROLE_L
        return roles

    # -- translation unit ---------------------------------------------------------------------
    def generate(self):
        order, seen = [], set()

        def visit(n):  # callees first (C++ declaration order, dev_mod_sc of callees)
            if n in seen:
                return
            seen.add(n)
            calls = set()
            _names_in(self.p.routines[n].body, set(), calls)
            for c in sorted(calls):
                if c in self.p.device_routines:
                    visit(c)
            order.append(n)

        for n in sorted(self.p.device_routines):
            visit(n)
        for n in order:
            self.gen_devfn(self.p.routines[n])
        host_names = [n for n in self.p.routines if n not in self.p.device_routines]
        for n in host_names:
            self.gen_host(self.p.routines[n])
        lines = [f"// generated by paper_1710_08616_b200.hfc from program '{self.p.name}'",
                 "// (Hybrid-Fortran dialect -> CUDA C++ for sm_100a); do not edit", PRELUDE]
        lines.append("namespace {")
        names = sorted(self.em.nids, key=self.em.nids.get) or ["?"]
        lines.append("const char* const kNames[] = {" + ", ".join(f'"{n}"' for n in names) + "};")
        lines.append(f"constexpr bool kDeviceErrors = {'true' if self.em.used_idiv else 'false'};")
        lines.append(HOST_HELPERS.replace("@MODULE@", self.p.state.name))
        for sig, body in self.devfns:
            lines.append(sig + " {")
            lines += body
            lines.append("}")
        for sig, body in self.kernels:
            lines.append(sig + " {")
            lines += body
            lines.append("}")
        for n in host_names:
            lines.append(self.host_signature(self.p.routines[n]) + ";")
        for sig, body in self.hostfns:
            lines.append(sig + " {")
            lines += body
            lines.append("}")
        lines.append(self.descriptor(host_names))
        lines.append("}  // namespace")
        lines.append(EXPORT)
        return "\n".join(lines) + "\n"

    def descriptor(self, host_names):
        st = self.p.state
        sc = [(n, d) for n, d in st.decls.items() if not d.dims]
        ar = [(n, d) for n, d in st.decls.items() if d.dims]
        out = []
        out.append("const hfb_plugin_scalar kScalars[] = {")
        for n, d in sc:
            out.append(f"  {{\"{n}\", {['int', 'real', 'logical'].index(d.type)}}},")
        out.append("  {nullptr, 0}};")
        out.append("const hfb_plugin_array kArrays[] = {")
        for n, d in ar:
            los = ", ".join(f"\"{self.dimtext(a)}\"" for a, _ in d.dims)
            his = ", ".join(f"\"{self.dimtext(b)}\"" for _, b in d.dims)
            roles = ", ".join(str(x) for x in self.p.module_roles[n])
            out.append(f"  {{\"{n}\", {len(d.dims)}, {{{los}}}, {{{his}}}, {{{roles}}}}},")
        out.append("  {nullptr, 0, {}, {}, {}}};")
        host_names = [n for n in host_names if not self.p.routines[n].args]
        out.append("const char* kEntries[] = {")
        for n in host_names:
            out.append(f"  \"{n}\",")
        out.append("  nullptr};")
        trans = [n for n in host_names if self.transfers_closure(n)]
        out.append("const char* kTransferEntries[] = {")
        for n in trans:
            out.append(f"  \"{n}\",")
        out.append("  nullptr};")
        out.append("void dispatch(Run& R, const char* routine) {")
        for n in host_names:
            out.append(f"  if (!std::strcmp(routine, \"{n}\")) {{ host_{n}(R); return; }}")
        out.append("  throw static_cast<int>(HFB_CONFIG);")
        out.append("}")
        h = hashlib.sha1(self.p.name.encode()).hexdigest()[:8]
        out.append(f"const char kProgram[] = \"{self.p.name}\";")
        out.append(f"const char kModule[] = \"{st.name}\";  // build {h}")
        return "\n".join(out)

    def transfers_closure(self, n, seen=None):
        seen = seen or set()
        if n in seen:
            return False
        seen.add(n)
        if self.routine_transfers.get(n):
            return True

        def calls(ss):
            for s in ss:
                if isinstance(s, Call):
                    yield s.name
                elif isinstance(s, Do):
                    yield from calls(s.body)
                elif isinstance(s, If):
                    for _, b in s.branches:
                        yield from calls(b)

        return any(self.transfers_closure(c, seen) for c in calls(self.p.routines[n].body)
                   if c in self.p.routines and c not in self.p.device_routines)

    def dimtext(self, e):
        if isinstance(e, Num):
            return e.text
        if isinstance(e, Name) and e.name in self.p.params:
            pv = self.p.params[e.name].param
            if isinstance(pv, Num) and not pv.is_real:
                return pv.text
            raise GenError(f"parameter {e.name} used as an array bound must be an integer literal")
        if isinstance(e, Name):
            return e.name
        raise GenError("array dims must be literals or scalar names")


HOST_HELPERS = r"""
const char* const kMod = "@MODULE@";
int64_t hfc_geti(Run& R, const char* n) {
  int64_t v = 0;
  HFC_CHECK(hfb_get_scalar_i64(R.ctx, kMod, n, &v));
  return v;
}
double hfc_getr(Run& R, const char* n) {
  double v = 0;
  HFC_CHECK(hfb_get_scalar_f64(R.ctx, kMod, n, &v));
  return v;
}
bool hfc_getl(Run& R, const char* n) { return hfc_geti(R, n) != 0; }
void hfc_seti(Run& R, const char* n, int64_t v) { HFC_CHECK(hfb_set_scalar_i64(R.ctx, kMod, n, v)); }
void hfc_setr(Run& R, const char* n, double v) { HFC_CHECK(hfb_set_scalar_f64(R.ctx, kMod, n, v)); }
void hfc_setl(Run& R, const char* n, bool v) { hfc_seti(R, n, v ? 1 : 0); }
// residency checks before a kernel reads (0) or reads+writes (2) an array
void hfc_prepare(Run& R, const char* n, int mode) { HFC_CHECK(hfb_plugin_prepare(R.ctx, n, mode)); }
void hfc_written(Run& R, const char* n) { HFC_CHECK(hfb_plugin_written(R.ctx, n)); }
// checked builds: the declared bounds and init flags of an array (device or host copy)
void hfc_checked(Run& R, const char* n, HArr& a, bool device) {
#ifdef HFC_CHECKED
  int rank = 0;
  int64_t lo[4], hi[4];
  uint8_t *dinit = nullptr, *hinit = nullptr;
  HFC_CHECK(hfb_plugin_array_info(R.ctx, n, &rank, lo, hi, &dinit, &hinit));
  for (int d = 0; d < 4; ++d) a.hi[d] = hi[d];
  a.init = device ? dinit : hinit;
#else
  (void)R, (void)n, (void)a, (void)device;
#endif
}
HArr hfc_array(Run& R, const char* n) {
  hfb_view v;
  HFC_CHECK(hfb_plugin_view(R.ctx, n, &v));
  HArr a = hfc_view(v);
  hfc_checked(R, n, a, true);
  return a;
}
void hfc_scratch(Run& R, const char* key, int rank, const int64_t* lo, const int64_t* hi,
                 const int* roles) {
  HFC_CHECK(hfb_plugin_scratch(R.ctx, key, rank, lo, hi, roles));
#ifdef HFC_CHECKED
  HFC_CHECK(hfb_plugin_scratch_clear_init(R.ctx, key));  // elaborate_locals: no element set
#endif
}
// host-side element access (host routines): the bound host buffer; write = 1 makes the
// host copy the newest
HArr hfc_host(Run& R, const char* n, int write) {
  hfb_view v;
  HFC_CHECK(hfb_plugin_host(R.ctx, n, write, &v));
  HArr a = hfc_view(v);
  hfc_checked(R, n, a, false);
  return a;
}
// per host-routine invocation: one cached reference per array, fetched on first access
struct HRef {
  hfb_host_ref r;
  bool ok = false;
};
inline HArr hfc_rd(Run& R, HRef& h, const char* n) {
  if (!h.ok) {
    HFC_CHECK(hfb_plugin_host_ref(R.ctx, n, &h.r));
    h.ok = true;
  }
  if (*h.r.residency == 1) return hfc_host(R, n, 0);  // raises the stale-copy error
  HArr a = hfc_view(h.r.view);
  hfc_checked(R, n, a, false);
  return a;
}
inline HArr hfc_wr(Run& R, HRef& h, const char* n) {
  if (!h.ok) {
    HFC_CHECK(hfb_plugin_host_ref(R.ctx, n, &h.r));
    h.ok = true;
  }
  if (*h.r.has_device) *h.r.residency = 0;  // the host copy is now the newest
  HArr a = hfc_view(h.r.view);
  hfc_checked(R, n, a, false);
  return a;
}
// the run's early-return counter (one device word, zeroed once per run)
unsigned long long* hfc_ret_counter(Run& R) {
  if (!R.ret) {
    const int64_t lo[] = {1}, hi[] = {1};
    const int roles[] = {0};
    HFC_CHECK(hfb_plugin_scratch(R.ctx, "@run.ret", 1, lo, hi, roles));
    hfb_view v;
    HFC_CHECK(hfb_plugin_view(R.ctx, "@run.ret", &v));
    R.ret = reinterpret_cast<unsigned long long*>(v.origin);
    if (cudaMemsetAsync(R.ret, 0, sizeof(unsigned long long), R.stream) != cudaSuccess)
      throw static_cast<int>(HFB_CUDA);
  }
  return R.ret;
}
int hfc_copy_in(Run& R, const char* n) {
  if (!R.allow_transfers) return HFB_CONFIG;
  return hfrt_copy_to_device(R.ctx, kMod, n);
}
int hfc_copy_out(Run& R, const char* n) { return hfrt_copy_from_device(R.ctx, kMod, n); }
// the generated code's launch accounting (interp.cpp:1417-1475): block 32 x 4
void hfc_count(Run& R, int64_t ex, int64_t ey) {
  if (ex <= 0 || ey <= 0) throw static_cast<int>(HFB_RUNTIME);
  const int64_t gx = (ex + 31) / 32, gy = (ey + 3) / 4, total = gx * gy * 128;
  R.st->launches += 1;
  R.st->threads += total;
  R.st->guard_returns += total - ex * ey;
}
// the device error record: HFB_RUNTIME with the reference's text if a thread failed
int hfc_check_err(Run& R) {
  HfcErr e{};
  if (cudaMemcpyFromSymbolAsync(&e, hfc_err, sizeof e, 0, cudaMemcpyDeviceToHost, R.stream) !=
          cudaSuccess ||
      cudaStreamSynchronize(R.stream) != cudaSuccess)
    return HFB_CUDA;
  if (e.code == 0) return HFB_OK;
  const HfcErr zero{};
  cudaMemcpyToSymbolAsync(hfc_err, &zero, sizeof zero, 0, cudaMemcpyHostToDevice, R.stream);
  cudaStreamSynchronize(R.stream);
  const HfcFail f = hfc_fail_msg(e.code, e.name, e.dim, e.idx, e.lo, e.hi);
  return hfb_plugin_error(R.ctx, f.status, f.msg);
}
int hfc_launched(Run& R) {
  R.st->native_launches += 1;
  if (cudaGetLastError() != cudaSuccess) return HFB_CUDA;
#ifdef HFC_CHECKED
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(R.stream, &cap);
  if (cap == cudaStreamCaptureStatusNone) return hfc_check_err(R);  // after every launch
#endif
  return HFB_OK;
}
double* hfc_red_alloc(Run& R, const char* key, int64_t n) {
  const int64_t lo[] = {1}, hi[] = {n + 1};
  const int roles[] = {0};
  HFC_CHECK(hfb_plugin_scratch(R.ctx, key, 1, lo, hi, roles));
  hfb_view v;
  HFC_CHECK(hfb_plugin_view(R.ctx, key, &v));
  return v.origin;
}
double hfc_red_finish(Run& R, double* partials, int64_t n, double init, int is_mul) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(R.stream, &cap);
  if (cap != cudaStreamCaptureStatusNone)  // the result is needed on the host now
    throw static_cast<int>(HFB_CONFIG);
  hfc_ordered<<<1, 1, 0, R.stream>>>(partials, n, init, is_mul, partials + n);
  HFC_CHECK(hfc_launched(R));
  double out = 0.0;
  if (cudaMemcpyAsync(&out, partials + n, sizeof(double), cudaMemcpyDeviceToHost, R.stream) !=
          cudaSuccess ||
      cudaStreamSynchronize(R.stream) != cudaSuccess)
    throw static_cast<int>(HFB_CUDA);
  R.st->native_launches -= 1;  // the combine is part of the one virtual launch
  return out;
}
"""

EXPORT = r"""
namespace {
int run_entry(hfb_ctx* ctx, const char* routine, hfb_launch_stats* stats, int allow_transfers) {
  Run R{ctx, stats, static_cast<cudaStream_t>(hfb_stream(ctx)), allow_transfers};
  try {
    try {
      dispatch(R, routine);
    } catch (const HfcStop&) {
      // the program stopped: the run ends here, state as left (run_program, interp.cpp)
    } catch (const HfcFail& f) {
      return hfb_plugin_error(ctx, f.status, f.msg);
    }
#ifdef HFC_CHECKED
    constexpr bool kCheck = true;
#else
    constexpr bool kCheck = kDeviceErrors;  // only programs whose kernels divide integers
#endif
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(R.stream, &cap);
    if (kCheck && cap == cudaStreamCaptureStatusNone) {  // device-side errors of the run
      const int rc = hfc_check_err(R);
      if (rc != HFB_OK) return rc;
    }
    if (R.ret) {  // kernel threads that returned early count as guard returns
      unsigned long long n = 0;
      if (cudaMemcpyAsync(&n, R.ret, sizeof n, cudaMemcpyDeviceToHost, R.stream) != cudaSuccess ||
          cudaStreamSynchronize(R.stream) != cudaSuccess)
        return HFB_CUDA;
      R.st->guard_returns += static_cast<int64_t>(n);
    }
  } catch (int rc) {
    return rc;
  }
  return HFB_OK;
}
const hfb_plugin_desc kDesc = {HFB_PLUGIN_ABI, kProgram, kModule, kScalars, kArrays,
                               kEntries, kTransferEntries, run_entry};
}  // namespace

extern "C" const hfb_plugin_desc* hfb_plugin(void) { return &kDesc; }
"""


def generate(sources, name):
    """[(path, text)] -> CUDA C++ translation unit (str)"""
    return Gen(Program(sources, name)).generate()
