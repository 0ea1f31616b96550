"""hfc on the CPU: the dialect parser, the generator's determinism and its refusals, and
the descriptor a built plugin exports (loaded with ctypes; no device work)."""
import ctypes
from pathlib import Path

import pytest

from paper_1710_08616_b200 import hfc
from paper_1710_08616_b200.hfc.gen import GenError, generate
from paper_1710_08616_b200.hfc.parse import Bin, Name, Num, Un, logical_lines, parse_decl, \
    parse_expr

ROOT = Path(__file__).resolve().parents[1]


# ---- parser -------------------------------------------------------------------------------
def test_expression_precedence():
    # unary minus binds looser than ** (Fortran): -a**2 == -(a**2)
    e = parse_expr("-a**2", 1)
    assert isinstance(e, Un) and isinstance(e.x, Bin) and e.x.op == "**"
    # ** is right-associative
    e = parse_expr("a**b**c", 1)
    assert e.op == "**" and isinstance(e.b, Bin) and e.b.op == "**"
    # left-associative + - (the evaluation order the bit-exactness depends on)
    e = parse_expr("a - b + c", 1)
    assert e.op == "+" and isinstance(e.a, Bin) and e.a.op == "-"
    # relational spellings
    assert parse_expr("a >= b", 1).op == ".ge."
    assert parse_expr("a .ne. b", 1).op == ".ne."
    e = parse_expr("1.5_r_size", 1)
    assert isinstance(e, Num) and e.is_real and e.text.startswith("1.5")


def test_continuations_and_comments():
    text = "x = a + &\n  & b ! tail comment\n! whole-line comment\ny = 1\n"
    lines = [t for _, t in logical_lines(text)]
    assert len(lines) == 2
    assert lines[0].replace(" ", "") == "x=a+b"


def test_parameter_declaration():
    [d] = parse_decl("integer(4), parameter :: ntlm = 4", 1)
    assert d.name == "ntlm" and d.type == "int" and isinstance(d.param, Num)
    [d] = parse_decl("real(r_size), intent(inout) :: swind(nx, ny)", 1)
    assert d.intent == "inout" and len(d.dims) == 2 and isinstance(d.dims[0][1], Name)


# ---- generator ----------------------------------------------------------------------------
def _src(paths):
    return [(str(p), Path(p).read_text()) for p in paths]


@pytest.mark.parametrize("name", sorted(hfc.BUILTIN_SOURCES))
def test_generation_is_deterministic(name):
    srcs = _src([ROOT / s for s in hfc.BUILTIN_SOURCES[name]])
    a = generate(srcs, name)
    b = generate(srcs, name)
    assert a == b
    assert "__global__" in a and "hfb_plugin(void)" in a


@pytest.mark.skipif(not hfc.REFERENCE_APPS.is_dir(), reason="reference corpus absent")
@pytest.mark.parametrize("name", sorted(hfc.CORPUS_SOURCES))
def test_reference_corpus_translates(name):
    code = generate(_src([hfc.REFERENCE_APPS / s for s in hfc.CORPUS_SOURCES[name]]), name)
    assert "hfk0_" in code
    if name == "reduction_gen":  # reduce(+:total): partials + the ordered combine
        assert "hfc_red_finish" in code and "hfc_red[" in code
    if name == "surface_flux_gen":
        # appliesTo(CPU) wrapper over GPU kernels: iterators pinned to the region start
        assert "l_i = INT64_C(1);" in code
        assert "hfc_wr(R, h_cover_frac, \"cover_frac\")" in code  # setup's host update


STATE = """module st
  implicit none
  integer(4), parameter :: np = 3
  integer(4) :: nx
  integer(4) :: ny
  integer(4) :: cnt
  real(r_size) :: s
  real(r_size) :: a(nx, ny)
end module
"""


def _gen(body):
    return generate([("st.h90", STATE), ("m.h90", "module m\ncontains\n" + body +
                                          "end module\n")], "t")


def _region(stmts, extra=""):
    return f"""  subroutine run()
    use st, only : nx, ny, cnt, s, a, np
    implicit none
    {extra}
    @domainDependant{{attribute(autoDom, present)}}
    a
    @end domainDependant
    @parallelRegion{{domName(i,j), domSize(nx,ny)}}
{stmts}
    @end parallelRegion
  end subroutine
"""


def test_plain_region_generates():
    code = _gen(_region("    a(i,j) = a(i,j) + real(np, r_size)"))
    assert "hfk0_run" in code and "INT64_C(3)" in code


@pytest.mark.parametrize("body,msg", [
    (_region("    cnt = cnt + 1"), "module scalar cnt written in a region"),
    (_region("    call nowhere(i)"), "unknown routine"),
    ("""  subroutine run()
    use st, only : np
    implicit none
    np = 2
  end subroutine
""", "parameter np"),
    ("""  subroutine run()
    use st, only : nx, ny, cnt, a
    implicit none
    @parallelRegion{domName(i,j), domSize(nx,ny), reduce(+:cnt)}
    cnt = cnt + 1
    @end parallelRegion
  end subroutine
""", "reduce needs"),
    (_region("    a(i,j) = a(i,j) ** 0.5_r_size"), "real exponent"),
])
def test_generator_refuses(body, msg):
    with pytest.raises(GenError) as ei:
        _gen(body)
    assert msg in str(ei.value)


def test_cpu_only_region_becomes_host_loops():
    body = """  subroutine run()
    use st, only : nx, ny, a
    implicit none
    integer(4) :: i
    integer(4) :: j
    @parallelRegion{appliesTo(CPU), domName(i,j), domSize(nx,ny)}
    a(i,j) = 2.0_r_size
    @end parallelRegion
  end subroutine
"""
    code = _gen(body)
    assert "__global__ void __launch_bounds__(128) hfk" not in code  # no kernel
    # last domain outermost (codegen.cpp:335-342)
    host = code[code.index("void host_run(Run& R) {"):]
    assert host.index("l_j = INT64_C(1)") < host.index("l_i = INT64_C(1)")


# ---- built plugins export their descriptor -------------------------------------------------
class _Desc(ctypes.Structure):
    _fields_ = [("abi", ctypes.c_int), ("program", ctypes.c_char_p),
                ("module", ctypes.c_char_p), ("scalars", ctypes.c_void_p),
                ("arrays", ctypes.c_void_p), ("entries", ctypes.POINTER(ctypes.c_char_p)),
                ("transfer_entries", ctypes.POINTER(ctypes.c_char_p)),
                ("run", ctypes.c_void_p)]


def _strings(p):
    out, k = [], 0
    while p[k]:
        out.append(p[k].decode())
        k += 1
    return out


@pytest.mark.parametrize("name,module,entries", [
    ("dycore_gen", "dyn_state", {"main", "main_full", "main_rk3", "dycore_step"}),
    ("kitchen_gen", "kit_state", {"main"}),
    ("surface_flux_gen", "sf_state", {"main", "setup", "simulation_run", "physics_run"}),
    ("reduction_gen", "red_state", {"main", "grid_total", "simulation_run"}),
])
def test_plugin_descriptor(name, module, entries):
    so = hfc.GEN_DIR / f"{name}.so"
    if not so.exists():
        pytest.skip(f"{so.name} not built")
    ctypes.CDLL(str(ROOT / "paper_1710_08616_b200" / "libhfb.so"), mode=ctypes.RTLD_GLOBAL)
    lib = ctypes.CDLL(str(so))
    lib.hfb_plugin.restype = ctypes.POINTER(_Desc)
    d = lib.hfb_plugin().contents
    assert d.abi == 1 and d.program.decode() == name and d.module.decode() == module
    got = set(_strings(d.entries))
    assert entries <= got
    # routines taking arguments are not entries (physics_main(i, j, swind))
    assert "physics_main" not in got
    assert set(_strings(d.transfer_entries)) <= got


def test_return_and_stop_statements():
    from paper_1710_08616_b200.hfc.parse import Return, Stop
    body = """  subroutine run()
    use st, only : nx, ny, a
    implicit none
    @domainDependant{attribute(autoDom, present)}
    a
    @end domainDependant
    @parallelRegion{domName(i,j), domSize(nx,ny)}
    if (i .EQ. nx) then
      return
    end if
    a(i,j) = 1.0_r_size
    @end parallelRegion
  end subroutine

  subroutine main()
    implicit none
    call run()
    stop 3
  end subroutine
"""
    code = _gen(body)
    # a kernel thread's return is counted like the launch guard (exec_launch)
    assert "atomicAdd(hfc_ret, 1ULL); return;" in code
    assert "throw HfcStop{3};" in code
    with pytest.raises(GenError):  # stop inside device code
        _gen(_region("    stop"))


def test_checked_build_uses_checked_accessors():
    """`hfc --checked` and the normal build come from one translation: array reads and
    writes go through HFC_RD / HFC_WR, which the checked build (-DHFC_CHECKED) maps to
    the bounds/init-checking accessors and the normal build to plain element access."""
    code = _gen(_region("    a(i,j) = a(i,j) + 1.0_r_size"))
    assert "HFC_WR(a, 0, i, j) = " in code and "HFC_RD(a, 0, i, j)" in code
    assert 'kNames[] = {"a"}' in code
    assert "#define HFC_RD(v, nm, ...) (v).at(__VA_ARGS__)" in code
