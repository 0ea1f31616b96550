"""Parser of the Hybrid-Fortran dialect (the reference's `.h90` input, SPEC.md §3) into a
small AST for the sm_100a code generator (gen.py).

Covered: modules with `integer(4)` / `real(r_size)` / `logical` scalars and arrays
(bounds `n` or `lo:hi`), `contains` routines with dummy arguments and `intent`,
`use m, only : ...`, `@domainDependant{...}` / `@parallelRegion{...}` blocks, block `if`
/ `else if` / `else`, counted `do` loops, `call`, assignments, and expressions with the
reference parser's precedence and associativity (`.or.` < `.and.` < `.not.` <
comparisons < `+ -` (left) < `* /` (left) < unary `-` < `**` (right);
/root/reference/proj/src/parser.cpp:95-211). Names are case-insensitive (lower-cased,
as MachineState keys are). Continuations (`&`) and `!` comments are merged first.
"""
import re
from dataclasses import dataclass, field


class ParseError(ValueError):
    pass


# ---- AST -------------------------------------------------------------------------------
@dataclass
class Num:
    text: str       # as written (without kind suffix)
    is_real: bool


@dataclass
class Name:
    name: str


@dataclass
class Ref:          # array element or function call: name(args)
    name: str
    args: list


@dataclass
class Un:
    op: str         # '-', '+', '.not.'
    x: object


@dataclass
class Bin:
    op: str         # + - * / ** .eq. .ne. .lt. .le. .gt. .ge. .and. .or.
    a: object
    b: object


@dataclass
class Logical:
    value: bool


@dataclass
class Assign:
    lhs: object     # Name or Ref
    rhs: object
    line: int


@dataclass
class Call:
    name: str
    args: list
    line: int


@dataclass
class Do:
    var: str
    lo: object
    hi: object
    body: list
    line: int


@dataclass
class If:
    branches: list  # [(cond or None, body)]
    line: int


@dataclass
class Return:       # leaves the routine (a kernel thread: counted like a guard return)
    line: int


@dataclass
class Stop:         # ends the program run (interp.cpp StopSignal)
    code: int
    line: int


@dataclass
class Region:
    attrs: dict     # domname: [..], domsize: [(lo, hi) exprs], startat, endat, reduce
    body: list
    line: int


@dataclass
class Decl:
    name: str
    type: str       # 'int' | 'real' | 'logical'
    dims: list      # [(lo_expr, hi_expr)] ; empty for scalars
    intent: str = ""
    param: object = None  # value expression of a `parameter`


@dataclass
class DomDep:
    names: list
    attrs: dict     # attribute: set(...), domname/domsize lists


@dataclass
class Routine:
    name: str
    args: list
    decls: dict = field(default_factory=dict)
    uses: dict = field(default_factory=dict)    # name -> module
    domdeps: list = field(default_factory=list)
    body: list = field(default_factory=list)


@dataclass
class Module:
    name: str
    decls: dict = field(default_factory=dict)
    routines: dict = field(default_factory=dict)


# ---- lexical helpers ---------------------------------------------------------------------
def logical_lines(text):
    """(line number, text) with comments stripped and continuations merged."""
    out, buf, start = [], "", 0
    for no, raw in enumerate(text.splitlines(), 1):
        s = raw.split("!", 1)[0].rstrip()
        st = s.strip()
        if not st:
            if buf:
                continue
            continue
        if buf:
            if st.startswith("&"):
                st = st[1:].lstrip()
            buf += " " + st
        else:
            buf, start = st, no
        if buf.endswith("&"):
            buf = buf[:-1].rstrip()
            continue
        out.append((start, buf))
        buf = ""
    if buf:
        out.append((start, buf))
    return out


_TOK = re.compile(r"""
    (?P<num>(\d+\.\d*|\.\d+|\d+)([eEdD][+-]?\d+)?(_[a-zA-Z_]\w*)?)
  | (?P<dot>\.(eq|ne|lt|le|gt|ge|and|or|not|true|false)\.)
  | (?P<name>[a-zA-Z_]\w*)
  | (?P<op>\*\*|==|/=|<=|>=|[-+*/(),:<>=%])
  | (?P<ws>\s+)
""", re.VERBOSE | re.IGNORECASE)


def tokenize(s, line):
    toks, pos = [], 0
    while pos < len(s):
        m = _TOK.match(s, pos)
        if not m:
            raise ParseError(f"line {line}: unexpected character {s[pos]!r}")
        pos = m.end()
        kind = m.lastgroup
        if kind == "ws":
            continue
        v = m.group(kind)
        if kind in ("name", "dot"):
            v = v.lower()
        toks.append((kind, v))
    return toks


class Expr:
    """Recursive descent over one token list (the reference parser's precedence)."""
    REL = {"==": ".eq.", "/=": ".ne.", "<": ".lt.", "<=": ".le.", ">": ".gt.", ">=": ".ge.",
           ".eq.": ".eq.", ".ne.": ".ne.", ".lt.": ".lt.", ".le.": ".le.", ".gt.": ".gt.",
           ".ge.": ".ge."}

    def __init__(self, toks, line):
        self.t, self.i, self.line = toks, 0, line

    def peek(self, k=0):
        return self.t[self.i + k] if self.i + k < len(self.t) else (None, None)

    def take(self, v=None):
        tok = self.peek()
        if tok[0] is None or (v is not None and tok[1] != v):
            raise ParseError(f"line {self.line}: expected {v!r}, got {tok[1]!r}")
        self.i += 1
        return tok

    def at_end(self):
        return self.i >= len(self.t)

    def parse(self):
        e = self.or_()
        return e

    def or_(self):
        a = self.and_()
        while self.peek()[1] == ".or.":
            self.take()
            a = Bin(".or.", a, self.and_())
        return a

    def and_(self):
        a = self.not_()
        while self.peek()[1] == ".and.":
            self.take()
            a = Bin(".and.", a, self.not_())
        return a

    def not_(self):
        if self.peek()[1] == ".not.":
            self.take()
            return Un(".not.", self.not_())
        return self.rel()

    def rel(self):
        a = self.add()
        op = self.peek()[1]
        if op in self.REL:
            self.take()
            a = Bin(self.REL[op], a, self.add())
        return a

    def add(self):
        a = self.mul()
        while self.peek()[1] in ("+", "-"):
            op = self.take()[1]
            a = Bin(op, a, self.mul())
        return a

    def mul(self):
        a = self.unary()
        while self.peek()[1] in ("*", "/"):
            op = self.take()[1]
            a = Bin(op, a, self.unary())
        return a

    def unary(self):
        if self.peek()[1] in ("-", "+"):
            op = self.take()[1]
            return Un(op, self.unary())
        return self.power()

    def power(self):
        a = self.primary()
        if self.peek()[1] == "**":
            self.take()
            a = Bin("**", a, self.unary())  # right associative
        return a

    def primary(self):
        kind, v = self.peek()
        if kind == "num":
            self.take()
            text = v.split("_")[0]
            is_real = any(ch in text for ch in ".eEdD") or "_" in v
            return Num(text.replace("d", "e").replace("D", "e"), is_real)
        if kind == "dot" and v in (".true.", ".false."):
            self.take()
            return Logical(v == ".true.")
        if kind == "name":
            self.take()
            if self.peek()[1] == "(":
                self.take("(")
                args = []
                if self.peek()[1] != ")":
                    args.append(self.slice_or_expr())
                    while self.peek()[1] == ",":
                        self.take()
                        args.append(self.slice_or_expr())
                self.take(")")
                return Ref(v, args)
            return Name(v)
        if v == "(":
            self.take()
            e = self.parse()
            self.take(")")
            return e
        raise ParseError(f"line {self.line}: unexpected token {v!r}")

    def slice_or_expr(self):
        return self.parse()


def parse_expr(s, line):
    p = Expr(tokenize(s, line), line)
    e = p.parse()
    if not p.at_end():
        raise ParseError(f"line {line}: trailing tokens in {s!r}")
    return e


def split_top(s, sep=","):
    """Split on `sep` outside parentheses/braces."""
    out, depth, cur = [], 0, ""
    for ch in s:
        if ch in "({":
            depth += 1
        elif ch in ")}":
            depth -= 1
        if ch == sep and depth == 0:
            out.append(cur.strip())
            cur = ""
        else:
            cur += ch
    if cur.strip():
        out.append(cur.strip())
    return out


def parse_dims(s, line):
    """`nz, 0:nx, ny` -> [(lo, hi)] with lo defaulting to 1."""
    dims = []
    for d in split_top(s):
        if ":" in d:
            lo, hi = d.split(":", 1)
            dims.append((parse_expr(lo, line), parse_expr(hi, line)))
        else:
            dims.append((Num("1", False), parse_expr(d, line)))
    return dims


def parse_attrs(s, line):
    """`domName(i,j), domSize(nx,ny), attribute(autoDom, present)` -> dict"""
    attrs = {}
    for a in split_top(s):
        m = re.match(r"(\w+)\s*\((.*)\)$", a.strip(), re.S)
        if not m:
            raise ParseError(f"line {line}: bad directive attribute {a!r}")
        key, val = m.group(1).lower(), m.group(2)
        attrs[key] = [x.strip() for x in split_top(val)]
    return attrs


_DECL = re.compile(r"^(integer\s*\(\s*4\s*\)|real\s*\(\s*r_size\s*\)|logical|type\s*\(\s*dim3\s*\))"
                   r"\s*(,\s*intent\s*\(\s*(in|out|inout)\s*\))?(\s*,\s*parameter)?\s*::\s*(.*)$",
                   re.I)


def parse_decl(text, line):
    m = _DECL.match(text)
    if not m:
        return None
    t = m.group(1).lower().replace(" ", "")
    typ = "int" if t.startswith("integer") else "real" if t.startswith("real") else (
        "logical" if t == "logical" else "dim3")
    intent = (m.group(3) or "").lower()
    is_param = m.group(4) is not None
    out = []
    for item in split_top(m.group(5)):
        mm = re.match(r"(\w+)\s*(\((.*)\))?\s*(=\s*(.*))?$", item.strip(), re.S)
        if not mm:
            raise ParseError(f"line {line}: bad declaration {item!r}")
        dims = parse_dims(mm.group(3), line) if mm.group(3) else []
        d = Decl(mm.group(1).lower(), typ, dims, intent)
        if is_param:
            if mm.group(5) is None or dims:
                raise ParseError(f"line {line}: a parameter needs a scalar value")
            d.param = parse_expr(mm.group(5), line)
        out.append(d)
    return out


class Parser:
    def __init__(self, text, path="<src>"):
        self.lines = logical_lines(text)
        self.i = 0
        self.path = path

    def err(self, msg, line=None):
        ln = line if line is not None else (self.lines[self.i][0] if self.i < len(self.lines) else -1)
        raise ParseError(f"{self.path}:{ln}: {msg}")

    def next(self):
        if self.i >= len(self.lines):
            self.err("unexpected end of file")
        ln, t = self.lines[self.i]
        self.i += 1
        return ln, t

    def peek(self):
        return self.lines[self.i] if self.i < len(self.lines) else (None, None)

    def modules(self):
        mods = {}
        while self.i < len(self.lines):
            ln, t = self.next()
            m = re.match(r"module\s+(\w+)$", t, re.I)
            if not m:
                self.err(f"expected 'module', got {t!r}", ln)
            mod = Module(m.group(1).lower())
            self.module_body(mod)
            mods[mod.name] = mod
        return mods

    def module_body(self, mod):
        while True:
            ln, t = self.next()
            low = t.lower()
            if re.match(r"end\s*module", low):
                return
            if low == "implicit none":
                continue
            if low == "contains":
                while True:
                    ln, t = self.peek()
                    if t is None:
                        self.err("missing 'end module'")
                    if re.match(r"end\s*module", t.lower()):
                        self.next()
                        return
                    r = self.routine()
                    mod.routines[r.name] = r
            d = parse_decl(t, ln)
            if d is None:
                self.err(f"unexpected module statement {t!r}", ln)
            for x in d:
                mod.decls[x.name] = x

    def routine(self):
        ln, t = self.next()
        m = re.match(r"subroutine\s+(\w+)\s*(\((.*)\))?$", t, re.I)
        if not m:
            self.err(f"expected 'subroutine', got {t!r}", ln)
        args = [a.strip().lower() for a in (m.group(3) or "").split(",") if a.strip()]
        r = Routine(m.group(1).lower(), args)
        r.body = self.block(r, ("end subroutine",))
        self.next()
        return r

    def block(self, r, enders):
        """statements until a line starting with one of `enders` (consumed)."""
        out = []
        while True:
            ln, t = self.peek()
            if t is None:
                self.err(f"missing {enders[0]!r}")
            low = t.lower()
            for e in enders:
                if re.match(e.replace(" ", r"\s*") + r"\b", low):
                    return out
            self.next()
            if low == "implicit none":
                continue
            m = re.match(r"use\s+(\w+)\s*,\s*only\s*:\s*(.*)$", low)
            if m:
                for n in split_top(m.group(2)):
                    r.uses[n.strip()] = m.group(1)
                continue
            d = parse_decl(t, ln)
            if d is not None:
                for x in d:
                    r.decls[x.name] = x
                continue
            if low.startswith("@domaindependant"):
                attrs = parse_attrs(t[t.index("{") + 1:t.rindex("}")], ln)
                names = []
                while True:
                    ln2, t2 = self.next()
                    if t2.lower().startswith("@end domaindependant"):
                        break
                    names += [n.strip().lower() for n in split_top(t2)]
                r.domdeps.append(DomDep(names, {k.lower(): [v.lower() for v in vs]
                                                for k, vs in attrs.items()}))
                continue
            if low.startswith("@parallelregion"):
                attrs = parse_attrs(t[t.index("{") + 1:t.rindex("}")], ln)
                body = self.block(r, ("@end parallelregion",))
                self.next()
                out.append(Region({k: v for k, v in attrs.items()}, body, ln))
                continue
            out.append(self.statement(r, ln, t))

    def statement(self, r, ln, t):
        low = t.lower()
        m = re.match(r"do\s+(\w+)\s*=\s*(.*)$", low)
        if m:
            bounds = split_top(m.group(2))
            if len(bounds) != 2:
                self.err("only `do v = lo, hi` loops (no strides, parser.cpp:648-649)", ln)
            body = self.block(r, ("end do", "enddo"))
            self.next()
            return Do(m.group(1), parse_expr(bounds[0], ln), parse_expr(bounds[1], ln), body, ln)
        m = re.match(r"if\s*\((.*)\)\s*then$", low)
        if m:
            branches = []
            cond = parse_expr(m.group(1), ln)
            while True:
                body = self.block(r, ("else if", "elseif", "else", "end if", "endif"))
                branches.append((cond, body))
                ln2, t2 = self.next()
                l2 = t2.lower()
                mm = re.match(r"else\s*if\s*\((.*)\)\s*then$", l2)
                if mm:
                    cond = parse_expr(mm.group(1), ln2)
                    continue
                if l2 == "else":
                    body = self.block(r, ("end if", "endif"))
                    self.next()
                    branches.append((None, body))
                return If(branches, ln)
        if low == "return":
            return Return(ln)
        m = re.match(r"stop(\s+(\d+))?$", low)
        if m:
            return Stop(int(m.group(2)) if m.group(2) else 0, ln)
        m = re.match(r"call\s+(\w+)\s*(\((.*)\))?$", low)
        if m:
            args = [parse_expr(a, ln) for a in split_top(m.group(3) or "")] if m.group(3) else []
            return Call(m.group(1), args, ln)
        parts = split_top(t, "=")
        if len(parts) == 2 and not re.search(r"[<>/=]$", parts[0]):
            return Assign(parse_expr(parts[0], ln), parse_expr(parts[1], ln), ln)
        self.err(f"unsupported statement {t!r}", ln)


def parse_program(sources):
    """sources: [(path, text)] -> {module name: Module}"""
    mods = {}
    for path, text in sources:
        mods.update(Parser(text, path).modules())
    return mods
