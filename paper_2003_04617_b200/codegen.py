"""Generic compilation of scalar reversible programs to one CUDA kernel
(the paper's "compile reversible programs to GPU
kernels" claim).

A function of the reference DSL over scalar cells — Float, ULog (log-domain)
and Int — is compiled to a batched kernel: one thread per argument row runs
the function forward (reference `run_function`), then its inverse in
gradient mode with the adjoint rules (reference `uncall_function` with
GVar cells, autodiff.py:136-180), every reversibility check on device.  The
generated code restates the reference interpreter's semantics:

  inversion and routine expansion  reverser.py:23-163
  statement checks                 interpreter.py:713-885 (If post == pre,
                                   While post false at entry / true after
                                   each iteration, For range and iterator,
                                   ancilla release |v - decl| <= tol)
  primal instructions              numerics.py:296-368 (_plus_minus_plain,
                                   _mul_div_plain, _log_contribution)
  adjoint rules                    numerics.py:419-505 (_g_accum,
                                   _plus_minus_adjoint, _mul_div_adjoint)
  partials                         numerics.py:70-118 (INSTR_FNS)
  conditions                       interpreter.py:200-300 (ULog compares as
                                   exp(log_x), Int % as Python's modulo)

The subset: Float / Int / Complex / Fixed scalar parameters (Float rows;
Int values uniform over the batch; Complex as re/im leaves with field views;
Fixed as raw int64 Q31.32 cells with `0.5fx` literals: + / - wrap mod 2^64,
a Float value enters through from_real, cotangents are Fixed and quantized
at every accumulation, values.py:28-86 / numerics.py:305-306, 419-428),
fixed-shape Float arrays (parameters and ancilla-free array arguments),
Float / ULog / Int / Fixed ancillas, `+= -= *= /=` instructions with the
INSTR_FNS functions, `xor=` on Int cells, calls between compiled functions
(inlined; recursive calls level by level up to REVGPU_CODEGEN_DEPTH, past
which the kernel reports the interpreter's RecursionError), bijector-view
call arguments over Int cells (`k |> addconst(-1)`: copy in through fwd,
write back through inv), `<-` / `->`, @routine / ~@routine, @invcheckoff,
for / while / if.  Records and Fixed arithmetic inside expressions are
rejected at compile time (UnsupportedProgram), as are the static aliasing
patterns the reference rejects at run time (AliasedArguments).

The kernel is built with nvcc for sm_100a into a cache directory
($REVGPU_CODEGEN_CACHE, default paper_2003_04617_b200/_codegen_cache) and bound with
ctypes; libdevice's exp/log/sin/cos/pow stand for the host libm (<= 1-2 ulp).
"""

import ctypes
import hashlib
import math
import os
import re
import subprocess
import tempfile
from dataclasses import dataclass

import numpy as np
import torch

from .errors import AliasedArguments, KindError, NativeLibraryError, UnsupportedProgram

# ---------------------------------------------------------------------------
# tokens
# ---------------------------------------------------------------------------

_PUNCT2 = ("<-", "->", "+=", "-=", "*=", "/=", "==", "!=", "<=", ">=", "&&", "||", "::", "|>")
_PUNCT1 = "()[],.:+-*/^%<>=~"
_KEYWORDS = {"fn", "end", "if", "else", "while", "for", "begin", "true", "false"}


def _tokenize(src):
    toks = []
    i, n = 0, len(src)
    while i < n:
        c = src[i]
        if c in " \t\r\n":
            i += 1
            continue
        if c == "#":
            while i < n and src[i] != "\n":
                i += 1
            continue
        if c == "@" or (c == "~" and src.startswith("~@", i)):
            j = i + (2 if c == "~" else 1)
            while j < n and (src[j].isalnum() or src[j] == "_"):
                j += 1
            word = src[i:j]
            if word not in ("@routine", "~@routine", "@safe", "@invcheckoff"):
                raise UnsupportedProgram(f"codegen: macro {word!r} is not supported")
            toks.append(("macro", word))
            i = j
            continue
        if c.isalpha() or c == "_":
            j = i
            while j < n and (src[j].isalnum() or src[j] == "_"):
                j += 1
            while j < n and src[j] == "!" and not (j + 1 < n and src[j + 1] == "="):
                j += 1
            if src[i:j] == "xor" and j < n and src[j] == "=" and not src.startswith("==", j):
                toks.append(("punct", "xor="))               # parser.py:92-100
                i = j + 1
                continue
            toks.append(("name", src[i:j]))
            i = j
            continue
        if c == "\u22bb" and src.startswith("=", i + 1):  # the Unicode spelling of xor=
            toks.append(("punct", "xor="))
            i += 2
            continue
        if c.isdigit() or (c == "." and i + 1 < n and src[i + 1].isdigit()):
            j = i
            is_float = False
            while j < n and src[j].isdigit():
                j += 1
            if j < n and src[j] == "." and j + 1 < n and src[j + 1].isdigit():
                is_float = True
                j += 1
                while j < n and src[j].isdigit():
                    j += 1
            if j < n and src[j] in "eE" and (
                    (j + 1 < n and src[j + 1].isdigit())
                    or (j + 2 < n and src[j + 1] in "+-" and src[j + 2].isdigit())):
                is_float = True
                j += 2
                while j < n and src[j].isdigit():
                    j += 1
            k = j
            while k < n and src[k].isalpha():
                k += 1
            body, suffix = src[i:j], src[j:k]
            if suffix == "fx":                     # parser.py:133
                toks.append(("num", FixLit(_fx_from_real(float(body)))))
            elif suffix:
                raise UnsupportedProgram("codegen: imaginary literals are not supported")
            else:
                toks.append(("num", float(body) if is_float else int(body)))
            i = k
            continue
        two = src[i:i + 2]
        if two in _PUNCT2:
            toks.append(("punct", two))
            i += 2
            continue
        if c in _PUNCT1:
            toks.append(("punct", c))
            i += 1
            continue
        raise UnsupportedProgram(f"codegen: unexpected character {c!r}")
    toks.append(("eof", None))
    return toks


# ---------------------------------------------------------------------------
# IR (scalar subset)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Lit:
    v: object


_FX_WRAP, _FX_SIGN = 1 << 64, 1 << 63


def _fx_wrap(raw):
    """values._wrap64: two's-complement wrap of a Q31.32 raw value."""
    raw &= _FX_WRAP - 1
    return raw - _FX_WRAP if raw & _FX_SIGN else raw


def _fx_from_real(v):
    """values.Fixed.from_real: round(float(v) * 2^32), half-even, wrapped."""
    return _fx_wrap(round(float(v) * (1 << 32)))


@dataclass(frozen=True)
class FixLit:
    """A Fixed (Q31.32) literal (parser.py:133: `1.5fx` = Fixed.from_real(1.5))."""
    raw: int

    def __neg__(self):
        return FixLit(_fx_wrap(-self.raw))

    def real(self):
        return self.raw / (1 << 32)          # values.Fixed.to_float (correctly rounded)


@dataclass(frozen=True)
class Var:
    name: str


@dataclass(frozen=True)
class IView:
    name: str
    idx: tuple             # Int index expressions (1-based)


@dataclass(frozen=True)
class NoCheck:
    """@invcheckoff stmt: the statement (and every call it makes) runs with
    the reversibility checks off (interpreter.py InvCheckOff, _checking)."""
    body: tuple


@dataclass(frozen=True)
class FView:
    """x.re / x.im of a Complex cell (a Float leaf)."""
    name: str
    field: str


@dataclass(frozen=True)
class Safe:
    kind: str              # "assert" | "print"
    exprs: tuple


@dataclass(frozen=True)
class PCall:
    """A statement call: a primitive (SWAP / ROT / IROT / NEG / INC / DEC) or
    a user function, `uncall` for the ~f(...) form (reference FnCall /
    UncallFn, reverser.py:96-103)."""
    f: str
    args: tuple            # views
    uncall: bool = False


@dataclass(frozen=True)
class ArgCheck:
    """Entry checks of an inlined call (interpreter.py:969-978): the strict
    alias pairs over its argument views, then their reads (bounds)."""
    views: tuple


# numerics.py:189-193: name -> number of constant arguments
BIJECTORS = {"neg": 0, "addconst": 1, "mulconst": 1}


@dataclass(frozen=True)
class BView:
    """`base |> bij(c...)` (ir.BijView): a call argument the callee reads as
    bij.fwd(base) and writes back through bij.inv (interpreter.py:565-583);
    storage identity is the base's (bijectors do not change identity)."""
    base: object
    bij: str
    args: tuple

    @property
    def name(self):
        return self.base.name

    def root(self):
        return self.base.root() if isinstance(self.base, BView) else self.base


@dataclass(frozen=True)
class BijIn:
    """Copy-in of a bijector-view argument into the callee's cell `tmp`."""
    tmp: str
    view: BView


@dataclass(frozen=True)
class BijOut:
    """Write-back of the callee's cell `tmp` through the view's inverses."""
    tmp: str
    view: BView


@dataclass(frozen=True)
class DepthErr:
    """A recursive call past the compiled inlining depth (RecursionError)."""


# numerics.py:30-33
PRIM_ARITY = {"SWAP": 2, "ROT": 3, "IROT": 3, "NEG": 1, "INC": 1, "DEC": 1}
PRIM_INV = {"SWAP": "SWAP", "ROT": "IROT", "IROT": "ROT", "NEG": "NEG", "INC": "DEC", "DEC": "INC"}


@dataclass(frozen=True)
class Un:
    op: str
    e: object


@dataclass(frozen=True)
class Bin:
    op: str
    l: object
    r: object


@dataclass(frozen=True)
class Call:
    f: str
    args: tuple


@dataclass(frozen=True)
class Instr:
    op: str
    target: object         # Var / IView
    fname: str
    args: tuple            # Lit / Var atoms


@dataclass(frozen=True)
class Alloc:
    name: str
    e: object


@dataclass(frozen=True)
class Dealloc:
    name: str
    e: object


@dataclass(frozen=True)
class RBegin:
    body: tuple


@dataclass(frozen=True)
class REnd:
    pass


@dataclass(frozen=True)
class For:
    var: str
    a: object
    s: object
    b: object
    body: tuple


@dataclass(frozen=True)
class While:
    pre: object
    post: object
    body: tuple


SAME = "~"     # If post == pre (re-evaluated after the branch)


@dataclass(frozen=True)
class If:
    pre: object
    post: object
    then: tuple
    els: tuple


_INSTR_BIN = {"+": "add", "-": "sub", "*": "mul", "/": "div", "^": "pow"}


class _Parser:
    def __init__(self, src):
        # the reference's Unicode spellings of the arrows (parser.py:143-164)
        self.t = _tokenize(src.replace("\u2190", "<-").replace("\u2192", "->"))
        self.i = 0
        self.arrays = {}

    @property
    def cur(self):
        return self.t[self.i]

    def peek(self, k=1):
        return self.t[min(self.i + k, len(self.t) - 1)]

    def adv(self):
        tok = self.t[self.i]
        self.i += 1
        return tok

    def at(self, kind, val=None):
        return self.cur[0] == kind and (val is None or self.cur[1] == val)

    def expect(self, kind, val=None):
        if not self.at(kind, val):
            raise UnsupportedProgram(f"codegen: expected {val or kind}, found {self.cur[1]!r}")
        return self.adv()

    def name(self):
        tok = self.expect("name")
        if tok[1] in _KEYWORDS:
            raise UnsupportedProgram(f"codegen: unexpected keyword {tok[1]!r}")
        return tok[1]

    def program(self):
        fns = {}
        while not self.at("eof"):
            self.expect("name", "fn")
            fname = self.name()
            self.expect("punct", "(")
            params = []
            arrays = set()
            while not self.at("punct", ")"):
                pn = self.name()
                params.append(pn)
                if self.at("punct", "::"):
                    self.adv()
                    if self.name() != "array":
                        raise UnsupportedProgram("codegen: only ::array parameters are supported")
                    arrays.add(pn)
                if self.at("punct", ","):
                    self.adv()
            self.adv()
            body = self.block(("end",))
            self.expect("name", "end")
            fns[fname] = (tuple(params), body)
            self.arrays[fname] = arrays
        return fns

    def block(self, stops):
        out = []
        while not (self.at("eof") or (self.cur[0] == "name" and self.cur[1] in stops)):
            out.append(self.stmt())
        return tuple(out)

    def stmt(self):
        if self.at("macro", "@routine"):
            self.adv()
            inner = self.stmt()
            return RBegin(inner if isinstance(inner, tuple) else (inner,))
        if self.at("macro", "~@routine"):
            self.adv()
            return REnd()
        if self.at("macro", "@invcheckoff"):
            self.adv()
            inner = self.stmt()
            return NoCheck(inner if isinstance(inner, tuple) else (inner,))
        if self.at("macro", "@safe"):
            self.adv()
            kind = self.name()
            if kind not in ("assert", "print"):
                raise UnsupportedProgram("codegen: @safe takes assert(...) or print(...)")
            self.expect("punct", "(")
            exprs = []
            while not self.at("punct", ")"):
                exprs.append(self.expr())
                if self.at("punct", ","):
                    self.adv()
            self.adv()
            return Safe(kind, tuple(exprs))
        if self.at("name", "begin"):
            self.adv()
            body = self.block(("end",))
            self.expect("name", "end")
            return body
        if self.at("name", "if"):
            self.adv()
            self.expect("punct", "(")
            pre = self.expr()
            self.expect("punct", ",")
            if self.at("punct", "~"):
                self.adv()
                post = SAME
            else:
                post = self.expr()
            self.expect("punct", ")")
            then = self.block(("else", "end"))
            els = ()
            if self.at("name", "else"):
                self.adv()
                els = self.block(("end",))
            self.expect("name", "end")
            return If(pre, post, then, els)
        if self.at("name", "while"):
            self.adv()
            self.expect("punct", "(")
            pre = self.expr()
            self.expect("punct", ",")
            post = self.expr()
            self.expect("punct", ")")
            body = self.block(("end",))
            self.expect("name", "end")
            return While(pre, post, body)
        if self.at("name", "for"):
            self.adv()
            var = self.name()
            self.expect("punct", "=")
            a = self.expr()
            self.expect("punct", ":")
            second = self.expr()
            if self.at("punct", ":"):
                self.adv()
                s, b = second, self.expr()
            else:
                s, b = Lit(1), second
            body = self.block(("end",))
            self.expect("name", "end")
            return For(var, a, s, b, body)
        if self.at("punct", "~"):
            self.adv()
            return PCall(self.name(), self.call_args(), True)
        target = self.name()
        if self.at("punct", "("):
            if target == "XOR":                         # XOR(a, b) == a xor= b (parser.py:381-384)
                views = self.call_args()
                if len(views) != 2:
                    raise UnsupportedProgram("codegen: XOR takes two arguments")
                return Instr("xor=", views[0], "identity", (views[1],))
            return PCall(target, self.call_args(), False)
        tview = self.index_tail(target)
        if self.at("punct", "<-") or self.at("punct", "->"):
            if isinstance(tview, IView):
                raise UnsupportedProgram("codegen: only a plain name can be (de)allocated")
            alloc = self.adv()[1] == "<-"
            return (Alloc if alloc else Dealloc)(target, self.expr())
        target = tview
        if self.cur[0] == "punct" and self.cur[1] in ("+=", "-=", "*=", "/=", "xor="):
            op = self.adv()[1]
            fname, args = self.instr_rhs()
            return Instr(op, target, fname, args)
        raise UnsupportedProgram(f"codegen: unsupported statement at {self.cur[1]!r}")

    def atom(self):
        if self.at("num"):
            return Lit(self.adv()[1])
        if self.at("punct", "-") and self.peek()[0] == "num":
            self.adv()
            return Lit(-self.adv()[1])
        if self.at("name", "true") or self.at("name", "false"):
            raise UnsupportedProgram("codegen: Bool cells are not supported")
        return self.index_tail(self.name())

    def call_args(self):
        self.expect("punct", "(")
        views = []
        while not self.at("punct", ")"):
            v = self.index_tail(self.name())
            while self.at("punct", "|>"):                # bijector views (numerics.py:189)
                self.adv()
                bij = self.name()
                cargs = []
                if self.at("punct", "("):
                    self.adv()
                    while not self.at("punct", ")"):
                        neg = self.at("punct", "-")
                        if neg:
                            self.adv()
                        if not self.at("num") or isinstance(self.cur[1], FixLit):
                            raise KindError("bijector arguments are numeric constants")
                        c = self.adv()[1]
                        cargs.append(-c if neg else c)
                        if self.at("punct", ","):
                            self.adv()
                    self.adv()
                if bij not in BIJECTORS:
                    raise KindError(f"no bijector named {bij!r}")
                if len(cargs) != BIJECTORS[bij] or (bij == "mulconst" and cargs[0] == 0):
                    raise KindError(f"invalid arguments for bijector {bij!r}")
                v = BView(v, bij, tuple(cargs))
            views.append(v)
            if self.at("punct", ","):
                self.adv()
        self.adv()
        return tuple(views)

    def index_tail(self, name):
        """name, name[i, j] or name.re / name.im (a view)."""
        if self.at("punct", "."):
            self.adv()
            field = self.name()
            if field not in ("re", "im"):
                raise UnsupportedProgram("codegen: records are not supported (only .re / .im)")
            return FView(name, field)
        if not self.at("punct", "["):
            return Var(name)
        self.adv()
        idx = []
        while not self.at("punct", "]"):
            idx.append(self.expr())
            if self.at("punct", ","):
                self.adv()
        self.adv()
        return IView(name, tuple(idx))

    def instr_rhs(self):
        if self.cur[0] == "name" and self.cur[1] not in _KEYWORDS and self.peek() == ("punct", "("):
            f = self.adv()[1]
            self.expect("punct", "(")
            atoms = []
            while not self.at("punct", ")"):
                atoms.append(self.atom())
                if self.at("punct", ","):
                    self.adv()
            self.adv()
            return f, tuple(atoms)
        if self.at("punct", "-"):
            self.adv()
            a = self.atom()
            if isinstance(a, Lit):
                return "identity", (Lit(-a.v),)
            return "neg", (a,)
        first = self.atom()
        if self.cur[0] == "punct" and self.cur[1] in _INSTR_BIN:
            op = self.adv()[1]
            return _INSTR_BIN[op], (first, self.atom())
        return "identity", (first,)

    # conditions / bounds / allocation values
    def expr(self):
        e = self.and_e()
        while self.at("punct", "||"):
            self.adv()
            e = Bin("||", e, self.and_e())
        return e

    def and_e(self):
        e = self.cmp_e()
        while self.at("punct", "&&"):
            self.adv()
            e = Bin("&&", e, self.cmp_e())
        return e

    def cmp_e(self):
        e = self.add_e()
        if self.cur[0] == "punct" and self.cur[1] in ("==", "!=", "<", "<=", ">", ">="):
            op = self.adv()[1]
            return Bin(op, e, self.add_e())
        return e

    def add_e(self):
        e = self.mul_e()
        while self.cur[0] == "punct" and self.cur[1] in ("+", "-"):
            op = self.adv()[1]
            e = Bin(op, e, self.mul_e())
        return e

    def mul_e(self):
        e = self.un_e()
        while self.cur[0] == "punct" and self.cur[1] in ("*", "/", "%"):
            op = self.adv()[1]
            e = Bin(op, e, self.un_e())
        return e

    def un_e(self):
        if self.at("punct", "-"):
            self.adv()
            inner = self.un_e()
            if isinstance(inner, Lit) and not isinstance(inner.v, bool):
                return Lit(-inner.v)
            return Un("-", inner)
        base = self.prim_e()
        if self.at("punct", "^"):
            self.adv()
            return Bin("^", base, self.un_e())
        return base

    def prim_e(self):
        if self.at("num"):
            return Lit(self.adv()[1])
        if self.at("name", "true") or self.at("name", "false"):
            return Lit(self.adv()[1] == "true")
        if self.at("punct", "("):
            self.adv()
            e = self.expr()
            self.expect("punct", ")")
            return e
        v = self.name()
        if self.at("punct", "("):
            self.adv()
            args = []
            while not self.at("punct", ")"):
                args.append(self.expr())
                if self.at("punct", ","):
                    self.adv()
            self.adv()
            return Call(v, tuple(args))
        return self.index_tail(v)


# ---------------------------------------------------------------------------
# inversion and routine expansion (reverser.py:23-163, restated)
# ---------------------------------------------------------------------------

def _neg_expr(e):
    if isinstance(e, Un) and e.op == "-":
        return e.e
    if isinstance(e, Lit) and isinstance(e.v, (int, float)) and not isinstance(e.v, bool):
        return Lit(-e.v)
    if isinstance(e, Bin) and e.op == "-" and isinstance(e.l, Lit) and e.l.v == 0:
        return e.r
    return Un("-", e)


_OP_INV = {"+=": "-=", "-=": "+=", "*=": "/=", "/=": "*=", "xor=": "xor="}


def _invert(s):
    if isinstance(s, Alloc):
        return Dealloc(s.name, s.e)
    if isinstance(s, Dealloc):
        return Alloc(s.name, s.e)
    if isinstance(s, Instr):
        return Instr(_OP_INV[s.op], s.target, s.fname, s.args)
    if isinstance(s, If):
        pre, post = (s.pre, s.post) if s.post is SAME else (s.post, s.pre)
        return If(pre, post, _invert_list(s.then), _invert_list(s.els))
    if isinstance(s, While):
        return While(s.post, s.pre, _invert_list(s.body))
    if isinstance(s, For):
        return For(s.var, s.b, _neg_expr(s.s), s.a, _invert_list(s.body))
    if isinstance(s, NoCheck):         # reverser.py: InvCheckOff(invert_statement(stmt))
        return NoCheck(_invert_list(s.body))
    if isinstance(s, Safe):
        return s                       # irreversible external statement: re-executed as is
    if isinstance(s, PCall):           # reverser.py:96-103
        if s.f in PRIM_INV:
            return PCall(PRIM_INV[s.f], s.args, False)
        return PCall(s.f, s.args, not s.uncall)
    if isinstance(s, tuple):
        return _invert_list(s)
    raise UnsupportedProgram(f"codegen: cannot invert {s!r}")


def _invert_list(stmts):
    opens, stack = {}, []
    for pos, s in enumerate(stmts):
        if isinstance(s, RBegin):
            stack.append(pos)
        elif isinstance(s, REnd):
            if not stack:
                raise UnsupportedProgram("codegen: routine close without an open")
            opens[pos] = stack.pop()
    if stack:
        raise UnsupportedProgram("codegen: routine block is never closed")
    out = []
    for pos in range(len(stmts) - 1, -1, -1):
        s = stmts[pos]
        if isinstance(s, REnd):
            out.append(RBegin(stmts[opens[pos]].body))
        elif isinstance(s, RBegin):
            out.append(REnd())
        else:
            out.append(_invert(s))
    return tuple(out)


def _expand(stmts):
    out, pending = [], []
    for s in stmts:
        if isinstance(s, RBegin):
            body = _expand(s.body)
            pending.append(body)
            out.extend(body)
        elif isinstance(s, REnd):
            if not pending:
                raise UnsupportedProgram("codegen: routine close without an open")
            out.extend(_invert_list(pending.pop()))
        elif isinstance(s, If):
            out.append(If(s.pre, s.post, _expand(s.then), _expand(s.els)))
        elif isinstance(s, While):
            out.append(While(s.pre, s.post, _expand(s.body)))
        elif isinstance(s, For):
            out.append(For(s.var, s.a, s.s, s.b, _expand(s.body)))
        elif isinstance(s, NoCheck):
            out.append(NoCheck(_expand(s.body)))
        elif isinstance(s, tuple):
            out.extend(_expand(s))
        else:
            out.append(s)
    if pending:
        raise UnsupportedProgram("codegen: routine block is never closed")
    return tuple(out)


# ---------------------------------------------------------------------------
# call inlining: a user call runs the callee's (or, for ~f, its inverse's)
# expanded body with the parameters bound to the argument views and fresh
# local names — the reference's fresh Frame per call with copy-in/copy-out
# (interpreter.py:969-989), equivalent because the strict alias check keeps
# the argument cells disjoint
# ---------------------------------------------------------------------------

def _expr_names(e, acc):
    if isinstance(e, Var):
        acc.add(e.name)
    elif isinstance(e, IView):
        acc.add(e.name)
        for x in e.idx:
            _expr_names(x, acc)
    elif isinstance(e, FView):
        acc.add(e.name)
    elif isinstance(e, Un):
        _expr_names(e.e, acc)
    elif isinstance(e, Bin):
        _expr_names(e.l, acc)
        _expr_names(e.r, acc)
    elif isinstance(e, Call):
        for x in e.args:
            _expr_names(x, acc)
    return acc


def _balanced(stmts, fname):
    """Every block releases what it allocates (else the reference raises
    DirtyAncilla for leaked bindings at the call's exit)."""
    cnt = {}
    for s in stmts:
        if isinstance(s, Alloc):
            cnt[s.name] = cnt.get(s.name, 0) + 1
        elif isinstance(s, Dealloc):
            cnt[s.name] = cnt.get(s.name, 0) - 1
        elif isinstance(s, (For, While, NoCheck)):
            _balanced(s.body, fname)
        elif isinstance(s, If):
            _balanced(s.then, fname)
            _balanced(s.els, fname)
    if any(cnt.values()):
        raise UnsupportedProgram(f"codegen: {fname} does not release every ancilla it allocates "
                                 "in the same block")


_MAX_DEPTH = int(os.environ.get("REVGPU_CODEGEN_DEPTH", "24"))   # inlined recursion levels
_MAX_INLINED = 4096                                   # inlined calls per generated kernel


def _unwrap(v):
    """The storage view under bijector views (their identity, interpreter.py:619)."""
    while isinstance(v, BView):
        v = v.base
    return v


class _Inliner:
    def __init__(self, fns):
        self.fns = fns
        self.n = 0

    def run(self, stmts, stack=()):
        out = []
        for s in stmts:
            if isinstance(s, PCall) and s.f not in PRIM_ARITY:
                out.extend(self.call(s, stack))
            elif isinstance(s, For):
                out.append(For(s.var, s.a, s.s, s.b, self.run(s.body, stack)))
            elif isinstance(s, While):
                out.append(While(s.pre, s.post, self.run(s.body, stack)))
            elif isinstance(s, If):
                out.append(If(s.pre, s.post, self.run(s.then, stack), self.run(s.els, stack)))
            elif isinstance(s, NoCheck):
                out.append(NoCheck(self.run(s.body, stack)))
            else:
                out.append(s)
        return tuple(out)

    def writes(self, fname, param, uncall, stack):
        """May function `fname` (its inverse when `uncall`) write `param`?
        Instruction targets, primitive and call arguments (followed into the
        callee), (de)allocations and loop variables are writes."""
        if fname not in self.fns or fname in stack[:-1]:
            return True
        params, body = self.fns[fname]

        def touched(ss):
            for st in ss:
                if isinstance(st, Instr) and st.target.name == param:
                    return True
                if isinstance(st, (Alloc, Dealloc)) and st.name == param:
                    return True
                if isinstance(st, For) and (st.var == param or touched(st.body)):
                    return True
                if isinstance(st, While) and touched(st.body):
                    return True
                if isinstance(st, If) and (touched(st.then) or touched(st.els)):
                    return True
                if isinstance(st, (RBegin, NoCheck)) and touched(st.body):
                    return True
                if isinstance(st, tuple) and touched(st):
                    return True
                if isinstance(st, PCall):
                    for q, a in zip(self.fns.get(st.f, ((),))[0] if st.f not in PRIM_ARITY
                                    else [None] * len(st.args), st.args):
                        if a.name != param:
                            continue
                        if st.f in PRIM_ARITY or q is None or \
                                self.writes(st.f, q, st.uncall, stack + (st.f,)):
                            return True
            return False
        return touched(body)

    def call(self, s, stack):
        if s.f not in self.fns:
            raise UnsupportedProgram(f"codegen: no function named {s.f!r}")
        if stack.count(s.f) >= _MAX_DEPTH:
            # recursion is inlined level by level (a fresh copy of the body per
            # level); a call past the compiled depth is the interpreter's
            # RecursionError when it runs
            return (ArgCheck(tuple(_unwrap(a) for a in s.args)), DepthErr())
        params, body = self.fns[s.f]
        if len(params) != len(s.args):
            raise KindError(f"{s.f} takes {len(params)} arguments, got {len(s.args)}")
        # a view argument whose index reads another argument of the call is
        # exact when inlined only if the callee never writes that parameter
        # (the reference re-evaluates the index when it writes the view back)
        for a in s.args:
            if not isinstance(a, IView):
                continue
            used = _expr_names(Call("", a.idx), set())
            for q, b in zip(params, s.args):
                if isinstance(b, Var) and b.name in used and \
                        self.writes(s.f, q, s.uncall, stack + (s.f,)):
                    raise UnsupportedProgram("codegen: an argument's index uses an argument the "
                                             "callee writes")
        body = _expand(_invert_list(body) if s.uncall else body)
        _balanced(body, s.f)
        self.n += 1
        if self.n > _MAX_INLINED:
            raise UnsupportedProgram(f"codegen: more than {_MAX_INLINED} inlined calls (a recursion "
                                     "with several call sites per level grows exponentially)")
        args, pre, post = [], [], []
        for a in s.args:                     # bijector views: copy in, run, write back
            if isinstance(a, BView):
                tmp = f"__bv{self.n}_{len(pre)}"
                pre.append(BijIn(tmp, a))
                post.append(BijOut(tmp, a))
                args.append(Var(tmp))
            else:
                args.append(a)
        env = dict(zip(params, args))
        tag = f"__{s.f}{self.n}"
        inl = _Subst(env, tag, set(params))
        return ((ArgCheck(tuple(_unwrap(a) for a in s.args)),) + tuple(pre)
                + self.run(inl.stmts(body), stack + (s.f,)) + tuple(post))


class _Subst:
    """Parameters -> argument views, callee locals -> fresh names."""

    def __init__(self, env, tag, params):
        self.env, self.tag, self.params = env, tag, params

    def local(self, n):
        if n in self.params:
            raise UnsupportedProgram(f"codegen: parameter {n!r} is (de)allocated or a loop variable")
        return n + self.tag

    def view(self, v):
        if isinstance(v, BView):
            return BView(self.view(v.base), v.bij, v.args)
        if isinstance(v, Var):
            return self.env.get(v.name, Var(v.name + self.tag))
        if isinstance(v, IView):
            base = self.env.get(v.name, Var(v.name + self.tag))
            if not isinstance(base, Var):
                raise KindError("indexing into a scalar cell")
            return IView(base.name, tuple(self.e(x) for x in v.idx))
        if isinstance(v, FView):
            base = self.env.get(v.name, Var(v.name + self.tag))
            if not isinstance(base, Var):
                raise KindError("a field of a non-Complex cell")
            return FView(base.name, v.field)
        return v

    def e(self, x):
        if isinstance(x, (Var, IView, FView)):
            return self.view(x)
        if isinstance(x, Un):
            return Un(x.op, self.e(x.e))
        if isinstance(x, Bin):
            return Bin(x.op, self.e(x.l), self.e(x.r))
        if isinstance(x, Call):
            return Call(x.f, tuple(self.e(a) for a in x.args))
        return x

    def stmts(self, ss):
        return tuple(self.stmt(s) for s in ss)

    def stmt(self, s):
        if isinstance(s, Instr):
            return Instr(s.op, self.view(s.target), s.fname, tuple(self.e(a) for a in s.args))
        if isinstance(s, Alloc):
            return Alloc(self.local(s.name), self.e(s.e))
        if isinstance(s, Dealloc):
            return Dealloc(self.local(s.name), self.e(s.e))
        if isinstance(s, For):
            return For(self.local(s.var), self.e(s.a), self.e(s.s), self.e(s.b), self.stmts(s.body))
        if isinstance(s, While):
            return While(self.e(s.pre), self.e(s.post), self.stmts(s.body))
        if isinstance(s, If):
            return If(self.e(s.pre), s.post if s.post is SAME else self.e(s.post),
                      self.stmts(s.then), self.stmts(s.els))
        if isinstance(s, Safe):
            return Safe(s.kind, tuple(self.e(x) for x in s.exprs))
        if isinstance(s, NoCheck):
            return NoCheck(self.stmts(s.body))
        if isinstance(s, PCall):
            return PCall(s.f, tuple(self.view(a) for a in s.args), s.uncall)
        raise UnsupportedProgram(f"codegen: cannot inline {s!r}")


# ---------------------------------------------------------------------------
# CUDA emission
# ---------------------------------------------------------------------------

_CODES = {"POST": 1, "DIRTY": 2, "DOMAIN": 3, "ITER": 4, "REV": 5, "FUEL": 6, "OVERFLOW": 9}

_PRELUDE = r"""
#include <math.h>
#include <stdint.h>
#include <cuda_runtime.h>
#include "fexp.cuh"
#define RC_POST 1
#define RC_DIRTY 2
#define RC_DOMAIN 3
#define RC_ITER 4
#define RC_REV 5
#define RC_FUEL 6
#define RC_OVERFLOW 9
#define RC_VALUE 12
#define RC_DEPTH 13
// mulconst's Int write-back (numerics._div_const): exact division or KindError
__device__ __forceinline__ long long rl_idivc(long long v, long long c, int &code) {
  if (v % c != 0) { if (!code) code = 7; return 0; }
  return v / c;
}
// Fixed (Q31.32, values.py:28-86): raw int64 cells, + / - wrap mod 2^64;
// to_float = raw / 2^32 (correctly rounded); from_real = round(v * 2^32)
// half-even, wrapped; round(inf) is Python's OverflowError, round(nan) its
// ValueError
__device__ __forceinline__ long long rl_fx_add(long long a, long long b) {
  return (long long)((unsigned long long)a + (unsigned long long)b);
}
__device__ __forceinline__ long long rl_fx_sub(long long a, long long b) {
  return (long long)((unsigned long long)a - (unsigned long long)b);
}
__device__ __forceinline__ long long rl_fx_neg(long long a) {
  return (long long)(0ULL - (unsigned long long)a);
}
__device__ __forceinline__ double rl_fx_tof(long long raw) {
  return __ll2double_rn(raw) * 0x1p-32;
}
__device__ __forceinline__ long long rl_fx_from(double v, int &code) {
  const double p = v * 4294967296.0;
  if (isnan(p)) { if (!code) code = RC_VALUE; return 0; }
  if (isinf(p)) { if (!code) code = RC_OVERFLOW; return 0; }
  const double r = rint(p);                              // round half to even
  if (fabs(r) < 9223372036854775808.0) return (long long)r;
  double m = fmod(r, 18446744073709551616.0);            // exact: r is an integer
  if (m < 0.0) m += 18446744073709551616.0;
  return (long long)(unsigned long long)m;
}
// values.s_* with the reference's error classes (values.py:343-431)
__device__ __forceinline__ double g_div(double a, double b, int &c) {
  if (b == 0.0) { if (!c) c = RC_DOMAIN; return 0.0; }
  return a / b;
}
__device__ __forceinline__ double g_sqrt(double x, int &c) {
  if (x < 0.0) { if (!c) c = RC_DOMAIN; return 0.0; }
  return sqrt(x);
}
__device__ __forceinline__ double g_log(double x, int &c) {
  if (!(x > 0.0)) { if (!c) c = RC_DOMAIN; return 0.0; }
  return log(x);
}
// exp: the series kernels' table exp (csrc/fexp.cuh: 0.5 ulp + O(2^-60), equal
// to the host libm's in ~99.9% of calls) inside (-708, 708), libdevice outside
__device__ rl::Exp2Tab rl_exp2tab[1024] = RL_EXP2_TABLE_INIT_1024;
__shared__ __align__(16) rl::Exp2Tab rl_exp2tab_s[1024];   // filled at kernel entry
__constant__ rl::ExpConsts1024 rl_expk = RL_EXP_CONSTS_1024_INIT;
__device__ __forceinline__ double g_exp(double x, int &c) {
  const double r = fabs(x) < 708.0 ? rl::fexp1024(x, [](int q) {
    const rl::Exp2Tab e = rl_exp2tab_s[q];
    return make_double2(e.hi, e.lo); }, rl_expk) : exp(x);
  if (isinf(r) && isfinite(x)) { if (!c) c = RC_OVERFLOW; }
  return r;
}
// log of an Int: CPython's math.log(i) for 1 <= i < 4096 from the host table
// `logtab` (a kernel argument), libdevice beyond
__shared__ double rl_logtab_s[512];        // lt[0, 512) staged at kernel entry
__device__ __forceinline__ double g_logi(long long k, const double *lt, int &c) {
  if (k >= 1 && k < 512) return rl_logtab_s[k];
  if (k >= 1 && k < 4096) return lt[k];
  return g_log((double)k, c);
}
// CPython float ** float (s_pow, values.py:408-421): x ** 0 and 1 ** y are 1.0,
// 0 ** negative raises, a finite result that overflows raises OverflowError;
// otherwise the host's correctly rounded pow().  The exponents whose correctly
// rounded power is one IEEE operation take it (libdevice pow is not exact
// there: 3.0 ** 1.0 would come out 1 ulp low).
__device__ __forceinline__ double g_pow(double a, double b, int &c) {
  if (b == 0.0 || a == 1.0) return 1.0;
  if ((a == 0.0 && b < 0.0) || (a < 0.0 && b != floor(b))) { if (!c) c = RC_DOMAIN; return 0.0; }
  double r;
  if (b == 1.0) r = a;
  else if (b == 2.0) r = a * a;
  else if (b == -1.0) r = 1.0 / a;
  else if (b == 0.5) r = a == 0.0 ? 0.0 : sqrt(a);   // pow(-0, 0.5) = +0
  else r = pow(a, b);
  if (isinf(r) && isfinite(a) && isfinite(b)) { if (!c) c = RC_OVERFLOW; }
  return r;
}
// ---- Dual numbers (reference values.py:258-431): the Hessian build runs the
// same generated code with R = Dl.  Doubles promote to Dl(d, 0) (_as_dual);
// comparisons and (double) see the primal (Dual.__float__ / __lt__ ...).
struct Dl {
  double p, t;
  __device__ __forceinline__ Dl() : p(0.0), t(0.0) {}
  __device__ __forceinline__ Dl(double a, double b = 0.0) : p(a), t(b) {}
  __device__ __forceinline__ explicit operator double() const { return p; }
};
__device__ __forceinline__ Dl operator+(Dl a, Dl b) { return Dl(a.p + b.p, a.t + b.t); }
__device__ __forceinline__ Dl operator-(Dl a, Dl b) { return Dl(a.p - b.p, a.t - b.t); }
__device__ __forceinline__ Dl operator*(Dl a, Dl b) { return Dl(a.p * b.p, a.t * b.p + a.p * b.t); }
__device__ __forceinline__ Dl operator/(Dl a, Dl b) {
  const double q = a.p / b.p;
  return Dl(q, (a.t - q * b.t) / b.p);
}
__device__ __forceinline__ Dl operator-(Dl a) { return Dl(-a.p, -a.t); }
__device__ __forceinline__ Dl operator+(Dl a, double b) { return a + Dl(b); }
__device__ __forceinline__ Dl operator+(double a, Dl b) { return Dl(a) + b; }
__device__ __forceinline__ Dl operator-(Dl a, double b) { return a - Dl(b); }
__device__ __forceinline__ Dl operator-(double a, Dl b) { return Dl(a) - b; }
__device__ __forceinline__ Dl operator*(Dl a, double b) { return a * Dl(b); }
__device__ __forceinline__ Dl operator*(double a, Dl b) { return Dl(a) * b; }
__device__ __forceinline__ Dl operator/(Dl a, double b) { return a / Dl(b); }
__device__ __forceinline__ Dl operator/(double a, Dl b) { return Dl(a) / b; }
__device__ __forceinline__ double rl_p(double x) { return x; }
__device__ __forceinline__ double rl_p(Dl x) { return x.p; }
__device__ __forceinline__ double rl_t(double) { return 0.0; }
__device__ __forceinline__ double rl_t(Dl x) { return x.t; }
__device__ __forceinline__ Dl g_div(Dl a, Dl b, int &c) {
  if (b.p == 0.0) { if (!c) c = RC_DOMAIN; return Dl(0.0); }
  return a / b;
}
__device__ __forceinline__ Dl g_sqrt(Dl x, int &c) {
  if (x.p <= 0.0 && x.t != 0.0) { if (!c) c = RC_DOMAIN; return Dl(0.0); }
  const double r = g_sqrt(x.p, c);
  return Dl(r, x.t / (2.0 * r));
}
__device__ __forceinline__ Dl g_log(Dl x, int &c) { return Dl(g_log(x.p, c), x.t / x.p); }
__device__ __forceinline__ Dl g_exp(Dl x, int &c) {
  const double r = g_exp(x.p, c);
  return Dl(r, x.t * r);
}
// exp of a ULog cell, memoised on the argument's bits: a while loop reads
// convert(s) in its condition and again in its body (and gradient mode a
// third time for the adjoint) with s unchanged in between.  exp is a pure
// function of its argument (the error class included), so reusing the value
// changes nothing the reference would observe.
struct ExpMemo {
  double in, out;
  int code, valid;
};
__device__ __forceinline__ double g_expm(double x, int &c, ExpMemo &m) {
  if (m.valid && __double_as_longlong(x) == __double_as_longlong(m.in)) {
    if (m.code && !c) c = m.code;
    return m.out;
  }
  int cc = 0;
  const double r = g_exp(x, cc);
  m.in = x;
  m.out = r;
  m.code = cc;
  m.valid = 1;
  if (cc && !c) c = cc;
  return r;
}
__device__ __forceinline__ Dl g_expm(Dl x, int &c, ExpMemo &) { return g_exp(x, c); }
__device__ __forceinline__ Dl sin(Dl x) { return Dl(sin(x.p), x.t * cos(x.p)); }
// s_atan2 over Duals (values.py): (atan2(yp, xp), (xp yt - yp xt) / (yp^2 + xp^2))
__device__ __forceinline__ Dl atan2(Dl y, Dl x) {
  const double r2 = y.p * y.p + x.p * x.p;
  return Dl(atan2(y.p, x.p), (x.p * y.t - y.p * x.t) / r2);
}
__device__ __forceinline__ Dl cos(Dl x) { return Dl(cos(x.p), -x.t * sin(x.p)); }
__device__ __forceinline__ double g_abs(double x, int &) { return fabs(x); }
__device__ __forceinline__ Dl g_abs(Dl x, int &c) {
  if (x.p == 0.0 && x.t != 0.0) { if (!c) c = RC_DOMAIN; return Dl(0.0); }
  return Dl(fabs(x.p), x.p >= 0.0 ? x.t : -x.t);
}
__device__ __forceinline__ Dl g_pow(Dl a, Dl b, int &c) {
  const double r = g_pow(a.p, b.p, c);
  double t = 0.0;
  if (a.t != 0.0) t = t + b.p * g_pow(a.p, b.p - 1.0, c) * a.t;
  if (b.t != 0.0) t = t + r * g_log(a.p, c) * b.t;
  return Dl(r, t);
}
#define RC_KIND 7
#define RC_INDEX 8
#define RC_ALIAS 10
#define RC_ASSERT 11
// Array._offset (values.py:172-183): 1-based, row-major, IndexOutOfBounds
__device__ __forceinline__ long long rl_off1(long long i, long long n, int &c) {
  if (i < 1 || i > n) { if (!c) c = RC_INDEX; return 0; }
  return i - 1;
}
__device__ __forceinline__ long long rl_off2(long long i, long long n1, long long j, long long n2,
                                             int &c) {
  if (i < 1 || i > n1 || j < 1 || j > n2) { if (!c) c = RC_INDEX; return 0; }
  return (i - 1) * n2 + (j - 1);
}
__device__ __forceinline__ long long rl_offbad(int &c) {   // wrong number of indices
  if (!c) c = RC_INDEX;
  return 0;
}
__device__ __forceinline__ long long g_imod(long long a, long long b, int &c) {
  if (b == 0) { if (!c) c = RC_DOMAIN; return 0; }
  long long r = a % b;
  if (r != 0 && ((r < 0) != (b < 0))) r += b;     // Python's modulo
  return r;
}

// Chunk sort by a loop-driving key (generate: `sort key`): each block takes
// RLG_C elements, counting-sorts their indices by 256 linear buckets of the
// key over the chunk's range, and runs warp rounds of 32 key-neighbours, so
// a warp's lanes run their data-dependent loops for (nearly) the same trip
// count (the hand-written Bessel kernel's z-bucket rounds, besselj.cu).
#ifndef RLG_BLOCK
#define RLG_BLOCK 128
#endif
#ifndef RLG_M
#define RLG_M 16
#endif
#ifndef RLG_MINB
#define RLG_MINB 6           // (build() sets it: the tightest budget without spills)
#endif
#define RLG_C (RLG_BLOCK * RLG_M)
__device__ __forceinline__ void rlg_sort_chunk(const double *__restrict__ key, int cnt, int *hist,
                                               unsigned short *perm, double *red) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  double kv[RLG_M];
  double lo = INFINITY, hi = -INFINITY;
#pragma unroll
  for (int m = 0; m < RLG_M; ++m) {
    const int e = m * RLG_BLOCK + tid;
    kv[m] = e < cnt ? key[e] : NAN;
    if (isfinite(kv[m])) { lo = fmin(lo, kv[m]); hi = fmax(hi, kv[m]); }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (lane == 0) { red[w] = lo; red[RLG_BLOCK / 32 + w] = hi; }
  for (int b = tid; b < 256; b += RLG_BLOCK) hist[b] = 0;
  __syncthreads();
  lo = red[0];
  hi = red[RLG_BLOCK / 32];
  for (int q = 1; q < RLG_BLOCK / 32; ++q) { lo = fmin(lo, red[q]); hi = fmax(hi, red[RLG_BLOCK / 32 + q]); }
  const double sc = hi > lo ? 255.5 / (hi - lo) : 0.0;
  int bk[RLG_M], rk[RLG_M];
#pragma unroll
  for (int m = 0; m < RLG_M; ++m) {
    const int e = m * RLG_BLOCK + tid;
    if (e < cnt) {
      int b = isfinite(kv[m]) ? (int)((kv[m] - lo) * sc) : 255;
      bk[m] = b < 0 ? 0 : (b > 255 ? 255 : b);
      rk[m] = atomicAdd(&hist[bk[m]], 1);
    }
  }
  __syncthreads();
  if (w == 0) {                       // exclusive scan: lane l owns buckets 8l .. 8l+7
    int loc[8], t = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) { loc[q] = t; t += hist[8 * lane + q]; }
    int x = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    const int basep = x - t;
#pragma unroll
    for (int q = 0; q < 8; ++q) hist[8 * lane + q] = basep + loc[q];
  }
  __syncthreads();
#pragma unroll
  for (int m = 0; m < RLG_M; ++m) {
    const int e = m * RLG_BLOCK + tid;
    if (e < cnt) perm[hist[bk[m]] + rk[m]] = (unsigned short)e;
  }
  __syncthreads();
}
"""


def _c_double(v):
    if isinstance(v, bool):
        raise UnsupportedProgram("codegen: Bool values are not supported")
    if isinstance(v, int):
        return f"{float(v)!r}"
    if math.isnan(v) or math.isinf(v):
        raise UnsupportedProgram("codegen: non-finite literals are not supported")
    return float(v).hex()


@dataclass(frozen=True)
class _Ref:
    """A storage cell an instruction touches: C lvalues of its value and
    cotangent, its kind, the root name and (array cells) the offset temp."""
    v: str
    g: str
    kind: str
    root: str
    off: object = None


class _Emitter:
    def __init__(self, params, kinds, body, fname, shapes=None):
        self.params = params
        self.kinds = dict(kinds)      # name -> "f" | "u" | "i"  ("a": Float array param)
        self.shapes = dict(shapes or {})
        self.body = body
        self.fname = fname
        self.lines = []
        self.depth = 1
        self.tmp = 0
        self.loop = 0

    # kinds ------------------------------------------------------------
    def kind(self, name):
        k = self.kinds.get(name)
        if k is None:
            raise UnsupportedProgram(f"codegen: {name!r} is used before it is allocated")
        if k in ("a", "ai"):
            raise KindError(f"{name!r} is an array; index it (instructions and expressions "
                            "take scalar cells)")
        if k == "c":
            raise KindError(f"{name!r} is Complex: use {name}.re / {name}.im, or abs / abs2 / "
                            "angle as an instruction argument")
        return k

    def cell_kind(self, v):
        """Kind of a view's cell: array cells are Float ("a") or Int ("ai")."""
        if isinstance(v, FView):
            if self.kinds.get(v.name) != "c":
                raise KindError(f"{v.name!r} has no field {v.field!r}")
            return "f"
        if isinstance(v, IView):
            if v.name not in self.shapes:
                raise KindError(f"{v.name!r} is not an array parameter")
            return "i" if self.kinds.get(v.name) == "ai" else "f"
        return self.kind(v.name)

    def offset(self, v, pre=None):
        """C expression of the row-major offset of view v (Array._offset,
        values.py:172-183); an out-of-range index sets RC_INDEX.  `pre`:
        index values already evaluated into temps."""
        shape = self.shapes.get(v.name)
        if shape is None:
            raise KindError(f"{v.name!r} is not an array parameter")
        idx = pre if pre is not None else [self.int_expr(e, "array index") for e in v.idx]
        if len(idx) != len(shape):
            return "rl_offbad(code)"
        if len(idx) == 1:
            return f"rl_off1({idx[0]}, {shape[0]}LL, code)"
        return f"rl_off2({idx[0]}, {shape[0]}LL, {idx[1]}, {shape[1]}LL, code)"

    def idx_temps(self, a):
        """Evaluate a view's index expressions into temps (storage ids of
        the alias checks, interpreter.py:600-622); None for a plain name."""
        if not isinstance(a, IView):
            return None
        out = []
        for e in a.idx:
            t = self.new("ix")
            self.w(f"const long long {t} = {self.int_expr(e, 'array index')};")
            out.append(t)
        return out

    def alias_pre(self, views, pres, label):
        """Strict pairwise alias checks on storage ids, before any read (prim
        statements and calls, interpreter.py:961-964, 999-1002)."""
        for i in range(len(views)):
            for j in range(i + 1, len(views)):
                a, b = views[i], views[j]
                if a.name != b.name:
                    continue
                if isinstance(a, FView) and isinstance(b, FView) and a.field != b.field:
                    continue                                   # .re and .im are disjoint
                if pres[i] is None or pres[j] is None:      # a whole cell / array
                    self.w("if (!code) code = RC_ALIAS;")
                elif len(pres[i]) == len(pres[j]):
                    same = " && ".join(f"{x} == {y}" for x, y in zip(pres[i], pres[j]))
                    self.w(f"if ({same} && !code) code = RC_ALIAS;")

    def view_ref(self, a, pre=None):
        """_Ref of an instruction operand; array offsets land in temps (the
        reference's readers evaluate indices in operand order)."""
        if isinstance(a, FView):
            self.cell_kind(a)
            c = _cid(a.name)
            return _Ref(f"v_{c}_{a.field}", f"g_{c}_{a.field}", "f", a.name, ("field", a.field))
        if isinstance(a, Var) and self.kinds.get(a.name) == "c":
            c = _cid(a.name)                          # the whole Complex value
            return _Ref(c, c, "c", a.name)
        if isinstance(a, IView):
            o = self.new("o")
            self.w(f"const long long {o} = {self.offset(a, pre)};")
            c = _cid(a.name)
            k = self.cell_kind(a)
            return _Ref(f"v_{c}[{o}]", f"g_{c}[{o}]" if k == "f" else None, k, a.name, o)
        k = self.kind(a.name)
        c = _cid(a.name)
        return _Ref(f"v_{c}", f"g_{c}", k, a.name)

    def alias(self, a, b, label):
        """_alias_checks (interpreter.py:624-657): same root and overlapping
        storage ids -> AliasedArguments, at run time like the reference."""
        if a is None or b is None or a.root != b.root:
            return
        if isinstance(a.off, tuple) or isinstance(b.off, tuple):      # Complex fields
            if isinstance(a.off, tuple) and isinstance(b.off, tuple) and a.off != b.off:
                return                                 # .re and .im are disjoint
            self.w("if (!code) code = RC_ALIAS;")
            return
        if a.off is None or b.off is None:
            self.w("if (!code) code = RC_ALIAS;")
        else:
            self.w(f"if ({a.off} == {b.off} && !code) code = RC_ALIAS;")

    def infer_alloc(self, name, e):
        k = "u" if isinstance(e, Call) and e.f == "ulog" else self.expr_kind(e)
        if k not in ("i", "f", "u", "x"):
            raise UnsupportedProgram(f"codegen: {name!r} is allocated with a {k!r} value")
        old = self.kinds.get(name)
        if old is not None and old != k:
            raise UnsupportedProgram(f"codegen: {name!r} is re-allocated with another kind")
        self.kinds[name] = k

    def expr_kind(self, e):
        if isinstance(e, Lit):
            if isinstance(e.v, bool):
                return "b"
            if isinstance(e.v, FixLit):
                return "x"
            return "i" if isinstance(e.v, int) else "f"
        if isinstance(e, Var):
            k = self.kind(e.name)
            return "f" if k == "u" else k
        if isinstance(e, (IView, FView)):
            return self.cell_kind(e)
        if isinstance(e, Un):
            return self.expr_kind(e.e)
        if isinstance(e, Call):
            if e.f == "ulog":
                return "u"
            if e.f in ("length", "size"):
                return "i"
            if e.f in ("min", "max"):
                ks = {self.expr_kind(a) for a in e.args}
                if "x" in ks:
                    raise UnsupportedProgram("codegen: min / max of Fixed values are not compiled")
                return "i" if ks == {"i"} else "f"
            return "f"
        if isinstance(e, Bin):
            if e.op in ("&&", "||", "==", "!=", "<", "<=", ">", ">="):
                return "b"
            lk, rk = self.expr_kind(e.l), self.expr_kind(e.r)
            if "x" in (lk, rk):
                raise UnsupportedProgram("codegen: Fixed arithmetic inside expressions is not "
                                         "compiled (Fixed cells take +=, -=, convert and "
                                         "comparisons)")
            if e.op == "%":
                if lk != "i" or rk != "i":
                    raise UnsupportedProgram("codegen: % needs Int operands")
                return "i"
            if e.op == "/":
                if lk == "i" and rk == "i":
                    raise UnsupportedProgram("codegen: Int / Int (exact-or-float) is not supported")
                return "f"
            if e.op == "^":
                if lk == "i" and rk == "i":
                    raise UnsupportedProgram("codegen: Int ^ Int is not supported")
                return "f"
            return "i" if lk == "i" and rk == "i" else "f"
        raise UnsupportedProgram(f"codegen: bad expression {e!r}")

    # code helpers -----------------------------------------------------
    def w(self, line):
        self.lines.append("  " * self.depth + line)

    def new(self, prefix="t"):
        self.tmp += 1
        return f"{prefix}{self.tmp}"

    def fail_check(self, label):
        """Errors do not jump: the first one is recorded in `code` (every
        later write is guarded), loops stop on it and the element's results
        are discarded — structured control flow keeps the warp reconverging
        after every data-dependent loop and branch."""

    # expressions (conditions, bounds, allocation values) ---------------
    def expr(self, e):
        """C expression for e; kind in {f, i, b}.  Errors land in `code`."""
        if isinstance(e, Lit):
            if isinstance(e.v, bool):
                return ("true" if e.v else "false"), "b"
            if isinstance(e.v, FixLit):
                return f"{e.v.raw}LL", "x"
            return (f"{e.v}LL" if isinstance(e.v, int) else _c_double(e.v)), self.expr_kind(e)
        if isinstance(e, Var):
            k = self.kind(e.name)
            if k == "u":
                return f"g_expm(v_{_cid(e.name)}, code, xm)", "f"  # to_real(ULog)
            return f"v_{_cid(e.name)}", k
        if isinstance(e, IView):
            return f"v_{_cid(e.name)}[{self.offset(e)}]", self.cell_kind(e)
        if isinstance(e, FView):
            self.cell_kind(e)
            return f"v_{_cid(e.name)}_{e.field}", "f"
        if isinstance(e, Un):
            s, k = self.expr(e.e)
            if k == "x":
                return f"rl_fx_neg({s})", "x"            # Fixed.__neg__: wrapped raw
            return f"(-{s})", k
        if isinstance(e, Call) and e.f in ("length", "size"):
            # numerics._expr_length / _expr_size: shapes are compile-time here
            a0 = e.args[0] if e.args else None
            if not isinstance(a0, Var) or a0.name not in self.shapes:
                raise KindError(f"{e.f}() needs an array")
            shape = self.shapes[a0.name]
            if e.f == "length":
                if len(e.args) != 1:
                    raise KindError("length() takes one array")
                return f"{math.prod(shape)}LL", "i"
            if len(e.args) != 2:
                raise KindError("size() takes an array and a dimension")
            d0 = e.args[1]
            if isinstance(d0, Lit) and isinstance(d0.v, int) and not isinstance(d0.v, bool):
                if 1 <= d0.v <= len(shape):
                    return f"{shape[d0.v - 1]}LL", "i"
                return "rl_offbad(code)", "i"
            d = self.int_expr(d0, "size dimension")
            tab = ", ".join(f"{n}LL" for n in shape)
            return (f"([&]() -> long long {{ const long long d_ = {d}; const long long s_[] = {{{tab}}};"
                    f" if (d_ < 1 || d_ > {len(shape)}) {{ if (!code) code = RC_INDEX; return 0; }}"
                    f" return s_[d_ - 1]; }}())"), "i"
        if isinstance(e, Call):
            args = [self.expr(a) for a in e.args]
            f = e.f
            if f == "ulog":
                (a, _), = args
                return f"g_log(R({a}), code)", "u"
            if f == "log" and args[0][1] == "i":
                return f"R(g_logi({args[0][0]}, logtab, code))", "f"
            if f in ("sqrt", "exp", "log"):
                (a, _), = args
                return f"g_{f}(R({a}), code)", "f"
            if f in ("sin", "cos"):
                (a, _), = args
                return f"{f}(R({a}))", "f"
            if f == "abs":
                (a, k), = args
                return (f"(({a}) < 0 ? -({a}) : ({a}))" if k == "i" else f"g_abs(R({a}), code)"), k
            if f == "abs2":
                (a, k), = args
                return f"(({a}) * ({a}))", k
            if f == "float":
                (a, ka), = args
                if ka == "x":
                    return "rl_fx_tof(" + a + ")", "f"   # float(Fixed): raw / 2^32
                return f"R((double)({a}))", "f"          # float(Dual) is its primal
            if f in ("min", "max"):
                (a, ka), (b, kb) = args
                if ka == "i" and kb == "i":
                    return f"({f}({a}, {b}))", "i"
                # Python min/max keep the chosen operand (primal comparison)
                cmp = "<" if f == "min" else ">"
                return f"((double)R({b}) {cmp} (double)R({a}) ? R({b}) : R({a}))", "f"
            raise UnsupportedProgram(f"codegen: expression function {f!r} is not supported")
        if isinstance(e, Bin):
            ls, lk = self.expr(e.l)
            rs, rk = self.expr(e.r)
            op = e.op
            if op in ("&&", "||"):
                return f"(({ls}) {op} ({rs}))", "b"
            if op in ("==", "!=", "<", "<=", ">", ">="):
                if "x" in (lk, rk):
                    # Fixed.__eq__ is False against any non-Fixed value; the
                    # orderings coerce the other side with from_real (values.py)
                    if lk == rk:
                        return f"(({ls}) {op} ({rs}))", "b"
                    if op in ("==", "!="):
                        return ("false" if op == "==" else "true"), "b"
                    if lk != "x":
                        ls = f"rl_fx_from((double)R({ls}), code)"
                    if rk != "x":
                        rs = f"rl_fx_from((double)R({rs}), code)"
                    return f"(({ls}) {op} ({rs}))", "b"
                if lk == "i" and rk == "i":
                    return f"(({ls}) {op} ({rs}))", "b"
                return f"((double)R({ls}) {op} (double)R({rs}))", "b"
            k = self.expr_kind(e)
            if op == "%":
                if isinstance(e.r, Lit) and type(e.r.v) is int and e.r.v > 0 and \
                        e.r.v & (e.r.v - 1) == 0:
                    # Python's x % 2^m (non-negative for a positive divisor)
                    # is the two's-complement low bits
                    return f"(({ls}) & {e.r.v - 1}LL)", "i"
                return f"g_imod({ls}, {rs}, code)", "i"
            if op == "/":
                return f"g_div(R({ls}), R({rs}), code)", "f"
            if op == "^":
                return f"g_pow(R({ls}), R({rs}), code)", "f"
            if k == "i":
                return f"(({ls}) {op} ({rs}))", "i"
            return f"(R({ls}) {op} R({rs}))", "f"
        raise UnsupportedProgram(f"codegen: bad expression {e!r}")

    def cond(self, e):
        s, k = self.expr(e)
        if k != "b":
            raise KindError("condition must be Bool")
        return s

    def int_expr(self, e, what):
        s, k = self.expr(e)
        if k != "i":
            raise KindError(f"{what} must be an Int")
        return s

    # instruction atoms ------------------------------------------------
    def atom_real(self, a, r):
        """The real value of an instruction argument (_arg_real)."""
        if isinstance(a, Lit):
            if isinstance(a.v, bool):
                raise UnsupportedProgram("codegen: Bool arguments are not supported")
            if isinstance(a.v, FixLit):
                return _c_double(a.v.real())
            return _c_double(a.v)
        if r.kind == "u":
            return f"g_expm({r.v}, code, xm)"
        if r.kind == "x":
            return f"rl_fx_tof({r.v})"                    # to_real(Fixed)
        if r.kind == "i":
            return f"R((double){r.v})"
        return r.v

    @staticmethod
    def tracked(r):
        return r is not None and r.kind in ("f", "u", "x")

    def gacc(self, r, delta, indent=""):
        """_g_accum (numerics.py:419-428): a Fixed cotangent takes
        Fixed.from_real(delta), anything else the plain sum."""
        if r.kind == "x":
            self.w(f"{indent}{r.g} = rl_fx_add({r.g}, rl_fx_from((double)({delta}), code));")
        else:
            self.w(f"{indent}{r.g} = {r.g} + {delta};")

    def apply_fn(self, fname, xs):
        if fname == "identity":
            return xs[0]
        if fname == "add":
            return f"(R({xs[0]}) + R({xs[1]}))"
        if fname == "sub":
            return f"(R({xs[0]}) - R({xs[1]}))"
        if fname == "mul":
            return f"(R({xs[0]}) * R({xs[1]}))"
        if fname == "div":
            return f"g_div(R({xs[0]}), R({xs[1]}), code)"
        if fname == "pow":
            return f"g_pow(R({xs[0]}), R({xs[1]}), code)"
        if fname == "neg":
            return f"(-R({xs[0]}))"
        if fname == "abs":
            return f"g_abs({xs[0]}, code)"
        if fname == "abs2":
            return f"(R({xs[0]}) * R({xs[0]}))"
        if fname in ("sqrt", "log", "exp"):
            return f"g_{fname}(R({xs[0]}), code)"
        if fname in ("sin", "cos"):
            return f"{fname}(R({xs[0]}))"
        raise UnsupportedProgram(f"codegen: instruction function {fname!r} is not supported")

    def partials(self, fname, xs):
        """INSTR_FNS partials (numerics.py:70-118); None = undefined there."""
        if fname == "identity":
            return ["1.0"]
        if fname == "add":
            return ["1.0", "1.0"]
        if fname == "sub":
            return ["1.0", "-1.0"]
        if fname == "mul":
            return [xs[1], xs[0]]
        if fname == "div":
            return [f"g_div(R(1.0), R({xs[1]}), code)",
                    f"(-g_div(R({xs[0]}), R({xs[1]}) * R({xs[1]}), code))"]
        if fname == "pow":
            first = f"({xs[1]} * g_pow(R({xs[0]}), R({xs[1]}) - 1.0, code))"
            second = (f"((double)R({xs[0]}) > 0.0 ? g_pow(R({xs[0]}), R({xs[1]}), code) * "
                      f"g_log(R({xs[0]}), code) : R(NAN))")
            return [first, ("POW2", second, xs[0])]
        if fname == "neg":
            return ["-1.0"]
        if fname == "abs":
            return [("ABS", f"((double)R({xs[0]}) > 0.0 ? 1.0 : -1.0)", xs[0])]
        if fname == "abs2":
            return [f"(2.0 * R({xs[0]}))"]
        if fname == "sqrt":
            return [f"g_div(R(0.5), g_sqrt(R({xs[0]}), code), code)"]
        if fname == "exp":
            return [f"g_expm(R({xs[0]}), code, xm)"]
        if fname == "log":
            return [f"g_div(R(1.0), R({xs[0]}), code)"]
        if fname == "sin":
            return [f"cos(R({xs[0]}))"]
        if fname == "cos":
            return [f"(-sin(R({xs[0]})))"]
        raise UnsupportedProgram(f"codegen: no gradient rule for {fname!r}")

    # statements -------------------------------------------------------
    def stmts(self, ss, grad, label):
        for s in ss:
            self.stmt(s, grad, label)

    def stmt(self, s, grad, label):
        if isinstance(s, Instr):
            self.instr(s, grad, label)
        elif isinstance(s, NoCheck):
            n = self.new("chk")
            self.w(f"{{ const int {n} = chk; chk = 0;")
            self.depth += 1
            self.stmts(s.body, grad, label)
            self.depth -= 1
            self.w(f"  chk = {n}; }}")
        elif isinstance(s, (BijIn, BijOut)):
            self.bijector(s)
        elif isinstance(s, DepthErr):
            self.w("if (!code) code = RC_DEPTH;")
        elif isinstance(s, ArgCheck):
            self.w("{")
            self.depth += 1
            pres = [self.idx_temps(a) for a in s.views]
            if any(p is not None for p in pres):
                self.fail_check(label)
            self.alias_pre(s.views, pres, label)
            for a, pre in zip(s.views, pres):              # the readers: bounds
                if pre is not None:
                    self.w(f"(void){self.offset(a, pre)};")
                elif a.name not in self.kinds:
                    raise UnsupportedProgram(f"codegen: {a.name!r} is used before it is allocated")
            if any(p is not None for p in pres):
                self.fail_check(label)
            self.depth -= 1
            self.w("}")
        elif isinstance(s, PCall):
            if s.f not in PRIM_ARITY:
                raise UnsupportedProgram(f"codegen: call of {s.f!r} was not inlined")
            self.w("{")
            self.depth += 1
            self.prim(s, grad, label)
            self.depth -= 1
            self.w("}")
        elif isinstance(s, Safe):
            if s.kind != "assert":
                raise UnsupportedProgram("codegen: @safe print has no device equivalent")
            for e in s.exprs:                 # interpreter.py:800-811
                c = self.cond(e)
                self.w(f"{{ const bool ok = {c};")
                self.w("  if (!ok && !code) code = RC_ASSERT; }")
        elif isinstance(s, Alloc):
            if s.name in self.shapes:
                raise UnsupportedProgram(f"codegen: {s.name!r} shadows a parameter")
            self.infer_alloc(s.name, s.e)
            k = self.kinds[s.name]
            val, vk = self.expr(s.e)
            if k == "i":
                self.w(f"v_{_cid(s.name)} = {val};")
            elif k == "x":
                self.w(f"v_{_cid(s.name)} = {val};")
                if grad:
                    self.w(f"g_{_cid(s.name)} = 0;")        # zero_like(Fixed) = Fixed(0)
            else:
                self.w(f"v_{_cid(s.name)} = {val};")
                if grad:
                    self.w(f"g_{_cid(s.name)} = 0.0;")      # wrap_gvar: zero_like
            self.fail_check(label)
        elif isinstance(s, Dealloc):
            k = self.kind(s.name)
            val, vk = self.expr(s.e)
            self.fail_check(label)
            if k == "i":
                self.w(f"if (chk && v_{_cid(s.name)} != ({val}) && !code) code = RC_DIRTY;")
            elif k == "x":
                # values_close: Fixed values match only as equal raw Fixed values
                if vk == "x":
                    self.w(f"if (chk && v_{_cid(s.name)} != ({val}) && !code) code = RC_DIRTY;")
                else:
                    self.w("if (chk && !code) code = RC_DIRTY;")
            else:
                # _ancilla_residual: |cur - decl| > tol fails (NaN passes); ULog by exponent
                d = self.new("d")
                self.w(f"{{ const double {d} = fabs(rl_p(v_{_cid(s.name)} - R({val})));")
                self.w(f"  if (chk && {d} > tol && !code) code = RC_DIRTY; }}")
        elif isinstance(s, If):
            took = self.new("took")
            pre = self.cond(s.pre)
            self.w(f"{{ const bool {took} = {pre};")
            self.fail_check(label)
            self.w(f"  if ({took}) {{")
            self.depth += 1
            self.stmts(s.then, grad, label)
            self.depth -= 1
            self.w("  } else {")
            self.depth += 1
            self.stmts(s.els, grad, label)
            self.depth -= 1
            self.w("  }")
            post = pre if s.post is SAME else self.cond(s.post)
            self.w(f"  if (chk) {{ const bool after = {post};")
            self.w(f"    if (after != {took} && !code) code = RC_POST; }}")
            self.w("}")
        elif isinstance(s, While):
            pre, post = self.cond(s.pre), self.cond(s.post)
            self.w("{")
            self.depth += 1
            self.w(f"if (chk) {{ const bool p0 = {post};")
            self.w("  if (p0 && !code) code = RC_POST; }")
            self.w("#pragma unroll 1")
            self.w("for (;;) {")
            self.depth += 1
            self.w(f"const bool go = ({pre}) && !code;")
            self.w("if (!go) break;")
            self.w("if (++ticks > fuel) { if (!code) code = RC_FUEL; break; }")
            self.stmts(s.body, grad, label)
            self.w(f"if (chk) {{ const bool p1 = {post};")
            self.w("  if (!p1 && !code) code = RC_POST; }")
            self.depth -= 1
            self.w("}")
            self.depth -= 1
            self.w("}")
        elif isinstance(s, For):
            self.loop += 1
            L = self.loop
            old = self.kinds.get(s.var)
            if old is not None and s.var in self.params:
                raise UnsupportedProgram(f"codegen: loop variable {s.var!r} shadows a parameter")
            a = self.int_expr(s.a, "loop start")
            st = self.int_expr(s.s, "loop step")
            b = self.int_expr(s.b, "loop stop")
            self.w(f"{{ const long long n1_{L} = {a}, n2_{L} = {st}, n3_{L} = {b};")
            self.fail_check(label)
            self.w(f"  if (n2_{L} == 0 && !code) code = RC_DOMAIN;")
            # program loops stay rolled: with array extents folded to constants
            # nvcc would unroll nested loops around inlined bodies (minutes of
            # compile time, hundreds of registers and spills)
            self.w("  #pragma unroll 1")
            self.w(f"  for (long long x_{L} = n1_{L}; !code && (n2_{L} > 0 ? x_{L} <= n3_{L} : "
                   f"x_{L} >= n3_{L}); x_{L} += n2_{L}) {{")
            self.depth += 1
            self.kinds[s.var] = "i"
            self.w("if (++ticks > fuel) { if (!code) code = RC_FUEL; break; }")
            self.w(f"v_{_cid(s.var)} = x_{L};")
            self.stmts(s.body, grad, label)
            self.w(f"if (chk && v_{_cid(s.var)} != x_{L} && !code) code = RC_ITER;")
            self.depth -= 1
            self.w("  }")
            self.w(f"  if (chk && (({a}) != n1_{L} || ({st}) != n2_{L} || ({b}) != n3_{L})) "
                   f"{{ if (!code) code = RC_ITER; }}")
            self.w("}")
        else:
            raise UnsupportedProgram(f"codegen: unsupported statement {s!r}")

    def bijector(self, s):
        """Copy-in / write-back of a bijector-view call argument (numerics.py:
        153-193 on Int cells: neg, addconst, mulconst with Int constants;
        a mulconst write-back that does not divide exactly is the
        reference's KindError)."""
        base = _unwrap(s.view)
        if not isinstance(base, Var) or self.kind(base.name) != "i":
            raise UnsupportedProgram("codegen: bijector views are compiled over Int scalar cells")
        chain = []
        v = s.view
        while isinstance(v, BView):
            if any(not isinstance(c, int) or isinstance(c, bool) for c in v.args):
                raise UnsupportedProgram("codegen: bijector constants on Int cells must be Int")
            chain.append((v.bij, v.args))
            v = v.base
        chain.reverse()                                  # base outward
        if isinstance(s, BijIn):
            self.kinds[s.tmp] = "i"
            val = f"v_{_cid(base.name)}"
            for bij, args in chain:
                val = {"neg": lambda: f"(-({val}))",
                       "addconst": lambda: f"(({val}) + {args[0]}LL)",
                       "mulconst": lambda: f"(({val}) * {args[0]}LL)"}[bij]()
            self.w(f"v_{_cid(s.tmp)} = {val};")
            return
        val = f"v_{_cid(s.tmp)}"
        for bij, args in reversed(chain):
            val = {"neg": lambda: f"(-({val}))",
                   "addconst": lambda: f"(({val}) - {args[0]}LL)",
                   "mulconst": lambda: f"rl_idivc({val}, {args[0]}LL, code)"}[bij]()
        self.w(f"v_{_cid(base.name)} = {val};")

    def prim(self, s, grad, label):
        """SWAP / ROT / IROT / NEG / INC / DEC (numerics.py:391-415 plain,
        :508-537 and :564-571 in gradient mode)."""
        kind = PRIM_INV[s.f] if s.uncall else s.f
        if len(s.args) != PRIM_ARITY[s.f]:
            raise KindError(f"{s.f} takes {PRIM_ARITY[s.f]} arguments")
        pres = [self.idx_temps(a) for a in s.args]
        if any(p is not None for p in pres):
            self.fail_check(label)
        self.alias_pre(s.args, pres, label)
        refs = [self.view_ref(a, pre) for a, pre in zip(s.args, pres)]
        if any(p is not None for p in pres):
            self.fail_check(label)
        if kind == "SWAP":
            a, b = refs
            if a.kind != b.kind:
                raise UnsupportedProgram("codegen: SWAP of cells of different kinds")
            ty = "long long" if a.kind == "i" else "R"
            t = self.new("sw")
            self.w(f"{{ const {ty} {t} = {a.v}; {a.v} = {b.v}; {b.v} = {t}; }}")
            if grad and a.kind != "i":                 # the GVar cells trade places
                self.w(f"{{ const R {t} = {a.g}; {a.g} = {b.g}; {b.g} = {t}; }}")
            return
        if kind == "NEG":
            (a,) = refs
            if a.kind == "u":
                raise UnsupportedProgram("codegen: NEG of a logarithmic number")
            self.w(f"{a.v} = -{a.v};")
            if grad and a.kind == "f":                 # _neg_adjoint
                self.w(f"{a.g} = -{a.g};")
            return
        if kind in ("INC", "DEC"):
            (a,) = refs
            if a.kind != "i":                          # _prim_plain: Int (or Fixed) only
                self.w("if (!code) code = RC_KIND;")
                return
            self.w(f"{a.v} = {a.v} {'+' if kind == 'INC' else '-'} 1;")
            return
        # ROT / IROT: (a c - b s, a s + b c), theta unchanged
        a, b, th = refs
        if a.kind != "f" or b.kind != "f" or th.kind not in ("f", "i"):
            raise UnsupportedProgram("codegen: ROT / IROT rotate Float cells by a Float or Int angle")
        thv = th.v if th.kind == "f" else f"R((double){th.v})"
        n = self.new("r")
        if not grad:
            self.w(f"{{ const R th{n} = {thv if kind == 'ROT' else '-' + thv};")
            self.w(f"  const R c{n} = cos(th{n}), s{n} = sin(th{n});")
            self.w(f"  const R a{n} = {a.v} * c{n} - {b.v} * s{n}, b{n} = {a.v} * s{n} + {b.v} * c{n};")
            self.w(f"  {a.v} = a{n}; {b.v} = b{n}; }}")
            return
        # _rot_adjoint: IROT is the reverse of a forward ROT by theta
        self.w(f"{{ const R ax{n} = {a.v}, bx{n} = {b.v}, ga{n} = {a.g}, gb{n} = {b.g};")
        if kind == "IROT":
            self.w(f"  const R d{n} = -bx{n} * ga{n} + ax{n} * gb{n};")
        else:
            self.w(f"  const R d{n} = bx{n} * ga{n} - ax{n} * gb{n};")
        if th.kind == "f":
            self.w(f"  {th.g} = {th.g} + d{n};")
        self.w(f"  const R th{n} = {('-' + thv) if kind == 'IROT' else thv};")
        self.w(f"  const R c{n} = cos(th{n}), s{n} = sin(th{n});")
        self.w(f"  {a.v} = ax{n} * c{n} - bx{n} * s{n}; {b.v} = ax{n} * s{n} + bx{n} * c{n};")
        self.w(f"  {a.g} = ga{n} * c{n} - gb{n} * s{n}; {b.g} = ga{n} * s{n} + gb{n} * c{n}; }}")

    def complex_instr(self, s, grad, tr, refs):
        """y += f(x) with x Complex, f in abs / abs2 / angle (numerics.py
        _COMPLEX_FNS: value and (d/dre, d/dim); _plus_minus_adjoint
        accumulates (sign gy) d/dre and (sign gy) d/dim)."""
        if s.op not in ("+=", "-=") or s.fname not in ("abs", "abs2", "angle") \
                or len(refs) != 1 or tr.kind != "f":
            raise UnsupportedProgram("codegen: a Complex operand takes +=/-= abs, abs2 or angle "
                                     "into a Float target")
        c = refs[0].v
        a, b = f"R(v_{c}_re)", f"R(v_{c}_im)"
        sq = f"({a} * {a} + {b} * {b})"
        val = {"abs": f"g_sqrt({sq}, code)", "abs2": sq, "angle": f"atan2({b}, {a})"}[s.fname]
        n = self.new("cx")
        self.w(f"{{ const R v{n} = {val};")
        self.w(f"  {tr.v} = {tr.v} {'+' if s.op == '+=' else '-'} v{n}; }}")
        if not grad:
            return
        sign = "1.0" if s.op == "-=" else "-1.0"
        if s.fname == "abs":
            dre, dim = f"g_div({a}, r{n}, code)", f"g_div({b}, r{n}, code)"
        elif s.fname == "abs2":
            dre, dim = f"(2.0 * {a})", f"(2.0 * {b})"
        else:
            dre, dim = f"g_div(-{b}, {sq}, code)", f"g_div({a}, {sq}, code)"
        self.w(f"{{ const R sg{n} = {sign} * {tr.g}; const R r{n} = {val};")
        self.w(f"  g_{c}_re = g_{c}_re + sg{n} * {dre};")
        self.w(f"  g_{c}_im = g_{c}_im + sg{n} * {dim}; }}")

    def instr(self, s, grad, label):
        self.w("{")
        self.depth += 1
        self.instr_body(s, grad, label)
        self.depth -= 1
        self.w("}")

    def instr_body(self, s, grad, label):
        args = s.args
        # readers first (target, then inputs: index errors), then the alias
        # checks (interpreter.py:887-948)
        tr = self.view_ref(s.target)
        refs = [None if isinstance(a, Lit) else self.view_ref(a) for a in args]
        if tr.off is not None or any(r is not None and r.off is not None for r in refs):
            self.fail_check(label)
        for r in refs:
            self.alias(tr, r, label)          # an instruction's target may not alias its inputs
        if grad:                              # shared reads under differentiation
            for i in range(len(refs)):
                for j in range(i + 1, len(refs)):
                    self.alias(refs[i], refs[j], label)
        tk = tr.kind
        TV, TG = tr.v, tr.g
        if any(r is not None and r.kind == "c" for r in refs):
            self.complex_instr(s, grad, tr, refs)
            return
        if s.op == "xor=":
            # numerics._xor_plain: Int targets with Int values (Bool is not
            # compiled); anything else is the reference's KindError, raised
            # when the statement runs.  Self-inverse, no adjoint on Ints.
            if tk != "i" or any(isinstance(a, Lit) and not isinstance(a.v, int) or
                                (r is not None and r.kind != "i") for a, r in zip(args, refs)) \
                    or s.fname not in ("identity", "add", "sub", "neg"):
                self.w("if (!code) code = RC_KIND;")
                return
            xs = [(f"{a.v}LL" if isinstance(a, Lit) else r.v) for a, r in zip(args, refs)]
            fv = {"identity": lambda: xs[0], "add": lambda: f"({xs[0]} + {xs[1]})",
                  "sub": lambda: f"({xs[0]} - {xs[1]})", "neg": lambda: f"(-{xs[0]})"}[s.fname]()
            self.w(f"{TV} = {TV} ^ ({fv});")
            return
        if s.op in ("+=", "-="):
            if tk == "u":
                raise KindError("+=/-= on a logarithmic number")
            if tk == "i":
                if s.fname not in ("identity", "add", "sub", "neg") or any(
                        isinstance(a, Lit) and isinstance(a.v, (float, FixLit)) or
                        (r is not None and r.kind != "i") for a, r in zip(args, refs)):
                    raise UnsupportedProgram("codegen: Int targets take Int +, - and identity")
                xs = [(f"{a.v}LL" if isinstance(a, Lit) else r.v) for a, r in zip(args, refs)]
                fv = {"identity": lambda: xs[0], "add": lambda: f"({xs[0]} + {xs[1]})",
                      "sub": lambda: f"({xs[0]} - {xs[1]})", "neg": lambda: f"(-{xs[0]})"}[s.fname]()
                self.w(f"{TV} = {TV} {'+' if s.op == '+=' else '-'} ({fv});")
                return
            fixed_lit = lambda a: isinstance(a, Lit) and isinstance(a.v, FixLit)  # noqa: E731
            if s.fname == "convert":
                (a,), xs = args, None
                fv = self.atom_real(a, refs[0])
            else:
                xs = [self.atom_real(a, r) for a, r in zip(args, refs)]
                if tk == "x" and s.fname in ("identity", "add", "sub") and all(
                        fixed_lit(a) or (r is not None and r.kind == "x")
                        for a, r in zip(args, refs)):
                    xr = [(f"{a.v.raw}LL" if isinstance(a, Lit) else r.v)
                          for a, r in zip(args, refs)]
                    fv = {"identity": lambda: xr[0], "add": lambda: f"rl_fx_add({xr[0]}, {xr[1]})",
                          "sub": lambda: f"rl_fx_sub({xr[0]}, {xr[1]})"}[s.fname]()
                    fv = ("RAW", fv)                   # Fixed values add raw
                else:
                    fv = self.apply_fn(s.fname, xs)   # a Fixed argument enters as its float
            if tk == "x":
                # numerics._plus_minus_plain, Fixed target: a Fixed value adds
                # raw, any other value enters as Fixed.from_real(float(fv));
                # both wrap mod 2^64
                inc = fv[1] if isinstance(fv, tuple) else f"rl_fx_from((double)({fv}), code)"
                iv = self.new("fi")
                self.w(f"{{ const long long {iv} = {inc};")
                self.w(f"  {TV} = {'rl_fx_add' if s.op == '+=' else 'rl_fx_sub'}({TV}, {iv}); }}")
            else:
                fvv = self.new("fv")
                self.w(f"{{ const R {fvv} = {fv};")
                self.w(f"  {TV} = {TV} {'+' if s.op == '+=' else '-'} {fvv}; }}")
            if not grad:
                return
            sign = "1.0" if s.op == "-=" else "-1.0"
            sg = self.new("sg")
            gy = f"rl_fx_tof({TG})" if tk == "x" else TG          # _gy_real
            self.w(f"{{ const R {sg} = {sign} * {gy};")
            if s.fname == "convert":
                r = refs[0]
                if self.tracked(r):
                    if r.kind == "u":
                        # d value / d exponent = value
                        self.gacc(r, f"{sg} * g_expm({r.v}, code, xm)", "  ")
                    else:
                        self.gacc(r, sg, "  ")
            else:
                parts = self.partials(s.fname, xs)
                for r, p in zip(refs, parts):
                    if not self.tracked(r):
                        continue
                    if isinstance(p, tuple):
                        tag, pv, x0 = p
                        cond = (f"(double)R({x0}) == 0.0" if tag == "ABS"
                                else f"!((double)R({x0}) > 0.0)")
                        self.w(f"  if (({cond}) && !code) code = RC_DOMAIN;")
                        p = pv
                    self.gacc(r, f"{sg} * {p}", "  ")
            self.w("}")
            return
        # *= and /= : the target is a logarithmic number
        if tk != "u":
            raise KindError(f"{s.op} target must be a logarithmic number")
        if s.fname in ("identity", "convert"):
            (a,) = args
            r = refs[0]
            if r is not None and r.kind == "u":
                contrib = r.v
            elif r is not None and r.kind == "i":
                contrib = f"R(g_logi({r.v}, logtab, code))"
            else:
                contrib = f"g_log({self.atom_real(a, r)}, code)"
        else:
            if len(args) != 1 and grad:
                raise UnsupportedProgram("codegen: *= / /= take one argument under differentiation")
            contrib = f"g_log({self.apply_fn(s.fname, [self.atom_real(a, r) for a, r in zip(args, refs)])}, code)"
        cv = self.new("c")
        self.w(f"{{ const R {cv} = {contrib};")
        self.w(f"  {TV} = {TV} {'+' if s.op == '*=' else '-'} {cv}; }}")
        if not grad:
            return
        (a,) = args
        r = refs[0]
        if self.tracked(r):
            sign = "1.0" if s.op == "/=" else "-1.0"
            if r.kind == "u":
                self.w(f"{r.g} = {r.g} + {sign} * {TG};")
            else:
                # exponent contribution log(value(a)): a.g += sign * gy / a
                self.gacc(r, f"g_div({sign} * {TG}, {self.atom_real(a, r)}, code)")
                self.fail_check(label)


def _cid(name):
    return name.replace("!", "_x").replace("~", "_t")


def _collect_vars(stmts, acc):
    for s in stmts:
        if isinstance(s, (Alloc, Dealloc)):
            acc.add(s.name)
        elif isinstance(s, BijIn):
            acc.add(s.tmp)
        elif isinstance(s, For):
            acc.add(s.var)
            _collect_vars(s.body, acc)
        elif isinstance(s, While):
            _collect_vars(s.body, acc)
        elif isinstance(s, If):
            _collect_vars(s.then, acc)
            _collect_vars(s.els, acc)
        elif isinstance(s, NoCheck):
            _collect_vars(s.body, acc)
    return acc


def _leaf_paths(shape):
    """autodiff.leaf_paths (autodiff.py:41-63) of a Float array of `shape`."""
    if len(shape) == 1:
        return [(("idx", (i,)),) for i in range(1, shape[0] + 1)]
    return [(("idx", (i, j)),) for i in range(1, shape[0] + 1) for j in range(1, shape[1] + 1)]


def _check_shapes(arrays, declared, params):
    shapes = {}
    for p, shp in dict(arrays or {}).items():
        if p not in params:
            raise KindError(f"array_shapes names unknown parameter {p!r}")
        shp = tuple(int(v) for v in (shp if isinstance(shp, (tuple, list)) else (shp,)))
        if len(shp) not in (1, 2) or min(shp) < 1:
            raise KindError(f"{p}: arrays are 1-d or 2-d with positive extents, got {shp}")
        shapes[p] = shp
    for p in declared:
        if p not in shapes:
            raise KindError(f"{p!r} is declared ::array; give its shape in array_shapes")
    return shapes


_LAUNCH = r"""
extern "C" int rlg_launch(long long n, const double *fin, const long long *iin, const double *seeds,
                          double tol, int chk, long long fuel, double *fout, double *gout,
                          unsigned char *fail, int dir, double *hout, long long *iout,
                          const double *logtab, void *stream) {
  if (n <= 0) return 0;
  const int block = RLG_BLOCK;
  long long grid = (n + block - 1) / block;
  if (grid > 148 * 16) grid = 148 * 16;
  rlg_kernel<<<(unsigned)grid, block, 0, (cudaStream_t)stream>>>(n, fin, iin, seeds, tol, chk, fuel,
                                                                fout, gout, fail, dir, hout, iout,
                                                                logtab);
  return (int)cudaGetLastError();
}
"""


def _rw(stmts, reads, writes):
    """Names read and written by inlined statements; False if a statement
    kind is not analysed (the caller then keeps every sweep)."""
    for s in stmts:
        if isinstance(s, Instr):
            writes.add(s.target.name)
            _expr_names(s.target, reads)
            for a in s.args:
                _expr_names(a, reads)
        elif isinstance(s, (Alloc, Dealloc)):
            writes.add(s.name)
            _expr_names(s.e, reads)
        elif isinstance(s, For):
            writes.add(s.var)
            for e in (s.a, s.s, s.b):
                _expr_names(e, reads)
            if not _rw(s.body, reads, writes):
                return False
        elif isinstance(s, (While, If)):
            for e in (s.pre, s.post):
                if e is not SAME:
                    _expr_names(e, reads)
            bodies = (s.body,) if isinstance(s, While) else (s.then, s.els)
            if not all(_rw(b, reads, writes) for b in bodies):
                return False
        elif isinstance(s, NoCheck):
            if not _rw(s.body, reads, writes):
                return False
        elif isinstance(s, PCall) and s.f in PRIM_ARITY:
            for v in s.args:
                writes.add(v.name)
                _expr_names(v, reads)
        elif isinstance(s, (ArgCheck, Safe)):
            for v in getattr(s, "views", ()) + getattr(s, "exprs", ()):
                _expr_names(v, reads)
        else:
            return False
    return True


def _flat(stmts, out):
    for st in stmts:
        out.append(st)
        for b in ((st.body,) if isinstance(st, (For, While, NoCheck)) else
                  (st.then, st.els) if isinstance(st, If) else ()):
            _flat(b, out)
    return out


def _loop_key(stmts, params, kinds):
    """The one Float scalar parameter that data-dependent while loops depend
    on (backward slice of their conditions through the statements that
    write the variables involved), or None: the sort key of the chunk sort."""
    flat = _flat(stmts, [])
    need = set()
    for st in flat:
        if isinstance(st, While):
            for e in (st.pre, st.post):
                if e is not SAME:
                    _expr_names(e, need)
    if not need:
        return None
    changed = True
    while changed:
        changed = False
        for st in flat:
            src = set()
            if isinstance(st, Instr) and st.target.name in need:
                for a in st.args:
                    _expr_names(a, src)
                _expr_names(st.target, src)
            elif isinstance(st, (Alloc, Dealloc)) and st.name in need:
                _expr_names(st.e, src)
            elif isinstance(st, For) and st.var in need:
                for e in (st.a, st.s, st.b):
                    _expr_names(e, src)
            elif isinstance(st, PCall) and st.f in PRIM_ARITY and \
                    any(v.name in need for v in st.args):
                for v in st.args:
                    _expr_names(v, src)
            if not src <= need:
                need |= src
                changed = True
    keys = [p for p in params if p in need and kinds.get(p) == "f"]
    return keys[0] if len(keys) == 1 else None


def _elision_split(body, inliner, fname, params):
    """Dead-sweep elision, the generated-kernel form of what
    the hand-written kernels do: a body `@routine R; M; ~@routine` whose R
    writes only its own ancillas (no parameter cells) and whose M writes
    nothing R reads or writes.  Then sweep 2 (f's ~R) and sweep 3 (~f's R)
    re-execute bit-identical primal arithmetic from the same state — R's
    ancillas are allocated afresh, the parameters it reads unchanged — so the
    gradient sweep starts from the forward's post-R state, and sweep 2's
    checks are exactly sweep 4's (the same operations in the same order).
    Returns (R, M, ~M ~R) as inlined statement tuples, or None."""
    if len(body) < 2 or not isinstance(body[0], RBegin) or not isinstance(body[-1], REnd):
        return None
    depth = 0
    for pos, st in enumerate(body):                 # the first open closes at the end
        depth += isinstance(st, RBegin) - isinstance(st, REnd)
        if depth == 0 and pos < len(body) - 1:
            return None
    try:
        R = inliner.run(_expand(body[0].body), (fname,))
        M = inliner.run(_expand(body[1:-1]), (fname,))
        # ~M then ~R, inverted at the source level (calls become uncalls) and
        # inlined afresh: callee ancillas live only inside their call
        G = inliner.run(_expand(_invert_list(body[1:-1])) + _invert_list(_expand(body[0].body)),
                        (fname,))
    except UnsupportedProgram:
        return None
    r_reads, r_writes, m_reads, m_writes = set(), set(), set(), set()
    if not (_rw(R, r_reads, r_writes) and _rw(M, m_reads, m_writes)):
        return None
    if r_writes & set(params):
        return None
    if m_writes & (r_reads | r_writes):
        return None
    return R, M, G


def generate(src, fname, int_params=(), mode="grad", array_shapes=None, complex_params=(),
             fixed_params=()):
    """CUDA source of the batched gradient (mode "grad"), forward-over-reverse
    Hessian-column (mode "hess": the same code over Dual numbers, tangent on
    the Float leaf `dir`) or plain run / uncall (modes "run" / "uncall": one
    sweep of f or ~f, reference interpreter.py:1021-1028) kernel of `fname`,
    and its layout: (source, float parameters, Int parameters, leaves) where
    leaves lists (parameter, leaf path) in the kernel's column order
    (scalars: path ()).  Every mode writes the primal Float leaves to fout and
    the Int leaves (scalars, then array cells) to iout after its first sweep."""
    if mode not in ("grad", "hess", "run", "uncall"):
        raise KindError(f"codegen mode {mode!r}")
    parser = _Parser(src)
    fns = parser.program()
    if fname not in fns:
        raise UnsupportedProgram(f"codegen: no function named {fname!r}")
    params, body = fns[fname]
    int_params = set(int_params)
    shapes = _check_shapes(array_shapes, parser.arrays.get(fname, ()), params)
    complex_params = set(complex_params)
    fixed_params = set(fixed_params)
    if fixed_params and mode == "hess":
        raise UnsupportedProgram("codegen: Hessians of Fixed parameters are not compiled")
    kinds = {p: ("ai" if p in shapes and p in int_params else "a" if p in shapes
                 else "i" if p in int_params else "c" if p in complex_params
                 else "x" if p in fixed_params else "f")
             for p in params}
    inliner = _Inliner(fns)
    fwd = inliner.run(_expand(body), (fname,))
    inv = inliner.run(_expand(_invert_list(body)), (fname,))
    floats = [p for p in params if kinds[p] in ("f", "a", "c", "x")]   # leaf columns
    ints = [p for p in params if kinds[p] in ("i", "ai")]
    leaves, base = [], {}
    for p in floats:
        base[p] = len(leaves)
        paths = (_leaf_paths(shapes[p]) if p in shapes else
                 [(("field", "re"),), (("field", "im"),)] if kinds[p] == "c" else [()])
        leaves += [(p, path) for path in paths]
    plain = mode in ("run", "uncall")
    split = None if plain or os.environ.get("REVGPU_CODEGEN_NO_ELIDE") else \
        _elision_split(body, inliner, fname, params)
    locals_ = sorted(_collect_vars(fwd, set()) | _collect_vars(inv, set())
                     | (set().union(*(_collect_vars(x, set()) for x in split)) if split else set()))
    em_f = _Emitter(params, kinds, inv if mode == "uncall" else fwd, fname, shapes)
    em_f.depth = 2
    if split is None:
        em_f.stmts(inv if mode == "uncall" else fwd, False, "fwd_done")
    else:
        # sweep 1 up to the end of R (ticks then = the ticks ~f's R would
        # spend), then M; f's ~R and ~f's R are elided
        R_, M_, _ = split
        em_f.stmts(R_, False, "fwd_done")
        em_f.w("const long long ticks_r = ticks;")
        em_f.stmts(M_, False, "fwd_done")
    em_g = _Emitter(params, dict(em_f.kinds), inv, fname, shapes)
    em_g.depth = 2
    if not plain:
        if split is None:
            em_g.stmts(inv, True, "grad_done")
        else:
            em_g.stmts(split[2], True, "grad_done")
    allk = dict(em_f.kinds)
    allk.update(em_g.kinds)
    decl = []
    for v in locals_:
        if v in params:
            raise UnsupportedProgram(f"codegen: {v!r} shadows a parameter")
        k = allk.get(v, "f")
        decl.append(f"    long long v_{_cid(v)} = 0;" if k == "i"
                    else f"    long long v_{_cid(v)} = 0, g_{_cid(v)} = 0;" if k == "x"
                    else f"    R v_{_cid(v)} = R(0.0), g_{_cid(v)} = R(0.0);")
    NL = len(leaves)
    hess = mode == "hess"
    tune = [f"#define {m} {os.environ[e]}" for m, e in (
        ("RLG_BLOCK", "REVGPU_CODEGEN_BLOCK"), ("RLG_M", "REVGPU_CODEGEN_M"),
        ("RLG_MINB", "REVGPU_CODEGEN_MINB")) if os.environ.get(e)]   # tuning sweeps only
    L = tune + [_PRELUDE, "typedef Dl R;" if hess else "typedef double R;",
         f"extern \"C\" __global__ void __launch_bounds__(RLG_BLOCK, RLG_MINB) rlg_kernel(long long n, const double *__restrict__ fin,"
         " const long long *__restrict__ iin, const double *__restrict__ seeds,"
         " double tol, int chk, long long fuel, double *__restrict__ fout,"
         " double *__restrict__ gout, unsigned char *__restrict__ fail, int dir,"
         " double *__restrict__ hout, long long *__restrict__ iout,"
         " const double *__restrict__ logtab) {",
         # the element loop is uniform over the warp and reconverges at every
         # element: lanes whose loops end early wait for the rest of the warp
         # instead of drifting onto their next element (a diverged warp ran
         # ~3 of 32 lanes per instruction)
         "  for (int q = threadIdx.x; q < 1024; q += blockDim.x) rl_exp2tab_s[q] = rl_exp2tab[q];",
         "  for (int q = threadIdx.x; q < 512; q += blockDim.x) rl_logtab_s[q] = logtab[q];",
         "  __syncthreads();"]
    key = None if os.environ.get("REVGPU_CODEGEN_NO_SORT") else _loop_key(fwd, params, kinds)
    if key is None:
        L += ["  for (long long base = (long long)blockIdx.x * blockDim.x; base < n;"
              " base += (long long)gridDim.x * blockDim.x) {",
              "    __syncwarp();",
              "    const long long i = base + threadIdx.x;",
              "    if (i >= n) continue;"]
    else:                               # rounds of key-sorted elements (rlg_sort_chunk)
        L += [f"  // chunk sort key: {key} (drives the data-dependent loops)",
              "  __shared__ int rlg_hist[256];",
              "  __shared__ unsigned short rlg_perm[RLG_C];",
              "  __shared__ double rlg_red[2 * RLG_BLOCK / 32];",
              "  for (long long cbase = (long long)blockIdx.x * RLG_C; cbase < n;"
              " cbase += (long long)gridDim.x * RLG_C) {",
              "    const int cnt = n - cbase < RLG_C ? (int)(n - cbase) : RLG_C;",
              f"    rlg_sort_chunk(fin + {base[key]}LL * n + cbase, cnt, rlg_hist, rlg_perm, rlg_red);",
              "    for (int m = 0; m < RLG_M; ++m) {",
              "    __syncwarp();",
              "    const int pos = m * RLG_BLOCK + (int)threadIdx.x;",
              "    if (pos >= cnt) continue;",
              "    const long long i = cbase + rlg_perm[pos];"]
    L += ["    int code = 0;", "    long long ticks = 0;",
          "    ExpMemo xm = {0.0, 0.0, 0, 0};"]
    # columns: leaf b of every element at fin[b * n + i] (coalesced across the batch)
    for p in floats:
        b, c = base[p], _cid(p)
        if p in shapes:
            m = math.prod(shapes[p])
            L.append(f"    R v_{c}[{m}], g_{c}[{m}];")
            L.append(f"    for (int e = 0; e < {m}; ++e) {{")
            L.append(f"      v_{c}[e] = R(fin[({b}LL + e) * n + i]"
                     + (f", dir == {b} + e ? 1.0 : 0.0);" if hess else ");"))
            L.append(f"      g_{c}[e] = R(0.0); }}")
        elif kinds[p] == "x":                       # Fixed: the raw int64 in the column's bits
            L.append(f"    long long v_{c} = __double_as_longlong(fin[{b}LL * n + i]), g_{c} = 0;")
        elif kinds[p] == "c":                       # Complex: two Float cells, re then im
            for q, fld in enumerate(("re", "im")):
                L.append(f"    R v_{c}_{fld} = R(fin[{b + q}LL * n + i]"
                         + (f", dir == {b + q} ? 1.0 : 0.0)" if hess else ")")
                         + f", g_{c}_{fld} = R(0.0);")
        else:
            L.append(f"    R v_{c} = R(fin[{b}LL * n + i]"
                     + (f", dir == {b} ? 1.0 : 0.0)" if hess else ")") + f", g_{c} = R(0.0);")
    ibase, nib = {}, 0
    for p in ints:                      # Int values (uniform over the batch) from iin
        ibase[p] = nib
        if p in shapes:
            m = math.prod(shapes[p])
            L.append(f"    long long v_{_cid(p)}[{m}];")
            L.append(f"    for (int e = 0; e < {m}; ++e) v_{_cid(p)}[e] = iin[{nib} + e];")
            nib += m
        else:
            L.append(f"    long long v_{_cid(p)} = iin[{nib}];")
            nib += 1
    L += decl

    def each_leaf(fmt, fmt_x=None):
        """C lines applying fmt(col_expr, value_lvalue, grad_lvalue) to every
        leaf (fmt_x to the Fixed ones: raw int64 cells)."""
        out = []
        for p in floats:
            b, c = base[p], _cid(p)
            if kinds[p] == "x":
                out.append("    " + fmt_x(f"{b}LL", f"v_{c}", f"g_{c}"))
                continue
            if p in shapes:
                m = math.prod(shapes[p])
                out.append(f"    for (int e = 0; e < {m}; ++e) {{ "
                           + fmt(f"({b}LL + e)", f"v_{c}[e]", f"g_{c}[e]") + " }")
            elif kinds[p] == "c":
                for q, fld in enumerate(("re", "im")):
                    out.append("    " + fmt(f"{b + q}LL", f"v_{c}_{fld}", f"g_{c}_{fld}"))
            else:
                out.append("    " + fmt(f"{b}LL", f"v_{c}", f"g_{c}"))
        return out

    L.append("    // ---- " + ("uncall_function (~f)" if mode == "uncall" else
                                "run_function (plain forward)") + " ----")
    L += em_f.lines
    L.append("    if (code) {")
    L.append(f"      for (int e = 0; e < {NL}; ++e) {{ fout[e * n + i] = NAN;"
             + ("" if plain else " gout[e * n + i] = NAN;")
             + (" hout[e * n + i] = NAN;" if hess else "") + " }")
    L.append(f"      for (int e = 0; e < {nib}; ++e) iout[e * n + i] = 0;")
    L.append("      fail[i] = (unsigned char)code; continue; }")
    L += each_leaf(lambda col, v, g: f"fout[{col} * n + i] = rl_p({v});",
                   lambda col, v, g: f"fout[{col} * n + i] = __longlong_as_double({v});")
    for p in ints:
        if p in shapes:
            L.append(f"    for (int e = 0; e < {math.prod(shapes[p])}; ++e)"
                     f" iout[({ibase[p]}LL + e) * n + i] = v_{_cid(p)}[e];")
        else:
            L.append(f"    iout[{ibase[p]}LL * n + i] = v_{_cid(p)};")
    close = ["  }", "}"] if key is None else ["    }", "    __syncthreads();", "  }", "}"]
    if plain:
        L += ["    fail[i] = 0;"] + close
        L.append(_LAUNCH)
        return "\n".join(L), floats, ints, leaves
    L.append("    // ---- uncall_function in gradient mode (seeded) ----")
    L.append("    // coerce_to_kind: a seed enters as Dual(seed, 0)")
    L += each_leaf(lambda col, v, g: f"{g} = R(seeds[{col}]);",
                   lambda col, v, g: f"{g} = __double_as_longlong(seeds[{col}]);")
    L.append("    ticks = 0;" if split is None else
             "    ticks = ticks_r;      // ~f's elided R spends the forward R's ticks")
    L += em_g.lines
    L.append("    if (!code) {      // the backward pass must restore every argument")
    L += ["  " + x for x in each_leaf(
        lambda col, v, g: f"if (!(fabs(rl_p({v}) - fin[{col} * n + i]) <= tol)) code = RC_REV;",
        lambda col, v, g: f"if ({v} != __double_as_longlong(fin[{col} * n + i])) code = RC_REV;")]
    for p in ints:
        if p in shapes:
            L.append(f"      for (int e = 0; e < {math.prod(shapes[p])}; ++e)"
                     f" if (v_{_cid(p)}[e] != iin[{ibase[p]} + e]) code = RC_REV;")
        else:
            L.append(f"      if (v_{_cid(p)} != iin[{ibase[p]}]) code = RC_REV;")
    L.append("    }")
    L += each_leaf(lambda col, v, g: f"gout[{col} * n + i] = code ? NAN : rl_p({g});"
                   + (f" hout[{col} * n + i] = code ? NAN : rl_t({g});" if hess else ""),
                   lambda col, v, g: f"gout[{col} * n + i] = __longlong_as_double({g});")
    L.append("    if (code) {")
    L.append(f"      for (int e = 0; e < {NL}; ++e) fout[e * n + i] = NAN;")
    L.append("    }")
    L.append("    fail[i] = (unsigned char)code;")
    L += close
    L.append(_LAUNCH)
    return "\n".join(L), floats, ints, leaves


# ---------------------------------------------------------------------------
# build + run
# ---------------------------------------------------------------------------

_CSRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc")
_LOGTABS = {}


def _logtab(dev):
    """CPython's math.log(i), i < 4096 (index 0: -inf), on `dev`: the integer
    logs of generated kernels are the reference's bit for bit."""
    key = str(dev)
    if key not in _LOGTABS:
        v = [-math.inf] + [math.log(i) for i in range(1, 4096)]
        _LOGTABS[key] = torch.tensor(v, dtype=torch.float64, device=dev)
    return _LOGTABS[key]


def _include_tag():
    """Hash of the csrc headers generated kernels include (part of the
    cached library's key)."""
    h = hashlib.sha256()
    for f in ("fexp.cuh", "exp2tab_1024.inc", "exp2tab_256.inc"):
        with open(os.path.join(_CSRC, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def _cache_dir():
    # in-tree by default (next to librevgpu.so), so generated kernels load from
    # the repository like the hand-written ones; $REVGPU_CODEGEN_CACHE overrides
    d = os.environ.get("REVGPU_CODEGEN_CACHE") or os.path.join(
        os.path.dirname(os.path.abspath(__file__)), "_codegen_cache")
    os.makedirs(d, exist_ok=True)
    return d


def _nvcc():
    import shutil
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        path = c if c and os.path.isabs(c) else (shutil.which(c) if c else None)
        if path and os.path.exists(path):
            return path
    raise NativeLibraryError("nvcc not found (codegen compiles generated kernels with it)")


def build(source):
    """Compile generated CUDA source to a cached shared library (sm_100a).
    The kernel's launch bounds take the tightest register budget that
    compiles with at most 256 bytes of spills (L1-resident): 8 blocks of 128
    threads per SM (64 registers; measured fastest on the Bessel batch),
    else 6, else the compiler's own."""
    h = hashlib.sha256((source + _include_tag() + "|minb-auto-v3").encode()).hexdigest()[:20]
    so = os.path.join(_cache_dir(), f"rlg_{h}.so")
    if not os.path.exists(so):
        with tempfile.TemporaryDirectory() as td:
            cu = os.path.join(td, "k.cu")
            tmp = os.path.join(td, "k.so")
            # a tuning define at the top (REVGPU_CODEGEN_MINB) fixes the budget
            explicit = any(ln.startswith("#define RLG_MINB") for ln in source.split("\n")[:4])
            for minb in ((None,) if explicit else (8, 6, 1)):
                with open(cu, "w") as fh:
                    fh.write(source if minb is None else f"#define RLG_MINB {minb}\n" + source)
                cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-fmad=false",
                       "-I", _CSRC, "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-o", tmp,
                       cu]
                r = subprocess.run(cmd, capture_output=True, text=True)
                if r.returncode != 0:
                    raise NativeLibraryError("codegen: nvcc failed:\n" + r.stderr[-4000:])
                spills = [int(x) for x in re.findall(r"(\d+) bytes spill stores", r.stderr)]
                if max(spills, default=0) <= 256:     # a few L1-resident slots are cheap
                    break
            os.replace(tmp, so)
    return so


class CompiledFunction:
    """A reversible function compiled to one batched CUDA kernel.

    `gradient(inputs, seeds)` is the batched `gradient(program,
    GradRequest(fname, args_i, seeds))`: a Float parameter takes a CUDA
    float64 tensor (one row per element) or a scalar, a Float array
    parameter (shape fixed at compile time through `array_shapes`) a tensor
    of shape (n, *shape) or one value of shape `shape` shared by every
    element, an Int parameter a Python int.  Seeds are the reference's
    (parameter, leaf path, cotangent) triples (autodiff.py:29-31; array
    cells: ((\"idx\", (i,)),) or ((\"idx\", (i, j)),), 1-based).  Returns
    (primal outputs, gradients, fail codes): dicts of tensors keyed by
    parameter name (arrays keep their shape; Int parameters carry no
    gradient)."""

    def __init__(self, source_text, fname, int_params=(), array_shapes=None, complex_params=(),
                 fixed_params=()):
        self.fname = fname
        self._text, self._ints, self._shapes = source_text, tuple(int_params), array_shapes
        self.complex = tuple(complex_params)
        self.fixed = tuple(fixed_params)
        self.source, self.floats, self.ints, self.leaves = generate(
            source_text, fname, int_params, array_shapes=array_shapes,
            complex_params=self.complex, fixed_params=self.fixed)
        self.params = _Parser(source_text).program()[fname][0]
        self.shapes = _check_shapes(array_shapes, (), self.params)
        self._lib = self._load(self.source)
        self._libs = {"grad": self._lib}

    @staticmethod
    def _load(source):
        lib = ctypes.CDLL(build(source))
        lib.rlg_launch.restype = ctypes.c_int
        lib.rlg_launch.argtypes = [ctypes.c_longlong] + [ctypes.c_void_p] * 3 + [
            ctypes.c_double, ctypes.c_int, ctypes.c_longlong] + [ctypes.c_void_p] * 3 + [
            ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        return lib

    def _lib_for(self, mode):
        if mode not in self._libs:
            self._libs[mode] = self._load(generate(self._text, self.fname, self._ints, mode=mode,
                                                   array_shapes=self._shapes,
                                                   complex_params=self.complex,
                                                   fixed_params=self.fixed)[0])
        return self._libs[mode]

    def run(self, inputs, direction=1, tol=1e-9, invcheck=True, max_steps=10**9):
        """Batched reference `run` (direction 1) / `uncall` (-1), interpreter.py:
        1021-1028: one sweep of f or ~f with every check.  Returns (outputs,
        fail codes), outputs keyed by parameter name (Int values as int64
        tensors of shape (n,) or (n, *shape))."""
        lib = self._lib_for("run" if direction > 0 else "uncall")
        primal, _, fail, _ = self._run(lib, inputs, [], tol, invcheck, max_steps)
        return primal, fail

    def _default_seeds(self):
        """autodiff.default_seeds (autodiff.py:99-110): the first parameter's
        single leaf."""
        first = self.params[0]
        paths = [path for p, path in self.leaves if p == first]
        if not paths:
            raise KindError(f"first argument {first!r} has no differentiable leaf; "
                            "pass explicit seeds")
        if len(paths) > 1 and first not in self.complex:     # a Complex seeds its real part
            raise KindError(f"first argument {first!r} is not scalar; pass explicit seeds")
        return [(first, paths[0], 1.0)]

    def hessian(self, inputs, tol=1e-9, invcheck=True, max_steps=10**9):
        """Batched reference `hessian(program, fname, args_i)` (autodiff.py:
        216-257) over the Float leaves (self.leaves order): the gradient
        sweeps over Dual numbers, one launch per tangent direction.  Returns
        (H, fail) with H of shape (n, NL, NL), H[:, k, j] = d(cotangent of
        leaf k) / d(leaf j)."""
        self._default_seeds()                 # the reference seeds by default
        hlib = self._lib_for("hess")
        cols = []
        fail = None
        for j in range(len(self.leaves)):
            _, _, f, h = self._run(hlib, inputs, None, tol, invcheck, max_steps, dir_=j)
            cols.append(h)
            fail = f if fail is None else torch.maximum(fail, f)
        H = torch.stack(cols, -1).permute(1, 0, 2).contiguous()   # (n, NL_k, NL_j)
        return H, fail

    def gradient(self, inputs, seeds=None, tol=1e-9, invcheck=True, max_steps=10**9):
        primal, grads, fail, _ = self._run(self._lib, inputs, seeds, tol, invcheck, max_steps)
        return primal, grads, fail

    def _columns(self, inputs, dev):
        """(NL, n) leaf columns of the Float inputs."""
        n = None
        for p in self.floats:
            v = inputs.get(p)
            shp = self.shapes.get(p, ())
            if p in self.fixed:                            # raw int64 tensor (n,) or one Fixed
                if isinstance(v, torch.Tensor) and v.dim() == 1:
                    if not v.is_cuda or v.dtype != torch.int64:
                        raise KindError(f"{p} must be a CUDA int64 tensor of Fixed raw values")
                    n = v.shape[0] if n is None else n
                    if v.shape[0] != n:
                        raise KindError("all batched inputs need the same length")
                continue
            if p in self.complex:
                if isinstance(v, torch.Tensor) and v.dim() == 1:
                    if not v.is_cuda or v.dtype != torch.complex128:
                        raise KindError(f"{p} must be a CUDA complex128 tensor")
                    n = v.shape[0] if n is None else n
                    if v.shape[0] != n:
                        raise KindError("all batched inputs need the same length")
                continue
            if isinstance(v, torch.Tensor) and v.dim() == len(shp) + 1:
                if not v.is_cuda or v.dtype != torch.float64 or tuple(v.shape[1:]) != shp:
                    raise KindError(f"{p} must be a CUDA float64 tensor of shape (n, *{shp})")
                n = v.shape[0] if n is None else n
                if v.shape[0] != n:
                    raise KindError("all batched inputs need the same length")
        if n is None:
            n = 1
        cols = []
        for p in self.floats:
            shp = self.shapes.get(p, ())
            m = math.prod(shp)
            v = inputs.get(p, 0.0)
            if p in self.fixed:                            # the raw value's bits
                if isinstance(v, torch.Tensor) and v.dim() == 1:
                    cols.append(v.view(torch.float64).reshape(1, n))
                else:
                    raw = v.raw if hasattr(v, "raw") else _fx_from_real(v)
                    cols.append(torch.tensor([raw], dtype=torch.int64, device=dev)
                                .view(torch.float64).reshape(1, 1).expand(1, n))
                continue
            if p in self.complex:                          # re and im columns
                if isinstance(v, torch.Tensor) and v.dim() == 1:
                    cols += [v.real.reshape(1, n), v.imag.reshape(1, n)]
                else:
                    z = complex(v.re, v.im) if hasattr(v, "re") else complex(v)
                    cols.append(torch.tensor([[z.real], [z.imag]], dtype=torch.float64,
                                             device=dev).expand(2, n))
                continue
            if isinstance(v, torch.Tensor) and v.dim() == len(shp) + 1:
                cols.append(v.reshape(n, m).t())
            else:
                t = torch.as_tensor(v, dtype=torch.float64).to(dev)
                if tuple(t.shape) != shp:
                    raise KindError(f"{p} must have shape {shp} (or (n, *{shp}))")
                cols.append(t.reshape(m, 1).expand(m, n))
        if not cols:
            return n, torch.zeros((0, n), dtype=torch.float64, device=dev)
        return n, torch.cat(cols).contiguous()

    def _run(self, lib, inputs, seeds, tol, invcheck, max_steps, dir_=-1):
        if not torch.cuda.is_available():
            raise UnsupportedProgram("codegen kernels need a CUDA device (no CPU path)")
        dev = torch.device("cuda", torch.cuda.current_device())
        n, fin = self._columns(inputs, dev)
        ivals = []
        for p in self.ints:
            v = inputs.get(p)
            if p in self.shapes:
                a = np.asarray(v)
                if a.shape != self.shapes[p] or a.dtype.kind not in "iu":
                    raise KindError(f"{p} must be an Int array of shape {self.shapes[p]}")
                ivals += [int(x) for x in a.ravel()]
                continue
            if not isinstance(v, int) or isinstance(v, bool):
                raise KindError(f"{p} must be an Int")
            ivals.append(v)
        iin = torch.tensor(ivals or [0], dtype=torch.int64, device=dev)
        col = {leaf: k for k, leaf in enumerate(self.leaves)}
        sv = [0] * max(1, len(self.leaves))           # bit patterns (Fixed leaves: raw)
        for pname, path, val in (self._default_seeds() if seeds is None else seeds):
            if path is None:
                path = ()
            if pname not in self.params:
                raise KindError(f"seed names unknown parameter {pname!r}")
            key = (pname, tuple((a, tuple(b) if isinstance(b, (tuple, list)) else b)
                                for a, b in path))
            if key not in col:
                raise KindError("seed target is not a differentiable leaf")
            # coerce_to_kind: a Fixed leaf's seed is Fixed.from_real(seed)
            sv[col[key]] = (_fx_from_real(val) if pname in self.fixed
                            else int(np.float64(float(val)).view(np.int64)))
        sv = torch.tensor(sv, dtype=torch.int64, device=dev).view(torch.float64)
        fout = torch.empty_like(fin)
        gout = torch.empty_like(fin)
        hout = torch.empty_like(fin) if dir_ >= 0 else None
        fail = torch.empty(n, dtype=torch.uint8, device=dev)
        iout = torch.empty((max(1, len(ivals)), n), dtype=torch.int64, device=dev)
        rc = lib.rlg_launch(n, fin.data_ptr(), iin.data_ptr(), sv.data_ptr(), float(tol),
                            int(bool(invcheck)), int(max_steps), fout.data_ptr(), gout.data_ptr(),
                            fail.data_ptr(), int(dir_),
                            hout.data_ptr() if hout is not None else None, iout.data_ptr(),
                            _logtab(dev).data_ptr(), torch.cuda.current_stream().cuda_stream)
        if rc:
            raise NativeLibraryError(f"codegen kernel launch failed (cudaError {rc})")
        primal, grads, b = {}, {}, 0
        for p in self.floats:
            if p in self.fixed:                            # raw int64 values / cotangents
                primal[p] = fout[b].contiguous().view(torch.int64)
                grads[p] = gout[b].contiguous().view(torch.int64)
                b += 1
                continue
            if p in self.complex:
                primal[p] = torch.complex(fout[b], fout[b + 1])
                grads[p] = torch.complex(gout[b], gout[b + 1])
                b += 2
                continue
            shp = self.shapes.get(p, ())
            m = math.prod(shp)
            primal[p] = fout[b:b + m].t().reshape((n,) + shp)
            grads[p] = gout[b:b + m].t().reshape((n,) + shp)
            b += m
        b = 0
        for p in self.ints:                  # the Int leaves after the first sweep
            shp = self.shapes.get(p, ())
            m = math.prod(shp)
            primal[p] = iout[b:b + m].t().reshape((n,) + shp)
            b += m
        return primal, grads, fail, hout


def compile_function(source_text, fname, int_params=(), array_shapes=None, complex_params=(),
                     fixed_params=()):
    """Compile function `fname` of reversible-DSL source to a batched CUDA
    gradient kernel (see CompiledFunction)."""
    return CompiledFunction(source_text, fname, int_params, array_shapes, complex_params,
                            fixed_params)
