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

The subset: scalar parameters (Float rows, or Int values uniform over the
batch), Float / ULog / Int ancillas, `+= -= *= /=` instructions with the
INSTR_FNS functions, `<-` / `->`, @routine / ~@routine, for / while / if.
Arrays, records, Fixed / Complex numbers, function calls and xor= are
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
import subprocess
import tempfile
from dataclasses import dataclass

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
            if word not in ("@routine", "~@routine"):
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
            toks.append(("name", src[i:j]))
            i = j
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
            if j < n and src[j].isalpha():
                raise UnsupportedProgram("codegen: Fixed / imaginary literals are not supported")
            body = src[i:j]
            toks.append(("num", float(body) if is_float else int(body)))
            i = j
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


@dataclass(frozen=True)
class Var:
    name: str


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
    target: str
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
        self.t = _tokenize(src)
        self.i = 0

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
            while not self.at("punct", ")"):
                params.append(self.name())
                if self.at("punct", "::"):
                    raise UnsupportedProgram("codegen: array / typed parameters are not supported")
                if self.at("punct", ","):
                    self.adv()
            self.adv()
            body = self.block(("end",))
            self.expect("name", "end")
            fns[fname] = (tuple(params), body)
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
            raise UnsupportedProgram("codegen: function (un)calls are not supported")
        target = self.name()
        if self.at("punct", "("):
            raise UnsupportedProgram("codegen: function calls / SWAP / ROT are not supported")
        if self.at("punct", "["):
            raise UnsupportedProgram("codegen: indexed views are not supported")
        if self.at("punct", "<-"):
            self.adv()
            return Alloc(target, self.expr())
        if self.at("punct", "->"):
            self.adv()
            return Dealloc(target, self.expr())
        if self.cur[0] == "punct" and self.cur[1] in ("+=", "-=", "*=", "/="):
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
        v = self.name()
        if self.at("punct", "[") or self.at("punct", "."):
            raise UnsupportedProgram("codegen: indexed views are not supported")
        return Var(v)

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
        if self.at("punct", "[") or self.at("punct", "."):
            raise UnsupportedProgram("codegen: indexed views are not supported")
        return Var(v)


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


_OP_INV = {"+=": "-=", "-=": "+=", "*=": "/=", "/=": "*="}


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
        elif isinstance(s, tuple):
            out.extend(_expand(s))
        else:
            out.append(s)
    if pending:
        raise UnsupportedProgram("codegen: routine block is never closed")
    return tuple(out)


# ---------------------------------------------------------------------------
# CUDA emission
# ---------------------------------------------------------------------------

_CODES = {"POST": 1, "DIRTY": 2, "DOMAIN": 3, "ITER": 4, "REV": 5, "FUEL": 6, "OVERFLOW": 9}

_PRELUDE = r"""
#include <math.h>
#include <stdint.h>
#include <cuda_runtime.h>
#define RC_POST 1
#define RC_DIRTY 2
#define RC_DOMAIN 3
#define RC_ITER 4
#define RC_REV 5
#define RC_FUEL 6
#define RC_OVERFLOW 9
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
__device__ __forceinline__ double g_exp(double x, int &c) {
  const double r = exp(x);
  if (isinf(r) && isfinite(x)) { if (!c) c = RC_OVERFLOW; }
  return r;
}
__device__ __forceinline__ double g_pow(double a, double b, int &c) {
  if ((a == 0.0 && b < 0.0) || (a < 0.0 && b != floor(b))) { if (!c) c = RC_DOMAIN; return 0.0; }
  return pow(a, b);
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
__device__ __forceinline__ Dl sin(Dl x) { return Dl(sin(x.p), x.t * cos(x.p)); }
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
__device__ __forceinline__ long long g_imod(long long a, long long b, int &c) {
  if (b == 0) { if (!c) c = RC_DOMAIN; return 0; }
  long long r = a % b;
  if (r != 0 && ((r < 0) != (b < 0))) r += b;     // Python's modulo
  return r;
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


class _Emitter:
    def __init__(self, params, kinds, body, fname):
        self.params = params
        self.kinds = dict(kinds)      # name -> "f" | "u" | "i"
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
        return k

    def infer_alloc(self, name, e):
        k = "u" if isinstance(e, Call) and e.f == "ulog" else self.expr_kind(e)
        k = {"i": "i", "f": "f", "u": "u"}[k]
        old = self.kinds.get(name)
        if old is not None and old != k:
            raise UnsupportedProgram(f"codegen: {name!r} is re-allocated with another kind")
        self.kinds[name] = k

    def expr_kind(self, e):
        if isinstance(e, Lit):
            if isinstance(e.v, bool):
                return "b"
            return "i" if isinstance(e.v, int) else "f"
        if isinstance(e, Var):
            k = self.kind(e.name)
            return "f" if k == "u" else k
        if isinstance(e, Un):
            return self.expr_kind(e.e)
        if isinstance(e, Call):
            if e.f == "ulog":
                return "u"
            if e.f in ("min", "max"):
                ks = {self.expr_kind(a) for a in e.args}
                return "i" if ks == {"i"} else "f"
            return "f"
        if isinstance(e, Bin):
            if e.op in ("&&", "||", "==", "!=", "<", "<=", ">", ">="):
                return "b"
            lk, rk = self.expr_kind(e.l), self.expr_kind(e.r)
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
        self.w(f"if (code) goto {label};")

    # expressions (conditions, bounds, allocation values) ---------------
    def expr(self, e):
        """C expression for e; kind in {f, i, b}.  Errors land in `code`."""
        if isinstance(e, Lit):
            if isinstance(e.v, bool):
                return ("true" if e.v else "false"), "b"
            return (f"{e.v}LL" if isinstance(e.v, int) else _c_double(e.v)), self.expr_kind(e)
        if isinstance(e, Var):
            k = self.kind(e.name)
            if k == "u":
                return f"g_exp(v_{_cid(e.name)}, code)", "f"       # to_real(ULog)
            return f"v_{_cid(e.name)}", k
        if isinstance(e, Un):
            s, k = self.expr(e.e)
            return f"(-{s})", k
        if isinstance(e, Call):
            args = [self.expr(a) for a in e.args]
            f = e.f
            if f == "ulog":
                (a, _), = args
                return f"g_log(R({a}), code)", "u"
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
                (a, _), = args
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
                if lk == "i" and rk == "i":
                    return f"(({ls}) {op} ({rs}))", "b"
                return f"((double)R({ls}) {op} (double)R({rs}))", "b"
            k = self.expr_kind(e)
            if op == "%":
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
    def atom_real(self, a):
        """The real value of an instruction argument (_arg_real)."""
        if isinstance(a, Lit):
            if isinstance(a.v, bool):
                raise UnsupportedProgram("codegen: Bool arguments are not supported")
            return _c_double(a.v)
        k = self.kind(a.name)
        if k == "u":
            return f"g_exp(v_{_cid(a.name)}, code)"
        if k == "i":
            return f"R((double)v_{_cid(a.name)})"
        return f"v_{_cid(a.name)}"

    def tracked(self, a):
        return isinstance(a, Var) and self.kind(a.name) in ("f", "u")

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
            return [f"g_exp(R({xs[0]}), code)"]
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
        elif isinstance(s, Alloc):
            self.infer_alloc(s.name, s.e)
            k = self.kinds[s.name]
            val, vk = self.expr(s.e)
            if k == "i":
                self.w(f"v_{_cid(s.name)} = {val};")
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
                self.w(f"if (chk && v_{_cid(s.name)} != ({val})) {{ code = RC_DIRTY; goto {label}; }}")
            else:
                # _ancilla_residual: |cur - decl| > tol fails (NaN passes); ULog by exponent
                d = self.new("d")
                self.w(f"{{ const double {d} = fabs(rl_p(v_{_cid(s.name)} - R({val})));")
                self.w(f"  if (chk && {d} > tol) {{ code = RC_DIRTY; goto {label}; }} }}")
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
            self.w(f"    if (code) goto {label};")
            self.w(f"    if (after != {took}) {{ code = RC_POST; goto {label}; }} }}")
            self.w("}")
        elif isinstance(s, While):
            pre, post = self.cond(s.pre), self.cond(s.post)
            self.w("{")
            self.depth += 1
            self.w(f"if (chk) {{ const bool p0 = {post}; if (code) goto {label};")
            self.w(f"  if (p0) {{ code = RC_POST; goto {label}; }} }}")
            self.w("for (;;) {")
            self.depth += 1
            self.w(f"const bool go = {pre};")
            self.fail_check(label)
            self.w("if (!go) break;")
            self.w(f"if (++ticks > fuel) {{ code = RC_FUEL; goto {label}; }}")
            self.stmts(s.body, grad, label)
            self.w(f"if (chk) {{ const bool p1 = {post}; if (code) goto {label};")
            self.w(f"  if (!p1) {{ code = RC_POST; goto {label}; }} }}")
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
            self.w(f"  if (n2_{L} == 0) {{ code = RC_DOMAIN; goto {label}; }}")
            self.w(f"  for (long long x_{L} = n1_{L}; n2_{L} > 0 ? x_{L} <= n3_{L} : x_{L} >= n3_{L};"
                   f" x_{L} += n2_{L}) {{")
            self.depth += 1
            self.kinds[s.var] = "i"
            self.w(f"if (++ticks > fuel) {{ code = RC_FUEL; goto {label}; }}")
            self.w(f"v_{_cid(s.var)} = x_{L};")
            self.stmts(s.body, grad, label)
            self.w(f"if (chk && v_{_cid(s.var)} != x_{L}) {{ code = RC_ITER; goto {label}; }}")
            self.depth -= 1
            self.w("  }")
            self.w(f"  if (chk && (({a}) != n1_{L} || ({st}) != n2_{L} || ({b}) != n3_{L})) "
                   f"{{ code = RC_ITER; goto {label}; }}")
            self.w("}")
        else:
            raise UnsupportedProgram(f"codegen: unsupported statement {s!r}")

    def instr(self, s, grad, label):
        t = s.target
        tk = self.kind(t)
        args = s.args
        for a in args:
            if isinstance(a, Var) and a.name == t:
                raise AliasedArguments("an instruction's target may not alias its inputs")
        if grad:
            names = [a.name for a in args if isinstance(a, Var)]
            if len(names) != len(set(names)):
                raise AliasedArguments("shared reads are rejected under differentiation "
                                       "(rewrite y += x * x as y += x ^ 2)")
        T = _cid(t)
        if s.op in ("+=", "-="):
            if tk == "u":
                raise KindError("+=/-= on a logarithmic number")
            if tk == "i":
                if s.fname not in ("identity", "add", "sub", "neg") or any(
                        isinstance(a, Lit) and isinstance(a.v, float) or
                        (isinstance(a, Var) and self.kind(a.name) != "i") for a in args):
                    raise UnsupportedProgram("codegen: Int targets take Int +, - and identity")
                xs = [(f"{a.v}LL" if isinstance(a, Lit) else f"v_{_cid(a.name)}") for a in args]
                fv = self.apply_fn(s.fname, xs)
                self.w(f"v_{T} = v_{T} {'+' if s.op == '+=' else '-'} ({fv});")
                return
            if s.fname == "convert":
                (a,), xs = args, None
                fv = self.atom_real(a)
            else:
                xs = [self.atom_real(a) for a in args]
                fv = self.apply_fn(s.fname, xs)
            fvv = self.new("fv")
            self.w(f"{{ const R {fvv} = {fv};")
            self.w(f"  if (code) goto {label};")
            self.w(f"  v_{T} = v_{T} {'+' if s.op == '+=' else '-'} {fvv}; }}")
            if not grad:
                return
            sign = "1.0" if s.op == "-=" else "-1.0"
            sg = self.new("sg")
            self.w(f"{{ const R {sg} = {sign} * g_{T};")
            if s.fname == "convert":
                (a,) = args
                if self.tracked(a):
                    if self.kind(a.name) == "u":
                        # d value / d exponent = value
                        self.w(f"  g_{_cid(a.name)} = g_{_cid(a.name)} + {sg} * g_exp(v_{_cid(a.name)}, code);")
                    else:
                        self.w(f"  g_{_cid(a.name)} = g_{_cid(a.name)} + {sg};")
            else:
                parts = self.partials(s.fname, xs)
                for a, p in zip(args, parts):
                    if not self.tracked(a):
                        continue
                    A = _cid(a.name)
                    if isinstance(p, tuple):
                        tag, pv, x0 = p
                        cond = (f"(double)R({x0}) == 0.0" if tag == "ABS"
                                else f"!((double)R({x0}) > 0.0)")
                        self.w(f"  if ({cond}) {{ if (!code) code = RC_DOMAIN; goto {label}; }}")
                        p = pv
                    self.w(f"  g_{A} = g_{A} + {sg} * {p};")
            self.w(f"  if (code) goto {label}; }}")
            return
        # *= and /= : the target is a logarithmic number
        if tk != "u":
            raise KindError(f"{s.op} target must be a logarithmic number")
        if s.fname in ("identity", "convert"):
            (a,) = args
            if isinstance(a, Var) and self.kind(a.name) == "u":
                contrib = f"v_{_cid(a.name)}"
            else:
                contrib = f"g_log({self.atom_real(a)}, code)"
        else:
            if len(args) != 1 and grad:
                raise UnsupportedProgram("codegen: *= / /= take one argument under differentiation")
            contrib = f"g_log({self.apply_fn(s.fname, [self.atom_real(a) for a in args])}, code)"
        cv = self.new("c")
        self.w(f"{{ const R {cv} = {contrib};")
        self.w(f"  if (code) goto {label};")
        self.w(f"  v_{T} = v_{T} {'+' if s.op == '*=' else '-'} {cv}; }}")
        if not grad:
            return
        (a,) = args
        if self.tracked(a):
            sign = "1.0" if s.op == "/=" else "-1.0"
            A = _cid(a.name)
            if self.kind(a.name) == "u":
                self.w(f"g_{A} = g_{A} + {sign} * g_{T};")
            else:
                self.w(f"g_{A} = g_{A} + g_div({sign} * g_{T}, {self.atom_real(a)}, code);")
                self.fail_check(label)


def _cid(name):
    return name.replace("!", "_x").replace("~", "_t")


def _collect_vars(stmts, acc):
    for s in stmts:
        if isinstance(s, (Alloc, Dealloc)):
            acc.add(s.name)
        elif isinstance(s, For):
            acc.add(s.var)
            _collect_vars(s.body, acc)
        elif isinstance(s, While):
            _collect_vars(s.body, acc)
        elif isinstance(s, If):
            _collect_vars(s.then, acc)
            _collect_vars(s.els, acc)
    return acc


def generate(src, fname, int_params=(), mode="grad"):
    """CUDA source of the batched gradient (mode "grad") or forward-over-reverse
    Hessian-column (mode "hess": the same code over Dual numbers, tangent on
    the Float parameter `dir`) kernel of `fname`, and its layout."""
    if mode not in ("grad", "hess"):
        raise KindError(f"codegen mode {mode!r}")
    fns = _Parser(src).program()
    if fname not in fns:
        raise UnsupportedProgram(f"codegen: no function named {fname!r}")
    params, body = fns[fname]
    int_params = set(int_params)
    kinds = {p: ("i" if p in int_params else "f") for p in params}
    fwd = _expand(body)
    inv = _expand(_invert_list(body))
    floats = [p for p in params if kinds[p] == "f"]
    ints = [p for p in params if kinds[p] == "i"]
    locals_ = sorted(_collect_vars(fwd, set()) | _collect_vars(inv, set()))
    em_f = _Emitter(params, kinds, fwd, fname)
    em_f.depth = 2
    em_f.stmts(fwd, False, "fwd_done")
    em_g = _Emitter(params, dict(em_f.kinds), inv, fname)
    em_g.depth = 2
    em_g.stmts(inv, True, "grad_done")
    allk = dict(em_f.kinds)
    allk.update(em_g.kinds)
    decl = []
    for v in locals_:
        if v in params:
            raise UnsupportedProgram(f"codegen: {v!r} shadows a parameter")
        k = allk.get(v, "f")
        decl.append(f"    long long v_{_cid(v)} = 0;" if k == "i"
                    else f"    R v_{_cid(v)} = R(0.0), g_{_cid(v)} = R(0.0);")
    NF, NI = len(floats), len(ints)
    L = [_PRELUDE, "typedef Dl R;" if mode == "hess" else "typedef double R;",
         f"extern \"C\" __global__ void rlg_kernel(long long n, const double *__restrict__ fin,"
         " const long long *__restrict__ iin, const double *__restrict__ seeds,"
         " double tol, int chk, long long fuel, double *__restrict__ fout,"
         " double *__restrict__ gout, unsigned char *__restrict__ fail, int dir,"
         " double *__restrict__ hout) {",
         "  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;"
         " i += (long long)gridDim.x * blockDim.x) {",
         "    int code = 0;", "    long long ticks = 0;"]
    for j, p in enumerate(floats):
        L.append(f"    const R in_{_cid(p)} = R(fin[{j}LL * n + i]"
                 + (f", dir == {j} ? 1.0 : 0.0);" if mode == "hess" else ");"))
        L.append(f"    R v_{_cid(p)} = in_{_cid(p)}, g_{_cid(p)} = R(0.0);")
    for j, p in enumerate(ints):
        L.append(f"    long long v_{_cid(p)} = iin[{j}];")
    L += decl
    L.append("    // ---- run_function (plain forward) ----")
    L += em_f.lines
    L.append("  fwd_done:")
    L.append("    if (code) {")
    for j, p in enumerate(floats):
        L.append(f"      fout[{j}LL * n + i] = NAN; gout[{j}LL * n + i] = NAN;")
        if mode == "hess":
            L.append(f"      hout[{j}LL * n + i] = NAN;")
    L.append("      fail[i] = (unsigned char)code; continue; }")
    for j, p in enumerate(floats):
        L.append(f"    fout[{j}LL * n + i] = rl_p(v_{_cid(p)});")
    L.append("    // ---- uncall_function in gradient mode (seeded) ----")
    for j, p in enumerate(floats):
        L.append(f"    g_{_cid(p)} = R(seeds[{j}]);            // coerce_to_kind: Dual(seed, 0)")
    L.append("    ticks = 0;")
    L += em_g.lines
    L.append("  grad_done:")
    L.append("    if (!code) {      // the backward pass must restore every argument")
    for p in floats:
        L.append(f"      if (!(fabs(rl_p(v_{_cid(p)}) - rl_p(in_{_cid(p)})) <= tol)) code = RC_REV;")
    for j, p in enumerate(ints):
        L.append(f"      if (v_{_cid(p)} != iin[{j}]) code = RC_REV;")
    L.append("    }")
    for j, p in enumerate(floats):
        L.append(f"    gout[{j}LL * n + i] = code ? NAN : rl_p(g_{_cid(p)});")
        if mode == "hess":
            L.append(f"    hout[{j}LL * n + i] = code ? NAN : rl_t(g_{_cid(p)});")
    L.append("    if (code) {")
    for j, p in enumerate(floats):
        L.append(f"      fout[{j}LL * n + i] = NAN;")
    L.append("    }")
    L.append("    fail[i] = (unsigned char)code;")
    L.append("  }")
    L.append("}")
    L.append(r"""
extern "C" int rlg_launch(long long n, const double *fin, const long long *iin, const double *seeds,
                          double tol, int chk, long long fuel, double *fout, double *gout,
                          unsigned char *fail, int dir, double *hout, void *stream) {
  if (n <= 0) return 0;
  const int block = 128;
  long long grid = (n + block - 1) / block;
  if (grid > 148 * 16) grid = 148 * 16;
  rlg_kernel<<<(unsigned)grid, block, 0, (cudaStream_t)stream>>>(n, fin, iin, seeds, tol, chk, fuel,
                                                                fout, gout, fail, dir, hout);
  return (int)cudaGetLastError();
}
""")
    return "\n".join(L), floats, ints


# ---------------------------------------------------------------------------
# build + run
# ---------------------------------------------------------------------------

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
    """Compile generated CUDA source to a cached shared library (sm_100a)."""
    h = hashlib.sha256(source.encode()).hexdigest()[:20]
    so = os.path.join(_cache_dir(), f"rlg_{h}.so")
    if not os.path.exists(so):
        with tempfile.TemporaryDirectory() as td:
            cu = os.path.join(td, "k.cu")
            with open(cu, "w") as fh:
                fh.write(source)
            tmp = os.path.join(td, "k.so")
            cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-fmad=false",
                   "-shared", "-Xcompiler", "-fPIC", "-o", tmp, cu]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise NativeLibraryError("codegen: nvcc failed:\n" + r.stderr[-4000:])
            os.replace(tmp, so)
    return so


class CompiledFunction:
    """A reversible function compiled to one batched CUDA kernel.

    `gradient(inputs, seeds)` is the batched `gradient(program,
    GradRequest(fname, args_i, seeds))`: every Float parameter takes a CUDA
    float64 tensor (one row per element) or a scalar, every Int parameter a
    Python int; returns (primal outputs, gradients, fail codes) as dicts of
    tensors keyed by parameter name (Int parameters carry no gradient)."""

    def __init__(self, source_text, fname, int_params=()):
        self.fname = fname
        self._text, self._ints = source_text, tuple(int_params)
        self.source, self.floats, self.ints = generate(source_text, fname, int_params)
        self._lib = self._load(self.source)
        self._hlib = None

    @staticmethod
    def _load(source):
        lib = ctypes.CDLL(build(source))
        lib.rlg_launch.restype = ctypes.c_int
        lib.rlg_launch.argtypes = [ctypes.c_longlong] + [ctypes.c_void_p] * 3 + [
            ctypes.c_double, ctypes.c_int, ctypes.c_longlong] + [ctypes.c_void_p] * 3 + [
            ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        return lib

    def hessian(self, inputs, tol=1e-9, invcheck=True, max_steps=10**9):
        """Batched reference `hessian(program, fname, args_i)` (autodiff.py:
        216-257) over the Float parameters: the gradient sweeps over Dual
        numbers, one launch per tangent direction.  Returns (H, fail) with H
        of shape (n, F, F), H[:, k, j] = d(cotangent k) / d(parameter j)."""
        if self._hlib is None:
            src, _, _ = generate(self._text, self.fname, self._ints, mode="hess")
            self._hlib = self._load(src)
        cols = []
        fail = None
        for j in range(len(self.floats)):
            _, _, f, h = self._run(self._hlib, inputs, None, tol, invcheck, max_steps, dir_=j)
            cols.append(h)
            fail = f if fail is None else torch.maximum(fail, f)
        H = torch.stack(cols, -1).permute(1, 0, 2).contiguous()   # (n, F_k, F_j)
        return H, fail

    def gradient(self, inputs, seeds=None, tol=1e-9, invcheck=True, max_steps=10**9):
        primal, grads, fail, _ = self._run(self._lib, inputs, seeds, tol, invcheck, max_steps)
        return primal, grads, fail

    def _run(self, lib, inputs, seeds, tol, invcheck, max_steps, dir_=-1):
        if not torch.cuda.is_available():
            raise UnsupportedProgram("codegen kernels need a CUDA device (no CPU path)")
        dev = torch.device("cuda", torch.cuda.current_device())
        n = None
        for p in self.floats:
            v = inputs.get(p)
            if isinstance(v, torch.Tensor):
                if not v.is_cuda or v.dtype != torch.float64 or v.dim() != 1:
                    raise KindError(f"{p} must be a 1-D CUDA float64 tensor")
                n = v.shape[0] if n is None else n
                if v.shape[0] != n:
                    raise KindError("all batched inputs need the same length")
        if n is None:
            n = 1
        cols = []
        for p in self.floats:
            v = inputs.get(p, 0.0)
            cols.append(v.contiguous() if isinstance(v, torch.Tensor)
                        else torch.full((n,), float(v), dtype=torch.float64, device=dev))
        fin = torch.stack(cols) if cols else torch.zeros((0, n), dtype=torch.float64, device=dev)
        ivals = []
        for p in self.ints:
            v = inputs.get(p)
            if not isinstance(v, int) or isinstance(v, bool):
                raise KindError(f"{p} must be an Int")
            ivals.append(v)
        iin = torch.tensor(ivals or [0], dtype=torch.int64, device=dev)
        sd = {self.floats[0]: 1.0} if seeds is None else {}
        if seeds is not None:
            for pname, path, val in seeds:
                if pname not in self.floats or path:
                    raise KindError(f"seed target {pname!r} is not a Float scalar parameter")
                sd[pname] = float(val)
        if seeds is None and not self.floats:
            raise KindError("no differentiable parameter to seed")
        sv = torch.tensor([sd.get(p, 0.0) for p in self.floats] or [0.0], dtype=torch.float64,
                          device=dev)
        fout = torch.empty_like(fin)
        gout = torch.empty_like(fin)
        hout = torch.empty_like(fin) if dir_ >= 0 else None
        fail = torch.empty(n, dtype=torch.uint8, device=dev)
        rc = lib.rlg_launch(n, fin.data_ptr(), iin.data_ptr(), sv.data_ptr(), float(tol),
                            int(bool(invcheck)), int(max_steps), fout.data_ptr(), gout.data_ptr(),
                            fail.data_ptr(), int(dir_),
                            hout.data_ptr() if hout is not None else None,
                            torch.cuda.current_stream().cuda_stream)
        if rc:
            raise NativeLibraryError(f"codegen kernel launch failed (cudaError {rc})")
        primal = {p: fout[j] for j, p in enumerate(self.floats)}
        primal.update({p: inputs[p] for p in self.ints})
        grads = {p: gout[j] for j, p in enumerate(self.floats)}
        return primal, grads, fail, hout


def compile_function(source_text, fname, int_params=()):
    """Compile function `fname` of reversible-DSL source to a batched CUDA
    gradient kernel (see CompiledFunction)."""
    return CompiledFunction(source_text, fname, int_params)
