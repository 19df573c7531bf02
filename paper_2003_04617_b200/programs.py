"""Programs and the device-kernel registry.

The reference's programs are `.rnl` text parsed into an IR (parser.py:593,
ir.py:235) and executed by an interpreter.  Here a program is recognised,
function by function, against the registered benchmark programs
(programs/*.rnl) by a normalised token fingerprint; each registered
function is bound to a hand-written sm_100a kernel.  Any other function is
compiled to a device kernel by codegen.py when it is called (generic.py);
there is no interpreter and no CPU fallback.

Fingerprints ignore comments, whitespace, line breaks, the ASCII/Unicode
spelling of arrows (parser.py:143-164) and the spelling of numeric
literals (1e-16 == 1.0e-16).  A registered function may declare literal
"holes" whose values become kernel parameters (the Bessel series
threshold), so that a user can change them without a new kernel.

Reference counterparts: `parse_program` (parser.py:593), `load_example` /
`CATALOG` (stdlib.py:18-49).
"""

import os
import re
from dataclasses import dataclass, field

from .errors import UnknownExample, UnknownFunction, UnsupportedProgram

PROG_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "programs")

_UNICODE = {"←": "<-", "→": "->", "⊻=": "xor="}
_TOKEN = re.compile(r"""
    (?P<num>(?:\d+\.\d*|\.\d+|\d+)(?:[eE][+-]?\d+)?(?:fx|ul|im)?)
  | (?P<name>~?@?[A-Za-z_][A-Za-z_0-9]*!?)
  | (?P<punct><-|->|\+=|-=|\*=|/=|xor=|==|!=|<=|>=|&&|\|\||\|>|::|[-+*/^%(),\[\]<>~:.=!])
  | (?P<ws>\s+)
""", re.VERBOSE)


def tokenize(text):
    """Normalised token stream: comments and whitespace dropped, numeric
    literals canonicalised to ('num', value)."""
    for u, a in _UNICODE.items():
        text = text.replace(u, a)
    text = re.sub(r"#[^\n]*", "", text)
    out = []
    pos = 0
    while pos < len(text):
        m = _TOKEN.match(text, pos)
        if not m:
            raise UnsupportedProgram(f"cannot tokenise program text near {text[pos:pos + 20]!r}")
        pos = m.end()
        kind = m.lastgroup
        tok = m.group(kind)
        if kind == "ws":
            continue
        if kind == "num":
            raw = tok
            if raw.endswith(("fx", "ul", "im")):
                out.append(("num", raw))
            elif re.fullmatch(r"\d+", raw):
                out.append(("int", int(raw)))
            else:
                out.append(("num", float(raw)))
        else:
            out.append((kind, tok))
    return out


_OPENERS = {"fn", "begin", "for", "while", "if"}


def split_functions(tokens):
    """{name: (params, token list)} for every `fn ... end` block."""
    funcs = {}
    i = 0
    while i < len(tokens):
        if tokens[i] != ("name", "fn"):
            raise UnsupportedProgram(f"expected 'fn', got {tokens[i][1]!r}")
        depth = 0
        j = i
        while j < len(tokens):
            kind, val = tokens[j]
            if kind == "name" and val in _OPENERS:
                depth += 1
            elif kind == "name" and val == "end":
                depth -= 1
                if depth == 0:
                    break
            j += 1
        if j >= len(tokens):
            raise UnsupportedProgram("unterminated function definition")
        body = tokens[i:j + 1]
        name = body[1][1]
        params = []
        k = 3  # fn NAME ( ...
        while body[k] != ("punct", ")"):
            if body[k][0] == "name" and body[k - 1] != ("punct", "::"):
                params.append(body[k][1])
            k += 1
        funcs[name] = (params, body)
        i = j + 1
    return funcs


@dataclass
class Hole:
    """A literal position in a registered template that becomes a kernel
    parameter; `default` is the value in the shipped program."""
    name: str
    default: float


@dataclass
class KernelFunction:
    """A registered function: its template token stream and its device
    handler name (see autodiff._HANDLERS)."""
    name: str
    params: list
    template: list
    handler: str
    holes: dict = field(default_factory=dict)

    def match(self, tokens):
        if len(tokens) != len(self.template):
            return None
        captured = {}
        for a, b in zip(self.template, tokens):
            if isinstance(a, Hole):
                if b[0] not in ("num", "int"):
                    return None
                captured[a.name] = float(b[1])
            elif a != b:
                return None
        return captured


@dataclass
class FunctionDef:
    """A function of a loaded program: bound to a kernel, or not."""
    name: str
    params: list
    kernel: KernelFunction = None
    constants: dict = field(default_factory=dict)

    def param_names(self):
        return list(self.params)


class Program:
    """A program whose functions are looked up by name (reference ir.Program,
    ir.py:235).  Unregistered functions are kept with their source text for
    the generic compiler (codegen.py / generic.py)."""

    def __init__(self, functions, source="", filename="<string>"):
        self.functions = {f.name: f for f in functions}
        self.source = source
        self.filename = filename

    def __iter__(self):
        return iter(self.functions.values())

    def get(self, name):
        f = self.functions.get(name)
        if f is None:
            raise UnknownFunction(f"no function named {name!r}")
        return f

    def __repr__(self):
        names = ", ".join(f"{n}{'' if f.kernel else ' (no kernel)'}"
                          for n, f in self.functions.items())
        return f"Program({self.filename}: {names})"


# --- registry -------------------------------------------------------------

_REGISTRY = {}          # function name -> KernelFunction
_HOLES = {"besselj": {("num", 1e-16): "thr"}}
_HANDLERS = {"besselj": "besselj", "ba_proj": "ba_proj", "rodrigues": None,
             "ba_weight": "ba_weight", "gmm": "gmm"}
CATALOG = {
    "besselj": ("besselj.rnl", "besselj"),
    "gmm": ("gmm.rnl", "gmm"),
    "ba_proj": ("ba.rnl", "ba_proj"),
    "ba_weight": ("ba.rnl", "ba_weight"),
}


def _register_file(filename):
    with open(os.path.join(PROG_DIR, filename)) as fh:
        funcs = split_functions(tokenize(fh.read()))
    for name, (params, toks) in funcs.items():
        holes = {}
        template = list(toks)
        for lit, hname in _HOLES.get(name, {}).items():
            for idx, tok in enumerate(template):
                if tok == lit:
                    template[idx] = Hole(hname, float(lit[1]))
                    holes[hname] = float(lit[1])
        _REGISTRY[name] = KernelFunction(name, params, template, _HANDLERS.get(name), holes)


for _f in ("besselj.rnl", "ba.rnl", "gmm.rnl"):
    _register_file(_f)


def registered_functions():
    return dict(_REGISTRY)


def program_text(name):
    with open(os.path.join(PROG_DIR, CATALOG[name][0])) as fh:
        return fh.read()


def parse_program(text, filename="<string>"):
    """Tokenise `text` and bind each function to its registered kernel.

    Mirrors reference parse_program (parser.py:593) for the registered
    programs.  A function whose text differs from every registered one is
    kept without a kernel (calling it compiles it with codegen.py).  Helper
    functions (rodrigues) bind only together with their caller."""
    funcs = split_functions(tokenize(text))
    out = []
    for name, (params, toks) in funcs.items():
        kf = _REGISTRY.get(name)
        captured = kf.match(toks) if kf is not None else None
        if captured is None:
            out.append(FunctionDef(name, params))
        else:
            consts = dict(kf.holes)
            consts.update(captured)
            out.append(FunctionDef(name, params, kf, consts))
    prog = Program(out, text, filename)
    # ba_proj calls rodrigues: both must be the registered versions
    ba = prog.functions.get("ba_proj")
    if ba is not None and ba.kernel is not None:
        rod = prog.functions.get("rodrigues")
        if rod is None or rod.kernel is None:
            ba.kernel = None
    return prog


def as_program(program):
    """Accept our Program or program source text (the reference's
    parse_program input, parser.py:593).  A reference revlang.Program object
    is not interpreted here — the product runs no reference code — pass its
    source (revlang.parser.pretty_print(p)) instead."""
    if isinstance(program, Program):
        return program
    if isinstance(program, str):
        return parse_program(program)
    raise UnsupportedProgram(
        f"cannot interpret {type(program).__name__} as a program: pass program text "
        "(e.g. revlang.parser.pretty_print(p)) or a Program from parse_program")


_cache = {}


def load_example(name):
    """Parse a registered benchmark program (reference stdlib.load_example,
    stdlib.py:38-49)."""
    if name not in CATALOG:
        raise UnknownExample(f"no example named {name!r}; known: {', '.join(sorted(CATALOG))}")
    filename = CATALOG[name][0]
    if filename not in _cache:
        with open(os.path.join(PROG_DIR, filename)) as fh:
            _cache[filename] = parse_program(fh.read(), filename)
    return _cache[filename]


def entry_function(name):
    return CATALOG[name][1]
