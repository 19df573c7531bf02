"""Error classes, mirroring the reference's `revlang.errors` (errors.py:33-140).

Names, hierarchy and meaning are the reference's, so code that catches
`revlang.RevError` / `DirtyAncilla` / ... keeps working.  Device kernels
cannot throw: they write a per-element status code
(include/revgpu.h `RL_ERR_*`), which `raise_for_code` maps back onto these
classes.
"""

from dataclasses import dataclass


@dataclass(frozen=True)
class SourceSpan:
    file: str = "<string>"
    line: int = 0
    col: int = 0
    end_line: int = 0
    end_col: int = 0

    def __str__(self):
        return f"{self.file}:{self.line}:{self.col}"


NO_SPAN = SourceSpan()


class RevLangError(Exception):
    """Base for all toolchain errors (reference errors.py:33-46)."""

    def __init__(self, message, span=None):
        super().__init__(message)
        self.message = message
        self.span = span if span is not None else NO_SPAN

    @property
    def name(self):
        return type(self).__name__

    def __str__(self):
        return f"{self.name} at {self.span}: {self.message}"


class RevError(RevLangError):
    """Runtime reversibility errors (reference errors.py:60)."""


class PostconditionMismatch(RevError):
    pass


class DirtyAncilla(RevError):
    def __init__(self, message, span=None, name=None, residual=None):
        super().__init__(message, span)
        self.var_name = name
        self.residual = residual


class LoopIteratorMutated(RevError):
    pass


class AliasedArguments(RevError):
    pass


class RevDomainError(RevError):
    pass


class FuelExhausted(RevError):
    pass


class IndexOutOfBounds(RevError):
    pass


class AssertFailed(RevError):
    pass


class KindError(RevError):
    pass


class MissingAdjoint(RevError):
    pass


class UnknownFunction(RevError):
    pass


class UnknownExample(RevLangError):
    pass


class UnsupportedProgram(RevLangError):
    """The program has no registered device kernel.  There is deliberately
    no CPU fallback (north star): register a kernel or use the reference
    interpreter."""


class NativeLibraryError(RuntimeError):
    """librevgpu.so is missing, failed to load, or reported a CUDA error."""


# include/revgpu.h status codes -> classes
_CODE_CLASSES = {
    1: PostconditionMismatch,
    2: DirtyAncilla,
    3: RevDomainError,
    4: LoopIteratorMutated,
    5: RevError,
    6: FuelExhausted,
    7: KindError,
    8: IndexOutOfBounds,
    9: OverflowError,  # CPython math.exp raises OverflowError (values.py:362)
    10: AliasedArguments,
    11: AssertFailed,
    12: ValueError,    # round(nan) in Fixed.from_real (generated kernels only)
    13: RecursionError,  # a recursive call past the generated kernel's inlined depth
}

CODE_NAMES = {0: "", 1: "PostconditionMismatch", 2: "DirtyAncilla", 3: "RevDomainError",
              4: "LoopIteratorMutated", 5: "RevError", 6: "FuelExhausted", 7: "KindError",
              8: "IndexOutOfBounds", 9: "OverflowError", 10: "AliasedArguments",
              11: "AssertFailed", 12: "ValueError", 13: "RecursionError"}

_MESSAGES = {
    1: "branch or loop postcondition mismatch",
    2: "ancilla released with a residual above the float tolerance",
    3: "value outside the domain of log/sqrt/division",
    4: "loop variable was modified in the body",
    5: "backward pass failed to restore an argument's primal value",
    6: "exceeded the statement budget",
    7: "value-kind mismatch",
    8: "index out of bounds",
    9: "math range error",
    10: "instruction arguments share storage",
    11: "@safe assertion failed",
    12: "cannot convert float NaN to integer",
    13: "recursion deeper than the generated kernel's inlined levels (REVGPU_CODEGEN_DEPTH)",
}


def error_for_code(code, where=""):
    cls = _CODE_CLASSES.get(int(code), RevError)
    msg = _MESSAGES.get(int(code), f"device status {int(code)}")
    if where:
        msg = f"{msg} ({where})"
    if cls in (OverflowError, ValueError, RecursionError):
        return cls(msg)
    return cls(msg)


def raise_for_code(code, where=""):
    if int(code) != 0:
        raise error_for_code(code, where)
