"""paper_2003_04617_b200 — B200-native reversible-AD gradient kernels.

The data-parallel hot path of arXiv 2003.04617 (NiLang) as re-stated by the
reference `revlang` package: forward run, uncompute and adjoint sweep of a
reversible program, independently over a large batch, compiled to ONE
sm_100a kernel per program with no tape (include/revgpu.h).

Public surface (mirrors `revlang.__init__`, reference __init__.py:8-31, for
the gradient path):
  parse_program, load_example, Program, GradRequest, ExecOptions,
  gradient, jacobian, the revlang error classes;
plus the batched device API over torch CUDA tensors:
  besselj_grad, ba_jacobian, gmm_grad (kernels.py) and the data-parallel
  helpers in parallel.py.
"""

from .autodiff import (ExecOptions, GradRequest, HessianResult, gradient, gradient_batch,
                       finite_difference, hessian, jacobian)
from .errors import (AliasedArguments, AssertFailed, DirtyAncilla, FuelExhausted, IndexOutOfBounds,
                     KindError, LoopIteratorMutated, MissingAdjoint, NativeLibraryError,
                     PostconditionMismatch, RevDomainError, RevError, RevLangError,
                     UnknownExample, UnknownFunction, UnsupportedProgram)
from .codegen import CompiledFunction, compile_function
from .interp import CheckReport, check_reversibility, run, uncall
from .kernels import (BACsr, BAResult, BesselHessResult, BesselResult, GMMResult, RunResult, ba_jacobian, ba_jacobian_csr,
                      ba_jacobian_csr_host, ba_residuals,
                      besselj_grad, besselj_grad_host, besselj_hess, besselj_run, gmm_grad, gmm_gradient,
                      gmm_objective, gmm_run, seq_sum)
from .programs import CATALOG, Program, entry_function, load_example, parse_program
from .values import Array, Fixed

__all__ = [
    "HessianResult", "finite_difference", "hessian", "gradient_batch", "CompiledFunction", "compile_function", "BesselHessResult", "besselj_hess",
    "AliasedArguments", "AssertFailed", "Array", "Fixed", "BACsr", "BAResult", "ba_jacobian_csr", "ba_jacobian_csr_host", "BesselResult", "CATALOG", "CheckReport",
    "DirtyAncilla", "RunResult", "ba_residuals", "besselj_run", "check_reversibility",
    "gmm_objective", "gmm_gradient", "gmm_run", "seq_sum", "run", "uncall",
    "ExecOptions", "FuelExhausted", "GMMResult", "GradRequest", "IndexOutOfBounds",
    "KindError", "LoopIteratorMutated", "MissingAdjoint", "NativeLibraryError",
    "PostconditionMismatch", "Program", "RevDomainError", "RevError", "RevLangError",
    "UnknownExample", "UnknownFunction", "UnsupportedProgram", "ba_jacobian", "besselj_grad",
    "besselj_grad_host", "entry_function", "gmm_grad", "gradient", "jacobian",
    "load_example", "parse_program",
]

__version__ = "0.1.0"
