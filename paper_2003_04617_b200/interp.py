"""Drop-in `run`, `uncall` and `check_reversibility` (reference
interpreter.py:1021-1069) for the registered programs, on the GPU.

`run(program, fname, args)` executes f forward and returns the updated
arguments; `uncall` executes the mechanically inverted ~f; both perform the
reference's reversibility checks on device and raise its exception classes.
`check_reversibility` runs f then ~f and reports the deviation of the
round trip, errors embedded in the report like the reference's.
"""

import json
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels
from .autodiff import (_check_opts, _device, _is_float, _is_int, _lookup, gmm_beyond_tiles,
                       ba_fuel_check, gmm_fuel_check)
from .errors import KindError, RevLangError, error_for_code
from .values import to_numpy


def _raise_first(fail, where):
    f = fail.cpu().numpy() if isinstance(fail, torch.Tensor) else np.asarray(fail)
    if f.any():
        raise error_for_code(int(f[np.nonzero(f)[0][0]]), where)


def _run_besselj(fdef, args, opts, direction):
    if len(args) != 3:
        raise KindError(f"besselj takes 3 arguments, got {len(args)}")
    out0, nu, z = args
    if not _is_int(nu) or not (_is_float(z) or _is_int(z)):
        raise KindError("besselj(out!, nu::Int, z)")
    dev = _device()
    t = lambda v: torch.tensor([float(v)], dtype=torch.float64, device=dev)  # noqa: E731
    r = kernels.besselj_run(t(z), int(nu), out_in=t(out0), direction=direction,
                            thr=fdef.constants.get("thr", 1e-16), tol=opts.float_tolerance,
                            invcheck=opts.invcheck, max_steps=opts.max_steps)
    _raise_first(r.fail, "besselj")
    return [float(r.out[0].item()), nu, z]


def _run_ba_proj(fdef, args, opts, direction):
    if len(args) != 7:
        raise KindError(f"ba_proj takes 7 arguments, got {len(args)}")
    e1, e2, cam, X, w, f1, f2 = args
    ba_fuel_check(to_numpy(cam, "cam"), opts.max_steps)
    dev = _device()
    tt = lambda a: torch.as_tensor(np.asarray(a, np.float64), device=dev)  # noqa: E731
    r = kernels.ba_residuals(tt(to_numpy(cam, "cam").reshape(1, 11)),
                             tt(to_numpy(X, "X").reshape(1, 3)), tt([float(w)]),
                             tt([[float(f1), float(f2)]]),
                             torch.zeros((1, 2), dtype=torch.int32, device=dev),
                             tol=opts.float_tolerance, invcheck=opts.invcheck)
    _raise_first(r.fail, "ba_proj")
    e = r.out[0].cpu().numpy()
    # e! +/-= w * d  (the residual is the device's; one IEEE add/sub here)
    s = 1.0 if direction > 0 else -1.0
    return [float(e1) + s * e[0], float(e2) + s * e[1], cam, X, w, f1, f2]


def _run_ba_weight(fdef, args, opts, direction):
    if len(args) != 2:
        raise KindError(f"ba_weight takes 2 arguments, got {len(args)}")
    e0, w = args
    ba_fuel_check(None, opts.max_steps, "ba_weight")
    dev = _device()
    tt = lambda a: torch.as_tensor(np.asarray(a, np.float64), device=dev)  # noqa: E731
    cam = np.zeros(11)
    cam[6] = 1.0
    r = kernels.ba_residuals(tt(cam.reshape(1, 11)), tt([[0.0, 0.0, 1.0]]), tt([float(w)]),
                             tt([[0.0, 0.0]]), torch.zeros((1, 2), dtype=torch.int32, device=dev),
                             tol=opts.float_tolerance, invcheck=opts.invcheck)
    _raise_first(r.fail, "ba_weight")
    ew = float(r.out[0, 2].item())
    return [float(e0) + (ew if direction > 0 else -ew), w]


def _run_gmm(fdef, args, opts, direction):
    if len(args) != 14:
        raise KindError(f"gmm takes 14 arguments, got {len(args)}")
    err0, alphas, means, icf, x = args[:5]
    names = fdef.param_names()
    for nm, s in zip(names[5:11], args[5:11]):
        if np.any(to_numpy(s, nm) != 0.0):
            raise KindError(f"scratch argument {nm!r} must be zero on entry")
    ga, wm, cst = args[11:14]
    dev = _device()
    tt = lambda v: torch.as_tensor(v, device=dev)  # noqa: E731
    a = (tt(to_numpy(alphas, "alphas", 1)), tt(to_numpy(means, "means", 2)),
         tt(to_numpy(icf, "icf", 2)), tt(to_numpy(x, "x", 2)), float(ga), int(wm), float(cst))
    # err! accumulated from err0 in the order of gmm (run) or ~gmm (uncall)
    r = kernels.gmm_run(*a, err0=float(err0), direction=direction, tol=opts.float_tolerance,
                        invcheck=opts.invcheck)
    gmm_fuel_check(a[0], a[1].shape[1], a[3].shape[0], r, opts.max_steps)
    return [float(r.out.item())] + list(args[1:])


_RUNNERS = {"besselj": _run_besselj, "ba_proj": _run_ba_proj, "ba_weight": _run_ba_weight,
            "gmm": _run_gmm}


def run(program, fname, args, opts=None):
    """Reference `run` (interpreter.py:1021): execute f forward on the device
    (a registered kernel, else the function compiled by codegen)."""
    return _dispatch(program, fname, args, opts, +1)


def _dispatch(program, fname, args, opts, direction):
    opts = _check_opts(opts)
    prog, fdef, reg = _lookup(program, fname)
    if not reg or gmm_beyond_tiles(fdef, list(args)):
        from . import generic
        return generic.run(prog, fdef, list(args), opts, direction)
    return _RUNNERS[fdef.kernel.handler](fdef, list(args), opts, direction)


def uncall(program, fname, args, opts=None):
    """Reference `uncall` (interpreter.py:1026): execute ~f; uncall(run(a)) == a."""
    return _dispatch(program, fname, args, opts, -1)


@dataclass
class CheckReport:
    fname: str
    ok: bool
    max_deviation: float
    error: str = None
    per_arg_deviation: list = None
    checks_passed: dict = None

    def to_json(self):
        return json.dumps({"function": self.fname, "ok": self.ok,
                           "max_deviation": self.max_deviation, "error": self.error,
                           "per_arg_deviation": self.per_arg_deviation,
                           "checks_passed": self.checks_passed}, sort_keys=True)


def _deviation(a, b):
    if _is_float(a) or _is_int(a):
        return abs(float(a) - float(b))
    return float(np.max(np.abs(to_numpy(a, "a") - to_numpy(b, "b")), initial=0.0))


def check_reversibility(program, fname, args, opts=None):
    """Reference `check_reversibility` (interpreter.py:1051): run f then ~f
    (both on the device, all checks on) and report the deviation from the
    original arguments; runtime errors are embedded, not raised.  The device
    does not count passed checks per kind (checks_passed = None)."""
    opts = _check_opts(opts)
    try:
        mid = run(program, fname, args, opts)
        back = uncall(program, fname, mid, opts)
        per_arg = [_deviation(o, r) for o, r in zip(args, back)]
        worst = max(per_arg, default=0.0)
        return CheckReport(fname, worst <= opts.float_tolerance, worst, None, per_arg, None)
    except (RevLangError, OverflowError) as err:
        return CheckReport(fname, False, float("inf"), str(err), None, None)
