"""Drop-in entry points for functions WITHOUT a hand-written kernel: the
function is compiled by codegen.py (the generic .rnl -> CUDA path) for the
kinds and array shapes of the call's arguments and run on the device.  There
is still no CPU path: no GPU, no result.

Used by autodiff.gradient / gradient_batch / hessian / jacobian and
interp.run / uncall / check_reversibility when the program's function is not
one of the registered benchmark kernels (besselj, ba_proj, ba_weight, gmm).
Argument kinds follow the reference's values: Python int -> Int, float ->
Float, Array (ours, the reference's, numpy, torch) of floats -> Float array,
of ints -> Int array, Complex -> two Float leaves, Fixed (anything with the
reference Fixed's `raw` / `to_float`) -> a raw int64 Q31.32 cell; ULog /
Record / Bool arguments are outside the compiled subset (UnsupportedProgram).  Results come back in the
reference's containers (floats, ints, Arrays of the caller's class) and a
device error raises the reference's exception class for that row.
"""

import numpy as np
import torch

from . import codegen
from .errors import KindError, UnsupportedProgram, error_for_code
from .values import Array

_CACHE = {}


def _is_int(v):
    return isinstance(v, (int, np.integer)) and not isinstance(v, (bool, np.bool_))


def _is_float(v):
    return isinstance(v, (float, np.floating))


def _is_fixed(v):
    """The reference's Fixed (values.py:28): a Q31.32 raw integer."""
    return hasattr(v, "raw") and hasattr(v, "to_float")


def _fx_float(raw):
    """values.Fixed.to_float of raw int64 values (numpy arrays): raw / 2^32."""
    return np.asarray(raw, dtype=np.int64).astype(np.float64) * 2.0 ** -32


def _as_array(v):
    """ndarray of an Array-like, or None."""
    if isinstance(v, torch.Tensor):
        return v.detach().cpu().numpy()
    if isinstance(v, np.ndarray):
        return v
    if hasattr(v, "data") and hasattr(v, "shape"):
        data = list(v.data)
        if data and all(_is_int(x) for x in data):
            return np.asarray(data, dtype=np.int64).reshape(tuple(v.shape))
        if not all(_is_float(x) or _is_int(x) for x in data):
            raise UnsupportedProgram("codegen: arrays hold Float or Int values only")
        if any(_is_int(x) for x in data):
            raise UnsupportedProgram("codegen: mixed Int / Float arrays are not supported")
        return np.asarray(data, dtype=np.float64).reshape(tuple(v.shape))
    return None


def _kind(v, name):
    """("f" | "i" | "a" | "ai", shape) of one argument value."""
    if isinstance(v, (bool, np.bool_)):
        raise UnsupportedProgram(f"codegen: Bool argument {name!r} is not supported")
    if _is_int(v):
        return "i", ()
    if _is_float(v):
        return "f", ()
    if _is_fixed(v):
        return "x", ()
    if isinstance(v, complex) or (hasattr(v, "re") and hasattr(v, "im")):
        return "c", ()                                 # Complex: two Float leaves
    a = _as_array(v)
    if a is None:
        raise UnsupportedProgram(f"codegen: argument {name!r} of kind {type(v).__name__} is "
                                 "outside the compiled subset")
    if a.ndim not in (1, 2):
        raise KindError(f"{name}: arrays are 1-d or 2-d")
    return ("ai" if a.dtype.kind in "iu" else "a"), tuple(a.shape)


def compiled(prog, fname, kinds):
    """The CompiledFunction of prog's `fname` for {param: (kind, shape)}."""
    if not torch.cuda.is_available():
        raise UnsupportedProgram(f"{fname}: no CUDA device (generated kernels have no CPU path)")
    ints = tuple(p for p, (k, _) in kinds.items() if k in ("i", "ai"))
    shapes = {p: s for p, (k, s) in kinds.items() if k in ("a", "ai")}
    cplx = tuple(p for p, (k, _) in kinds.items() if k == "c")
    fixed = tuple(p for p, (k, _) in kinds.items() if k == "x")
    key = (prog.source, fname, ints, tuple(sorted(shapes.items())), cplx, fixed)
    if key not in _CACHE:
        _CACHE[key] = codegen.CompiledFunction(prog.source, fname, ints, shapes, cplx, fixed)
    return _CACHE[key]


def _call_kinds(fdef, args):
    names = fdef.param_names()
    if len(args) != len(names):
        raise KindError(f"{fdef.name} takes {len(names)} arguments, got {len(args)}")
    return names, {p: _kind(v, p) for p, v in zip(names, args)}


def _inputs(names, kinds, args):
    out = {}
    for p, v in zip(names, args):
        k = kinds[p][0]
        out[p] = float(v) if k == "f" else int(v) if k == "i" else (
            complex(v) if k == "c" and isinstance(v, complex) else
            v if k in ("c", "x") else _as_array(v))
    return out


def _back(template, kind, value):
    """One output row in the reference's container."""
    v = value.cpu().numpy() if isinstance(value, torch.Tensor) else np.asarray(value)
    if kind == "f":
        return float(v)
    if kind == "i":
        return int(v)
    if kind == "x":                                   # the caller's Fixed class, from raw
        raw = int(v)
        return type(template)(raw) if _is_fixed(template) else raw
    if kind == "c":                                   # the caller's Complex class
        z = complex(v)
        if hasattr(template, "re") and hasattr(template, "im"):
            return type(template)(float(z.real), float(z.imag))
        return z
    data = [int(x) for x in v.ravel()] if kind == "ai" else [float(x) for x in v.ravel()]
    if isinstance(template, torch.Tensor):
        return torch.as_tensor(v.copy())
    if isinstance(template, np.ndarray):
        return v.copy()
    cls = type(template) if hasattr(template, "data") and hasattr(template, "shape") else Array
    try:
        return cls(data, v.shape)
    except TypeError:
        return Array(data, v.shape)


def _raise(fail, fname):
    code = int(fail[0].item())
    if code:
        raise error_for_code(code, fname)


def gradient(prog, fdef, req, opts):
    """Reference gradient() (autodiff.py:136-180) through a generated kernel."""
    names, kinds = _call_kinds(fdef, list(req.args))
    k = compiled(prog, fdef.name, kinds)
    primal, grads, fail = k.gradient(_inputs(names, kinds, req.args), seeds=req.seeds,
                                     tol=opts.float_tolerance, invcheck=opts.invcheck,
                                     max_steps=opts.max_steps)
    _raise(fail, fdef.name)
    outs = [_back(v, kinds[p][0], primal[p][0]) for p, v in zip(names, req.args)]
    report = req.wrt if req.wrt is not None else names
    g = {}
    for p in report:
        if p not in names:
            raise KindError(f"wrt names unknown parameter {p!r}")
        v = req.args[names.index(p)]
        g[p] = _back(v, kinds[p][0], grads[p][0]) if p in grads else None
    return outs, g


def run(prog, fdef, args, opts, direction):
    """Reference run / uncall (interpreter.py:1021-1028) through a generated kernel."""
    names, kinds = _call_kinds(fdef, list(args))
    k = compiled(prog, fdef.name, kinds)
    out, fail = k.run(_inputs(names, kinds, args), direction, tol=opts.float_tolerance,
                      invcheck=opts.invcheck, max_steps=opts.max_steps)
    _raise(fail, fdef.name)
    return [_back(v, kinds[p][0], out[p][0]) for p, v in zip(names, args)]


def hessian(prog, fdef, args, opts):
    """Reference hessian() (autodiff.py:216-257): forward-over-reverse over
    every Float leaf, one Dual-number launch per leaf."""
    names, kinds = _call_kinds(fdef, list(args))
    k = compiled(prog, fdef.name, kinds)
    H, fail = k.hessian(_inputs(names, kinds, args), tol=opts.float_tolerance,
                        invcheck=opts.invcheck, max_steps=opts.max_steps)
    _raise(fail, fdef.name)
    return H[0].cpu().numpy()


def gradient_batch(prog, fdef, inputs, seeds, wrt, opts):
    """Batched gradient: row i of every tensor is one call.  A Float
    parameter takes an (n,) tensor or a float, a Float array an (n, *shape)
    tensor or one Array-like shared by all rows, Int parameters plain ints /
    Int Array-likes (uniform over the batch).  Returns (primal, grads, fail)."""
    names = fdef.param_names()
    kinds, vals = {}, {}
    for p in names:
        if p not in inputs:
            raise KindError(f"gradient_batch: no input for parameter {p!r}")
        v = inputs[p]
        if isinstance(v, torch.Tensor) and v.dtype == torch.float64 and v.dim() >= 1:
            kinds[p] = ("f", ()) if v.dim() == 1 else ("a", tuple(v.shape[1:]))
            vals[p] = v
        elif isinstance(v, torch.Tensor) and v.dtype == torch.complex128 and v.dim() == 1:
            kinds[p] = ("c", ())
            vals[p] = v
        else:
            kinds[p] = _kind(v, p)
            vals[p] = _inputs([p], kinds, [v])[p]
    k = compiled(prog, fdef.name, kinds)
    primal, grads, fail = k.gradient(vals, seeds=seeds, tol=opts.float_tolerance,
                                     invcheck=opts.invcheck, max_steps=opts.max_steps)
    report = wrt if wrt is not None else [p for p in names if p in grads]
    for p in report:
        if p not in names:
            raise KindError(f"wrt names unknown parameter {p!r}")
        if p not in grads:
            raise KindError(f"{p!r} is an Int parameter: it has no cotangent")
    return primal, {p: grads[p] for p in report}, fail


def _cval(v):
    """A Complex argument (the caller's re/im class, complex or 0-d tensor) as complex."""
    if hasattr(v, "re") and hasattr(v, "im"):
        return complex(float(v.re), float(v.im))
    if isinstance(v, torch.Tensor):
        return complex(v.item())
    return complex(v)


def _leaf_rows(kinds, names, args):
    """[(param, flat index / "re" / "im" / None)] over the Float leaves, in
    leaf_paths order (a Complex is its re and im leaves, autodiff.py:46-47)."""
    out = []
    for p, v in zip(names, args):
        k, shp = kinds[p]
        if k in ("f", "x"):
            out.append((p, None))
        elif k == "c":
            out += [(p, "re"), (p, "im")]
        elif k == "a":
            out += [(p, i) for i in range(int(np.prod(shp)))]
    return out


def finite_difference(prog, fdef, args, h, seeds, opts):
    """Reference finite_difference (autodiff.py:270-318): central differences
    of the seeded scalar output per Float input leaf, every perturbed call of
    one leaf set run as ONE batched launch of the generated run kernel."""
    names, kinds = _call_kinds(fdef, list(args))
    k = compiled(prog, fdef.name, kinds)
    if seeds is None:
        seeds = k._default_seeds()
    base = _inputs(names, kinds, args)
    leaves = _leaf_rows(kinds, names, args)
    n = 2 * len(leaves)
    batch, steps = {}, []
    for p in names:
        kind, shp = kinds[p]
        if kind in ("f", "a", "c"):
            a = np.asarray(_cval(base[p]) if kind == "c" else base[p],
                           dtype=np.complex128 if kind == "c" else np.float64)
            batch[p] = np.broadcast_to(a, (max(n, 1),) + a.shape).copy()
        elif kind == "x":                                # raw int64 rows
            batch[p] = np.full(max(n, 1), int(base[p].raw), dtype=np.int64)
        else:
            batch[p] = base[p]
    for r, (p, i) in enumerate(leaves):
        if kinds[p][0] == "x":
            # the step is measured after Q31.32 quantization (autodiff.py:299-301)
            x = float(base[p].to_float())
            up, dn = codegen._fx_from_real(x + h), codegen._fx_from_real(x - h)
            steps.append(float(_fx_float(up) - _fx_float(dn)))
            batch[p][2 * r], batch[p][2 * r + 1] = up, dn
            continue
        if i in ("re", "im"):                            # a Complex leaf
            z = _cval(base[p])
            x = z.real if i == "re" else z.imag
            up, dn = x + h, x - h
            steps.append(up - dn)
            if i == "re":
                batch[p][2 * r], batch[p][2 * r + 1] = complex(up, z.imag), complex(dn, z.imag)
            else:
                batch[p][2 * r], batch[p][2 * r + 1] = complex(z.real, up), complex(z.real, dn)
            continue
        col = batch[p] if i is None else batch[p].reshape(n, -1)
        x = float(base[p]) if i is None else float(np.asarray(base[p]).ravel()[i])
        up, dn = x + h, x - h
        steps.append(up - dn)                            # the step actually taken
        if i is None:
            col[2 * r], col[2 * r + 1] = up, dn
        else:
            col[2 * r, i], col[2 * r + 1, i] = up, dn
    dev = torch.device("cuda", torch.cuda.current_device())
    tens = {p: (torch.as_tensor(v, device=dev) if kinds[p][0] in ("f", "a", "c", "x") else v)
            for p, v in batch.items()}
    out, fail = k.run(tens, 1, tol=opts.float_tolerance, invcheck=opts.invcheck,
                      max_steps=opts.max_steps)
    f = fail.cpu().numpy()
    if n and f.any():                                   # the reference stops at the first
        raise error_for_code(int(f[np.nonzero(f)[0][0]]), fdef.name)
    total = np.zeros(max(n, 1))
    for pname, path, seed in seeds:                      # seeded_scalar
        if pname not in names:
            raise KindError(f"seed names unknown parameter {pname!r}")
        v = out[pname].cpu().numpy().reshape(max(n, 1), -1)
        if path and path[0][0] == "field":               # Complex re / im (get_leaf)
            col = v[:, 0].real if path[0][1] == "re" else v[:, 0].imag
        elif path:
            idx = path[0][1]
            shp = kinds[pname][1]
            col = v[:, int(np.ravel_multi_index(tuple(x - 1 for x in idx), shp))]
        else:
            col = v[:, 0]
        if kinds[pname][0] == "x":                       # to_real(Fixed)
            col = _fx_float(col)
        total = total + float(seed) * np.real(col)
    grads = {}
    for p, v in zip(names, args):
        kind, shp = kinds[p]
        if kind in ("i", "ai"):
            grads[p] = None
            continue
        rows = [r for r, (q, _) in enumerate(leaves) if q == p]
        vals = [(total[2 * r] - total[2 * r + 1]) / steps[r] for r in rows]
        if kind == "c":                                  # Complex(grad re, grad im)
            grads[p] = _back(v, "c", complex(vals[0], vals[1]))
        else:
            grads[p] = float(vals[0]) if kind in ("f", "x") else \
                _back(v, "a", np.asarray(vals).reshape(shp))
    return grads
