"""Batched device entry points over torch CUDA tensors.

Each function launches ONE fused forward + reverse-sweep kernel of
librevgpu.so on the current torch stream (no synchronisation) and returns
device tensors.  These are the batched counterparts of the reference's
per-call `gradient` (autodiff.py:136-180): element i of every output equals
what `gradient(program, GradRequest(fname, args_i))` returns for the i-th
input, within the tolerance stated in DESIGN.md, and `fail[i]` carries the
revlang error class the reference would raise for it (include/revgpu.h).

torch is used for device memory and streams only; the arithmetic is in the
CUDA kernels.  No CPU path exists: non-CUDA inputs raise.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .errors import KindError

F64 = torch.float64
# ExecOptions.max_steps (reference interpreter.py:40) -> series-trip cap.
# The reference counts one step per statement execution (Interpreter._tick,
# interpreter.py:461-466) and raises FuelExhausted past max_steps, with a
# fresh count for the forward run and for the gradient's uncall.  For
# programs/besselj.rnl both sweeps execute exactly 31 + 6 nu + 22 T
# statements for T series trips (measured on the reference and pinned by
# tests/golden/bessel_fuel.npz), so an element exhausts the fuel iff it
# needs more than (max_steps - 31 - 6 nu) // 22 trips; -1 = even the
# prologue does not fit (every element that reaches the loop fails).
BJ_TICKS_BASE, BJ_TICKS_NU, BJ_TICKS_TRIP = 31, 6, 22


def bessel_trip_cap(max_steps, nu):
    cap = (int(max_steps) - BJ_TICKS_BASE - BJ_TICKS_NU * max(int(nu), 0)) // BJ_TICKS_TRIP
    return max(cap, -1)


def _stream_handle():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _require_cuda(name, t, dtype=F64, ndim=None, last=None):
    if not isinstance(t, torch.Tensor):
        raise KindError(f"{name} must be a torch tensor on a CUDA device")
    if not t.is_cuda:
        raise KindError(f"{name} must live on a CUDA device (no CPU path exists)")
    if t.dtype != dtype:
        raise KindError(f"{name} must be {dtype}, got {t.dtype}")
    if ndim is not None and t.dim() != ndim:
        raise KindError(f"{name} must have {ndim} dimensions, got shape {tuple(t.shape)}")
    if last is not None and t.shape[-1] != last:
        raise KindError(f"{name} must have trailing dimension {last}, got {tuple(t.shape)}")
    if t.device.index != torch.cuda.current_device():
        raise KindError(f"{name} is on {t.device} but the current device is "
                        f"cuda:{torch.cuda.current_device()} (use torch.cuda.device(...))")
    return t.contiguous()


def _check_out(name, t, like, dtype=F64, numel=None):
    """Caller-provided output buffers are written in place: they must be
    contiguous, of the right dtype and size, on the inputs' device."""
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or t.device != like.device or t.dtype != dtype:
        raise KindError(f"out tensor {name} must be a {dtype} tensor on {like.device}")
    if not t.is_contiguous():
        raise KindError(f"out tensor {name} must be contiguous")
    if numel is not None and t.numel() != numel:
        raise KindError(f"out tensor {name} must have {numel} elements, got {t.numel()}")
    return t


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


@dataclass
class BesselResult:
    J: torch.Tensor          # primal out! per element
    dJdz: torch.Tensor       # z cotangent (out!.g = seed)
    fail: torch.Tensor       # uint8 status per element (0 = ok)
    counters: torch.Tensor   # int64[2] device: [sum of series trips, failed elements]

    @property
    def sum_trips(self):
        return int(self.counters[0].item())

    @property
    def n_failed(self):
        return int(self.counters[1].item())


def besselj_grad(z, nu=2, *, seed=1.0, thr=1e-16, tol=1e-9, invcheck=True,
                 max_steps=500_000_000, out=None, counters=None):
    """J_nu(z) and dJ/dz for every element of z (CUDA float64) in one kernel.

    Batched `gradient(load_example("besselj"), GradRequest("besselj",
    [0.0, nu, z_i]))`.  `out` = (J, dJdz, fail) preallocated tensors, and
    `counters` an int64[2] device tensor accumulated in place (not reset),
    let a caller avoid allocation (e.g. under CUDA-graph capture)."""
    z = _require_cuda("z", z)
    n = z.numel()
    if out is None:
        J = torch.empty_like(z)
        dz = torch.empty_like(z)
        fail = torch.empty(z.shape, dtype=torch.uint8, device=z.device)
    else:
        J, dz, fail = (_check_out("J", out[0], z, numel=n), _check_out("dJdz", out[1], z, numel=n),
                       _check_out("fail", out[2], z, torch.uint8, n))
    if counters is None:
        counters = torch.zeros(2, dtype=torch.int64, device=z.device)
    counters = _check_out("counters", counters, z, torch.int64, 2)
    L = _native.lib()
    rc = L.rl_besselj_grad_f64(int(nu), _ptr(z), n, float(thr), float(tol), float(seed),
                               bessel_trip_cap(max_steps, nu), int(bool(invcheck)),
                               _ptr(J), _ptr(dz), _ptr(fail), _ptr(counters), _stream_handle())
    _native.check(rc, "rl_besselj_grad_f64")
    return BesselResult(J, dz, fail, counters)


@dataclass
class BesselHessResult:
    J: torch.Tensor          # primal (bit-identical to besselj_grad's)
    dJdz: torch.Tensor       # first derivative (bit-identical to besselj_grad's)
    d2Jdz2: torch.Tensor     # H[z, z] of autodiff.hessian
    fail: torch.Tensor
    counters: torch.Tensor

    @property
    def sum_trips(self):
        return int(self.counters[0].item())


def besselj_hess(z, nu=2, *, seed=1.0, thr=1e-16, tol=1e-9, invcheck=True,
                 max_steps=500_000_000, counters=None):
    """Batched forward-over-reverse Hessian: `hessian(load_example("besselj"),
    "besselj", [0.0, nu, z_i])[z, z]` (reference autodiff.py:216-257) for every
    element, with J and dJ/dz, in one kernel (Dual-number sweeps)."""
    z = _require_cuda("z", z)
    n = z.numel()
    J, dz, d2 = torch.empty_like(z), torch.empty_like(z), torch.empty_like(z)
    fail = torch.empty(z.shape, dtype=torch.uint8, device=z.device)
    if counters is None:
        counters = torch.zeros(2, dtype=torch.int64, device=z.device)
    L = _native.lib()
    rc = L.rl_besselj_hess_f64(int(nu), _ptr(z), n, float(thr), float(tol), float(seed),
                               bessel_trip_cap(max_steps, nu), int(bool(invcheck)),
                               _ptr(J), _ptr(dz), _ptr(d2), _ptr(fail), _ptr(counters),
                               _stream_handle())
    _native.check(rc, "rl_besselj_hess_f64")
    return BesselHessResult(J, dz, d2, fail, counters)


def besselj_grad_host(z, nu=2, *, seed=1.0, thr=1e-16, tol=1e-9, invcheck=True,
                      max_steps=500_000_000, device=None, out=None):
    """Host-buffer entry (numpy float64 or CPU tensor in, numpy out): the
    C-ABI `_host` call pipelines the copies with the kernel.  Synchronous."""
    import numpy as np

    zh = np.ascontiguousarray(z.numpy() if isinstance(z, torch.Tensor) else z, dtype=np.float64)
    n = zh.size
    if out is None:
        J = np.empty(n)
        dz = np.empty(n)
        fail = np.empty(n, np.uint8)
    else:
        J, dz, fail = out
    trips = ctypes.c_ulonglong(0)
    nfail = ctypes.c_ulonglong(0)
    dev = torch.cuda.current_device() if device is None else int(device)
    L = _native.lib()
    rc = L.rl_besselj_grad_f64_host(int(nu), zh.ctypes.data, n, float(thr), float(tol),
                                    float(seed), bessel_trip_cap(max_steps, nu),
                                    int(bool(invcheck)), J.ctypes.data, dz.ctypes.data,
                                    fail.ctypes.data, ctypes.byref(trips), ctypes.byref(nfail),
                                    dev)
    _native.check(rc, "rl_besselj_grad_f64_host")
    return J, dz, fail, int(trips.value), int(nfail.value)


@dataclass
class BAResult:
    J: torch.Tensor          # (p, 31): [de1/d(cam,X,w), de2/d(cam,X,w), d(1-w^2)/dw]
    err: torch.Tensor        # (p, 3) residuals [e1, e2, 1 - w^2] or None
    Jfeat: torch.Tensor      # (p, 4) feature columns or None
    fail: torch.Tensor
    counters: torch.Tensor

    @property
    def n_failed(self):
        return int(self.counters[1].item())


def ba_jacobian(cams, X, w, feats, obs, *, tol=1e-9, invcheck=True, want_err=True,
                want_feat=False, out=None, counters=None):
    """ADBench BA reprojection Jacobian blocks for every observation.

    Batched 2x `gradient(load_example("ba_proj"), GradRequest("ba_proj",
    [0, 0, cams[c_i], X[p_i], w_i, f_i1, f_i2], seeds=[e1!|e2!], wrt=[cam, X, w]))`
    plus `gradient(.., "ba_weight", [0, w_i])`; obs[i] = (c_i, p_i), 0-based."""
    cams = _require_cuda("cams", cams, ndim=2, last=11)
    X = _require_cuda("X", X, ndim=2, last=3)
    w = _require_cuda("w", w, ndim=1)
    feats = _require_cuda("feats", feats, ndim=2, last=2)
    obs = _require_cuda("obs", obs, dtype=torch.int32, ndim=2, last=2)
    p = w.shape[0]
    if feats.shape[0] != p or obs.shape[0] != p:
        raise KindError("w, feats and obs must have the same number of observations")
    dev = w.device
    if out is None:
        J = torch.empty((p, 31), dtype=F64, device=dev)
        err = torch.empty((p, 3), dtype=F64, device=dev) if want_err else None
        Jf = torch.empty((p, 4), dtype=F64, device=dev) if want_feat else None
        fail = torch.empty(p, dtype=torch.uint8, device=dev)
    else:
        J, err, Jf, fail = (_check_out("J", out[0], w, numel=31 * p),
                            _check_out("err", out[1], w, numel=3 * p),
                            _check_out("Jfeat", out[2], w, numel=4 * p),
                            _check_out("fail", out[3], w, torch.uint8, p))
    if counters is None:
        counters = torch.zeros(2, dtype=torch.int64, device=dev)
    counters = _check_out("counters", counters, w, torch.int64, 2)
    L = _native.lib()
    rc = L.rl_ba_jac_f64(cams.shape[0], X.shape[0], p, _ptr(cams), _ptr(X), _ptr(w), _ptr(feats),
                         _ptr(obs), float(tol), int(bool(invcheck)), _ptr(err), _ptr(J), _ptr(Jf),
                         _ptr(fail), _ptr(counters), _stream_handle())
    _native.check(rc, "rl_ba_jac_f64")
    return BAResult(J, err, Jf, fail, counters)


@dataclass
class GMMResult:
    err: torch.Tensor        # () objective
    g_alphas: torch.Tensor   # (K,)
    g_means: torch.Tensor    # (K, d)
    g_icf: torch.Tensor      # (K, d(d+1)/2)
    fail: torch.Tensor       # (N,) per point
    counters: torch.Tensor
    packed: torch.Tensor     # the contiguous [err, g_alphas, g_means, g_icf] vector
    resid: torch.Tensor = None         # () err! after the gradient sweep (gmm_gradient)
    restore_code: torch.Tensor = None  # () int32: 0, or 5 = RevError (autodiff.py:169-172)

    @property
    def n_failed(self):
        return int(self.counters[1].item())


GMM_MAX_D = 128      # widest tile of the hand-written GMM kernels (gmm.cu, dp_of)


def gmm_packed_size(d, K):
    return 1 + K + K * d + K * d * (d + 1) // 2


def unpack_gmm(packed, d, K, fail=None, counters=None):
    P = d * (d + 1) // 2
    o = 1
    ga = packed[o:o + K]
    o += K
    gm = packed[o:o + K * d].view(K, d)
    o += K * d
    gi = packed[o:o + K * P].view(K, P)
    return GMMResult(packed[0], ga, gm, gi, fail, counters, packed)


def gmm_grad(alphas, means, icf, x, gamma=1.0, m=0, cst=0.0, *, N_total=None,
             add_param_terms=True, tol=1e-9, invcheck=True, workspace=None, counters=None):
    """ADBench GMM objective and its gradient w.r.t. (alphas, means, icf).

    `gradient(load_example("gmm"), GradRequest("gmm", [0.0, alphas, means,
    icf, x, zeros.., gamma, m, cst], wrt=["alphas","means","icf"]))` with the
    points x on this device.  For a data-parallel shard pass
    add_param_terms=(rank == 0) and N_total = the global point count, then
    sum `result.packed` across ranks (see parallel.gmm_grad_distributed)."""
    alphas = _require_cuda("alphas", alphas, ndim=1)
    means = _require_cuda("means", means, ndim=2)
    K, d = means.shape
    icf = _require_cuda("icf", icf, ndim=2, last=d * (d + 1) // 2)
    x = _require_cuda("x", x, ndim=2, last=d)
    if alphas.shape[0] != K or icf.shape[0] != K:
        raise KindError("alphas, means and icf must agree on K")
    N = x.shape[0]
    dev = x.device
    L = _native.lib()
    wsb = L.rl_gmm_workspace_bytes(d, K, N)
    if workspace is not None:
        _check_out("workspace", workspace, x, torch.uint8)
    if workspace is None or workspace.numel() < wsb:
        workspace = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    packed = torch.empty(gmm_packed_size(d, K), dtype=F64, device=dev)
    fail = torch.empty(N, dtype=torch.uint8, device=dev)
    if counters is None:
        counters = torch.zeros(2, dtype=torch.int64, device=dev)
    counters = _check_out("counters", counters, x, torch.int64, 2)
    rc = L.rl_gmm_grad_f64(d, K, N, int(N if N_total is None else N_total), _ptr(alphas),
                           _ptr(means), _ptr(icf), _ptr(x), float(gamma), int(m), float(cst),
                           float(tol), int(bool(invcheck)), int(bool(add_param_terms)),
                           _ptr(packed), _ptr(fail), _ptr(counters), _ptr(workspace),
                           workspace.numel(), _stream_handle())
    _native.check(rc, "rl_gmm_grad_f64")
    return unpack_gmm(packed, d, K, fail, counters)


def gmm_statement_count(d, K, N, U, A):
    """Statements one sweep of programs/gmm.rnl executes in the reference
    (its fuel unit, interpreter.py:461-466): rl_gmm_statement_count."""
    return int(_native.lib().rl_gmm_statement_count(int(d), int(K), int(N), int(U), int(A)))


def gmm_alpha_updates(alphas):
    """Argmax record steps of the alphas' reversible logsumexp (gmm.rnl): how
    often a later alpha beats the running max."""
    a = np.asarray(alphas.cpu() if isinstance(alphas, torch.Tensor) else alphas, np.float64)
    n, best = 0, 0
    for k in range(1, a.shape[0]):
        if a[k] > a[best]:
            best, n = k, n + 1
    return n


def _gmm_args(alphas, means, icf, x):
    alphas = _require_cuda("alphas", alphas, ndim=1)
    means = _require_cuda("means", means, ndim=2)
    K, d = means.shape
    icf = _require_cuda("icf", icf, ndim=2, last=d * (d + 1) // 2)
    x = _require_cuda("x", x, ndim=2, last=d)
    if alphas.shape[0] != K or icf.shape[0] != K:
        raise KindError("alphas, means and icf must agree on K")
    return alphas, means, icf, x, K, d


def _gmm_workspace(L, d, K, N, workspace, x):
    wsb = L.rl_gmm_workspace_bytes(d, K, N)
    if workspace is not None:
        _check_out("workspace", workspace, x, torch.uint8)
    if workspace is None or workspace.numel() < wsb:
        workspace = torch.empty(max(wsb, 1), dtype=torch.uint8, device=x.device)
    return workspace


def gmm_gradient(alphas, means, icf, x, gamma=1.0, m=0, cst=0.0, *, err0=0.0, tol=1e-9,
                 invcheck=True, workspace=None, counters=None):
    """The whole reference `gradient(p, GradRequest("gmm", [err0, alphas,
    means, icf, x, zeros.., gamma, m, cst]))` on one device
    (rl_gmm_gradient_f64): err is err! accumulated in the program's order
    from err0 (the reference's primal output), `resid` is err! after the
    gradient sweep and `restore_code` the verdict of the reference's
    primal-restoration check (autodiff.py:169-172): 5 (RevError) when
    |resid - err0| > tol."""
    alphas, means, icf, x, K, d = _gmm_args(alphas, means, icf, x)
    N = x.shape[0]
    dev = x.device
    L = _native.lib()
    workspace = _gmm_workspace(L, d, K, N, workspace, x)
    packed = torch.empty(gmm_packed_size(d, K), dtype=F64, device=dev)
    fail = torch.empty(N, dtype=torch.uint8, device=dev)
    resid = torch.empty((), dtype=F64, device=dev)
    code = torch.empty((), dtype=torch.int32, device=dev)
    if counters is None:
        counters = torch.zeros(2, dtype=torch.int64, device=dev)
    counters = _check_out("counters", counters, x, torch.int64, 2)
    rc = L.rl_gmm_gradient_f64(d, K, N, _ptr(alphas), _ptr(means), _ptr(icf), _ptr(x),
                               float(gamma), int(m), float(cst), float(err0), float(tol),
                               int(bool(invcheck)), _ptr(packed), _ptr(resid), _ptr(code),
                               _ptr(fail), _ptr(counters), _ptr(workspace), workspace.numel(),
                               _stream_handle())
    _native.check(rc, "rl_gmm_gradient_f64")
    r = unpack_gmm(packed, d, K, fail, counters)
    r.resid, r.restore_code = resid, code
    return r


def gmm_run(alphas, means, icf, x, gamma=1.0, m=0, cst=0.0, *, err0=0.0, direction=1, tol=1e-9,
            invcheck=True, workspace=None, counters=None):
    """Reference `run(p, "gmm", [err0, ...])` (direction +1,
    interpreter.py:1021) or `uncall` (-1, :1026) on one device
    (rl_gmm_run_f64): err! after the program (its inverse), accumulated from
    err0 in that program's order."""
    alphas, means, icf, x, K, d = _gmm_args(alphas, means, icf, x)
    N = x.shape[0]
    L = _native.lib()
    workspace = _gmm_workspace(L, d, K, N, workspace, x)
    err = torch.empty(1, dtype=F64, device=x.device)
    fail = torch.empty(N, dtype=torch.uint8, device=x.device)
    if counters is None:
        counters = torch.zeros(2, dtype=torch.int64, device=x.device)
    rc = L.rl_gmm_run_f64(d, K, N, _ptr(alphas), _ptr(means), _ptr(icf), _ptr(x), float(gamma),
                          int(m), float(cst), float(err0), float(tol), int(bool(invcheck)),
                          int(direction), _ptr(err), _ptr(fail), _ptr(counters), _ptr(workspace),
                          workspace.numel(), _stream_handle())
    _native.check(rc, "rl_gmm_run_f64")
    return RunResult(err[0], fail, counters)


def seq_sum(t, e0=0.0, mark=None, *, force_serial=False):
    """e_{j+1} = fl(e_j + t_j) over the device array t from e0, bit-exactly
    the sequential binary64 chain (rl_seq_sum_f64).  Returns (e_mark, e_M,
    verified) as Python values; `verified` is True when the parallel path
    verified (else the sequential fallback produced the result)."""
    t = _require_cuda("t", t, ndim=1)
    M = t.shape[0]
    mark = M if mark is None else int(mark)
    out2 = torch.empty(2, dtype=F64, device=t.device)
    ver = torch.zeros((), dtype=torch.int32, device=t.device)
    rc = _native.lib().rl_seq_sum_f64(_ptr(t), M, float(e0), mark, int(bool(force_serial)),
                                      _ptr(out2), _ptr(ver), _stream_handle())
    _native.check(rc, "rl_seq_sum_f64")
    o = out2.cpu()
    return float(o[0]), float(o[1]), bool(ver.item())


# ---------------------------------------------------------------------------
# run / uncall / objective-only entries (primal sweeps with every check)
# ---------------------------------------------------------------------------

@dataclass
class RunResult:
    out: torch.Tensor        # updated output argument per element
    fail: torch.Tensor
    counters: torch.Tensor

    @property
    def n_failed(self):
        return int(self.counters[1].item())


def besselj_run(z, nu=2, *, out_in=None, direction=1, thr=1e-16, tol=1e-9, invcheck=True,
                max_steps=500_000_000, counters=None):
    """Batched `run(p, "besselj", [out_in_i, nu, z_i])` (direction +1,
    interpreter.py:1021) or `uncall(...)` (direction -1, :1026):
    out = out_in +/- J_nu(z), with every check of the primal sweeps.  Also the
    objective-only ("-O") timing of the Bessel program."""
    z = _require_cuda("z", z)
    if out_in is not None:
        out_in = _require_cuda("out_in", out_in)
        if out_in.shape != z.shape:
            raise KindError("out_in must have the shape of z")
    out = torch.empty_like(z)
    fail = torch.empty(z.shape, dtype=torch.uint8, device=z.device)
    if counters is None:
        counters = torch.zeros(2, dtype=torch.int64, device=z.device)
    rc = _native.lib().rl_besselj_run_f64(
        int(nu), _ptr(z), z.numel(), float(thr), float(tol),
        bessel_trip_cap(max_steps, nu), int(bool(invcheck)), int(direction),
        _ptr(out_in), _ptr(out), _ptr(fail), _ptr(counters), _stream_handle())
    _native.check(rc, "rl_besselj_run_f64")
    return RunResult(out, fail, counters)


def ba_residuals(cams, X, w, feats, obs, *, tol=1e-9, invcheck=True, counters=None):
    """Batched run of ba_proj / ba_weight on zero outputs: (p, 3) residuals
    [e1, e2, 1 - w^2] — the BA objective-only kernel."""
    cams = _require_cuda("cams", cams, ndim=2, last=11)
    X = _require_cuda("X", X, ndim=2, last=3)
    w = _require_cuda("w", w, ndim=1)
    feats = _require_cuda("feats", feats, ndim=2, last=2)
    obs = _require_cuda("obs", obs, dtype=torch.int32, ndim=2, last=2)
    p = w.shape[0]
    err = torch.empty((p, 3), dtype=F64, device=w.device)
    fail = torch.empty(p, dtype=torch.uint8, device=w.device)
    if counters is None:
        counters = torch.zeros(2, dtype=torch.int64, device=w.device)
    rc = _native.lib().rl_ba_residuals_f64(
        cams.shape[0], X.shape[0], p, _ptr(cams), _ptr(X), _ptr(w), _ptr(feats), _ptr(obs),
        float(tol), int(bool(invcheck)), _ptr(err), _ptr(fail), _ptr(counters), _stream_handle())
    _native.check(rc, "rl_ba_residuals_f64")
    return RunResult(err, fail, counters)


def gmm_objective(alphas, means, icf, x, gamma=1.0, m=0, cst=0.0, *, N_total=None,
                  add_param_terms=True, tol=1e-9, invcheck=True, workspace=None, counters=None):
    """Batched run of gmm: the objective only ("-O"), a 0-d tensor."""
    alphas = _require_cuda("alphas", alphas, ndim=1)
    means = _require_cuda("means", means, ndim=2)
    K, d = means.shape
    icf = _require_cuda("icf", icf, ndim=2, last=d * (d + 1) // 2)
    x = _require_cuda("x", x, ndim=2, last=d)
    N = x.shape[0]
    L = _native.lib()
    wsb = L.rl_gmm_workspace_bytes(d, K, N)
    if workspace is not None:
        _check_out("workspace", workspace, x, torch.uint8)
    if workspace is None or workspace.numel() < wsb:
        workspace = torch.empty(max(wsb, 1), dtype=torch.uint8, device=x.device)
    err = torch.empty(1, dtype=F64, device=x.device)
    fail = torch.empty(N, dtype=torch.uint8, device=x.device)
    if counters is None:
        counters = torch.zeros(2, dtype=torch.int64, device=x.device)
    rc = L.rl_gmm_objective_f64(d, K, N, int(N if N_total is None else N_total), _ptr(alphas),
                                _ptr(means), _ptr(icf), _ptr(x), float(gamma), int(m), float(cst),
                                float(tol), int(bool(invcheck)), int(bool(add_param_terms)),
                                _ptr(err), _ptr(fail), _ptr(counters), _ptr(workspace),
                                workspace.numel(), _stream_handle())
    _native.check(rc, "rl_gmm_objective_f64")
    return RunResult(err[0], fail, counters)


@dataclass
class BACsr:
    """The BA Jacobian in ADBench's BASparseMat layout (CSR, int32 indices):
    nrows = 3P (2 reprojection rows per observation, then one weight row per
    observation), ncols = 11 n_cams + 3 n_pts + P, nnz = 31P.  For a shard
    (obs_offset > 0 or n_obs_total > n_obs) the arrays are the shard's two
    pieces of the global arrays concatenated (include/revgpu.h)."""
    rows: object            # int32 [3 n_obs + 1] or None (values only)
    cols: object            # int32 [31 n_obs]    or None
    vals: object            # float64 [31 n_obs]
    fail: object            # uint8 [n_obs]
    shape: tuple            # (nrows, ncols) of the global matrix
    counters: object = None  # device counters, or the host call's failure count
    err: object = None      # (n_obs, 3) residuals when want_err

    def to_scipy(self):
        """scipy.sparse.csr_matrix of a whole-problem result."""
        import numpy as np
        import scipy.sparse as sp

        f = (lambda t: t.cpu().numpy()) if isinstance(self.vals, torch.Tensor) else np.asarray
        return sp.csr_matrix((f(self.vals), f(self.cols), f(self.rows)), shape=self.shape)


def _ba_shape(n_cams, n_pts, P):
    return (3 * P, 11 * n_cams + 3 * n_pts + P)


def ba_jacobian_csr(cams, X, w, feats, obs, *, obs_offset=0, n_obs_total=None, pattern=True,
                    tol=1e-9, invcheck=True, want_err=False, out=None, counters=None):
    """ba_jacobian stored as ADBench's BASparseMat (CSR).  `pattern=False`
    skips the row pointers / column indices (they depend on obs only)."""
    cams = _require_cuda("cams", cams, ndim=2, last=11)
    X = _require_cuda("X", X, ndim=2, last=3)
    w = _require_cuda("w", w, ndim=1)
    feats = _require_cuda("feats", feats, ndim=2, last=2)
    obs = _require_cuda("obs", obs, dtype=torch.int32, ndim=2, last=2)
    p = w.shape[0]
    if feats.shape[0] != p or obs.shape[0] != p:
        raise KindError("w, feats and obs must have the same number of observations")
    P = p + obs_offset if n_obs_total is None else int(n_obs_total)
    dev = w.device
    if out is None:
        vals = torch.empty(31 * p, dtype=F64, device=dev)
        rows = torch.empty(3 * p + 1, dtype=torch.int32, device=dev) if pattern else None
        cols = torch.empty(31 * p, dtype=torch.int32, device=dev) if pattern else None
        fail = torch.empty(p, dtype=torch.uint8, device=dev)
        err = torch.empty((p, 3), dtype=F64, device=dev) if want_err else None
    else:
        rows, cols, vals, fail, err = (
            _check_out("rows", out[0], w, torch.int32, 3 * p + 1),
            _check_out("cols", out[1], w, torch.int32, 31 * p),
            _check_out("vals", out[2], w, numel=31 * p),
            _check_out("fail", out[3], w, torch.uint8, p),
            _check_out("err", out[4], w, numel=3 * p))
        if (rows is None) != (cols is None):
            raise KindError("rows and cols are both given or both None")
    if counters is None:
        counters = torch.zeros(2, dtype=torch.int64, device=dev)
    L = _native.lib()
    rc = L.rl_ba_jac_csr_f64(cams.shape[0], X.shape[0], p, int(obs_offset), P, _ptr(cams), _ptr(X),
                             _ptr(w), _ptr(feats), _ptr(obs), float(tol), int(bool(invcheck)),
                             _ptr(err), _ptr(rows), _ptr(cols), _ptr(vals), _ptr(fail),
                             _ptr(counters), _stream_handle())
    _native.check(rc, "rl_ba_jac_csr_f64")
    return BACsr(rows, cols, vals, fail, _ba_shape(cams.shape[0], X.shape[0], P), counters, err)


def ba_jacobian_csr_host(cams, X, w, feats, obs, *, pattern=True, tol=1e-9, invcheck=True,
                         device=None):
    """Host-buffer entry (numpy in, numpy out) of ba_jacobian_csr for a whole
    problem: the C-ABI `_host` call pipelines the copies with the kernel."""
    import numpy as np

    c = lambda a, t: np.ascontiguousarray(a.numpy() if isinstance(a, torch.Tensor) else a,  # noqa
                                          dtype=t)
    cams, X, w, feats = (c(a, np.float64) for a in (cams, X, w, feats))
    obs = c(obs, np.int32)
    p = w.size
    vals = np.empty(31 * p)
    rows = np.empty(3 * p + 1, np.int32) if pattern else None
    cols = np.empty(31 * p, np.int32) if pattern else None
    fail = np.empty(p, np.uint8)
    nfail = ctypes.c_ulonglong(0)
    dev = torch.cuda.current_device() if device is None else int(device)
    L = _native.lib()
    rc = L.rl_ba_jac_csr_f64_host(cams.shape[0], X.shape[0], p, cams.ctypes.data, X.ctypes.data,
                                  w.ctypes.data, feats.ctypes.data, obs.ctypes.data, float(tol),
                                  int(bool(invcheck)), None if rows is None else rows.ctypes.data,
                                  None if cols is None else cols.ctypes.data, vals.ctypes.data,
                                  fail.ctypes.data, ctypes.byref(nfail), dev)
    _native.check(rc, "rl_ba_jac_csr_f64_host")
    return BACsr(rows, cols, vals, fail, _ba_shape(cams.shape[0], X.shape[0], p), int(nfail.value))
