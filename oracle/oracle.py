"""ctypes front end of the C oracle (oracle/revoracle.c) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this module.  The product package
(paper_2003_04617_b200) never does: it has no CPU path.

Each function restates `revlang.gradient` (reference autodiff.py:136-180)
for one benchmark program; see revoracle.c for the statement-level
citations.  The oracle is pinned bit-for-bit against golden vectors that
the reference interpreter itself produced (tests/golden, made by
oracle/gen_golden.py).
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_u8_p = ctypes.POINTER(ctypes.c_uint8)
_c_i32_p = ctypes.POINTER(ctypes.c_int32)
_lib = None


def build(force=False):
    """Compile revoracle.c with gcc (no contraction, no fast-math)."""
    src = os.path.join(HERE, "revoracle.c")
    if not force and os.path.exists(LIB_PATH) and \
            os.path.getmtime(LIB_PATH) >= os.path.getmtime(src):
        return LIB_PATH
    subprocess.check_call(["make", "-s", "-C", HERE])
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        L.orc_besselj_grad.restype = ctypes.c_int
        L.orc_besselj_grad.argtypes = [
            ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
            ctypes.c_double, ctypes.c_long, ctypes.c_int, _c_double_p, _c_double_p,
            ctypes.POINTER(ctypes.c_long)]
        L.orc_besselj_grad_batch.restype = ctypes.c_long
        L.orc_besselj_grad_batch.argtypes = [
            ctypes.c_int, _c_double_p, ctypes.c_long, ctypes.c_double, ctypes.c_double,
            ctypes.c_double, ctypes.c_long, ctypes.c_int, _c_double_p, _c_double_p, _c_u8_p]
        L.orc_besselj_hess_batch.restype = ctypes.c_long
        L.orc_besselj_hess_batch.argtypes = [
            ctypes.c_int, _c_double_p, ctypes.c_long, ctypes.c_double, ctypes.c_double,
            ctypes.c_double, ctypes.c_long, ctypes.c_int, _c_double_p, _c_double_p, _c_double_p,
            _c_u8_p]
        L.orc_ba_obs.restype = ctypes.c_int
        L.orc_ba_obs.argtypes = [_c_double_p, _c_double_p, ctypes.c_double, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                 _c_double_p, _c_double_p]
        L.orc_ba_jac_batch.restype = ctypes.c_long
        L.orc_ba_jac_batch.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_long, _c_double_p, _c_double_p, _c_double_p,
            _c_double_p, _c_i32_p, ctypes.c_double, ctypes.c_int, _c_double_p, _c_double_p,
            _c_u8_p]
        L.orc_gmm_grad.restype = ctypes.c_int
        L.orc_gmm_grad.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_double_p, _c_double_p, _c_double_p,
            _c_double_p, ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.c_double,
            ctypes.c_int, _c_double_p, _c_double_p, _c_double_p, _c_double_p]
        L.orc_gmm_grad_ex.restype = ctypes.c_int
        L.orc_gmm_grad_ex.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_double_p, _c_double_p, _c_double_p,
            _c_double_p, ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.c_double,
            ctypes.c_double, ctypes.c_int, ctypes.c_int, _c_double_p, _c_double_p, _c_double_p,
            _c_double_p, _c_double_p]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(_c_double_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# status codes (include/revgpu.h) -> reference exception class names
ERROR_NAMES = {0: "", 1: "PostconditionMismatch", 2: "DirtyAncilla", 3: "RevDomainError",
               4: "LoopIteratorMutated", 5: "RevError", 6: "FuelExhausted", 7: "KindError",
               8: "IndexOutOfBounds", 9: "OverflowError", 10: "AliasedArguments",
               11: "AssertFailed"}


def besselj_grad(nu, z, thr=1e-16, tol=1e-9, seed=1.0, max_trips=10**8, invcheck=True):
    """Batch over z (each element independent): returns J, dJdz, fail, sum_trips."""
    z = _f64(np.atleast_1d(z))
    n = z.size
    J = np.empty(n)
    dz = np.empty(n)
    fail = np.zeros(n, np.uint8)
    total = lib().orc_besselj_grad_batch(
        int(nu), _dp(z), n, thr, tol, seed, int(max_trips), int(bool(invcheck)), _dp(J),
        _dp(dz), fail.ctypes.data_as(_c_u8_p))
    return J, dz, fail, int(total)


def besselj_hess(nu, z, thr=1e-16, tol=1e-9, seed=1.0, max_trips=10**8, invcheck=True):
    """Forward-over-reverse second derivative (autodiff.hessian's H[z, z]) per
    z: returns J, dJdz, d2Jdz2, fail, sum_trips."""
    z = _f64(np.atleast_1d(z))
    n = z.size
    J, dz, d2 = np.empty(n), np.empty(n), np.empty(n)
    fail = np.zeros(n, np.uint8)
    total = lib().orc_besselj_hess_batch(
        int(nu), _dp(z), n, thr, tol, seed, int(max_trips), int(bool(invcheck)), _dp(J),
        _dp(dz), _dp(d2), fail.ctypes.data_as(_c_u8_p))
    return J, dz, d2, fail, int(total)


def ba_jac(cams, X, w, feats, obs, tol=1e-9, invcheck=True):
    """Per-observation Jacobian rows: J (p, 31), err (p, 3), fail (p,)."""
    cams, X, w, feats = _f64(cams), _f64(X), _f64(w), _f64(feats)
    obs = np.ascontiguousarray(obs, dtype=np.int32)
    p = w.size
    J = np.empty((p, 31))
    err = np.empty((p, 3))
    fail = np.zeros(p, np.uint8)
    lib().orc_ba_jac_batch(cams.shape[0], X.shape[0], p, _dp(cams), _dp(X), _dp(w),
                           _dp(feats), obs.ctypes.data_as(_c_i32_p), tol, int(bool(invcheck)),
                           _dp(err), _dp(J), fail.ctypes.data_as(_c_u8_p))
    return J, err, fail


def gmm_grad(alphas, means, icf, x, gamma, m, cst, tol=1e-9, invcheck=True):
    """Returns (rc, err, g_alphas, g_means, g_icf)."""
    alphas, means, icf, x = _f64(alphas), _f64(means), _f64(icf), _f64(x)
    K, d = means.shape
    N = x.shape[0]
    err = ctypes.c_double(np.nan)
    ga = np.zeros(K)
    gm = np.zeros((K, d))
    gi = np.zeros(icf.shape)
    rc = lib().orc_gmm_grad(d, K, N, _dp(alphas), _dp(means), _dp(icf), _dp(x), float(gamma),
                            int(m), float(cst), tol, int(bool(invcheck)), ctypes.byref(err),
                            _dp(ga), _dp(gm), _dp(gi))
    return rc, err.value, ga, gm, gi


def gmm_grad_ex(alphas, means, icf, x, gamma, m, cst, err0=0.0, tol=1e-9, invcheck=True,
                fresh=False):
    """gradient with err! = err0 on entry: returns (rc, err, resid, g_alphas,
    g_means, g_icf); resid = err! after the gradient sweep (what the
    reference's restoration check compares with err0, autodiff.py:169-172),
    reported whether or not that check passes (rc 5 = RevError).
    fresh=True is NOT the reference: scratch zeroed per (point, component),
    the device's semantics, to pin the device's verdict."""
    alphas, means, icf, x = _f64(alphas), _f64(means), _f64(icf), _f64(x)
    K, d = means.shape
    N = x.shape[0]
    err = ctypes.c_double(np.nan)
    resid = ctypes.c_double(np.nan)
    ga = np.zeros(K)
    gm = np.zeros((K, d))
    gi = np.zeros(icf.shape)
    rc = lib().orc_gmm_grad_ex(d, K, N, _dp(alphas), _dp(means), _dp(icf), _dp(x),
                               float(gamma), int(m), float(cst), float(err0), tol,
                               int(bool(invcheck)), int(bool(fresh)), ctypes.byref(err),
                               ctypes.byref(resid),
                               _dp(ga), _dp(gm), _dp(gi))
    return rc, err.value, resid.value, ga, gm, gi


def ba_sparse(n_cams, n_pts, obs, J31):
    """ADBench's BASparseMat built from per-observation Jacobian rows —
    TEST INFRASTRUCTURE (the checker of rl_ba_jac_csr_f64).

    Restates ADBench (github.com/microsoft/ADBench, src/cpp/shared/ba.h/.cpp
    `BASparseMat`; not part of /root/reference, which stops at the dense
    per-observation gradients): the constructor pushes rows = [0];
    `insert_reproj_err_block(i, cam, pt, J)` with J the column-major 2x15
    block (J[2*col + row]) appends two rows of 15 — 11 camera columns
    11*cam + k, 3 point columns 11*n + 3*pt + k, the weight column
    11*n + 3*m + i — for every observation in order; then
    `insert_w_err_block(i, w_d)` appends one row per observation with the
    single column 11*n + 3*m + i.  Plain loops on purpose: the kernel's
    indexing is checked against this, not against a vectorised copy of
    itself.  Layout unpinned against ADBench files (none are available
    here); values are pinned through the reference goldens of ba_jac."""
    obs = np.asarray(obs)
    p = obs.shape[0]
    rows, cols, vals = [0], [], []
    for i in range(p):
        cam, pt = int(obs[i, 0]), int(obs[i, 1])
        # our row: [de1/dcam(11) de1/dX(3) de1/dw | de2/dcam de2/dX de2/dw | dwerr/dw]
        Jcm = [0.0] * 30
        for col in range(15):
            Jcm[2 * col] = J31[i, col]
            Jcm[2 * col + 1] = J31[i, 15 + col]
        rows.append(rows[-1] + 15)
        rows.append(rows[-1] + 15)
        for r in range(2):
            for k in range(11):
                cols.append(11 * cam + k)
                vals.append(Jcm[2 * k + r])
            for k in range(3):
                cols.append(11 * n_cams + 3 * pt + k)
                vals.append(Jcm[22 + 2 * k + r])
            cols.append(11 * n_cams + 3 * n_pts + i)
            vals.append(Jcm[28 + r])
    for i in range(p):
        rows.append(rows[-1] + 1)
        cols.append(11 * n_cams + 3 * n_pts + i)
        vals.append(J31[i, 30])
    return (np.array(rows, np.int32), np.array(cols, np.int32), np.array(vals, np.float64),
            (3 * p, 11 * n_cams + 3 * n_pts + p))
