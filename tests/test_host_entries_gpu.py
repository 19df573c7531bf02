"""The host-buffer (`_host`) forms of the run / uncall / Hessian / residual
entries (include/revgpu.h) against their device-pointer forms: identical
outputs and status codes, chunk boundaries included."""

import ctypes

import numpy as np
import pytest
import torch

import paper_2003_04617_b200 as rg
from paper_2003_04617_b200 import _native, kernels

pytestmark = pytest.mark.gpu


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def test_besselj_run_and_hess_host(cuda):
    L = _native.lib()
    rng = np.random.default_rng(21)
    n = (1 << 22) + 12345                            # two chunks, the second ragged
    z = rng.uniform(0.05, 14.0, n)
    z[::100003] = -1.0                               # RevDomainError elements
    zin = rng.normal(0, 1, n)
    cap = kernels.bessel_trip_cap(500_000_000, 3)
    for direction in (1, -1):
        out, fail, nf = np.empty(n), np.empty(n, np.uint8), ctypes.c_ulonglong()
        rc = L.rl_besselj_run_f64_host(3, _p(z), n, 1e-16, 1e-9, cap, 1, direction, _p(zin),
                                       _p(out), _p(fail), ctypes.byref(nf), 0)
        assert rc == 0
        r = rg.besselj_run(torch.as_tensor(z, device=cuda), 3,
                           out_in=torch.as_tensor(zin, device=cuda), direction=direction)
        assert np.array_equal(fail, r.fail.cpu().numpy()) and nf.value == r.n_failed > 0
        ok = fail == 0
        assert np.array_equal(out[ok], r.out.cpu().numpy()[ok])
    J, dz, d2 = np.empty(n), np.empty(n), np.empty(n)
    fail, nf = np.empty(n, np.uint8), ctypes.c_ulonglong()
    rc = L.rl_besselj_hess_f64_host(3, _p(z), n, 1e-16, 1e-9, 1.0, cap, 1, _p(J), _p(dz), _p(d2),
                                    _p(fail), ctypes.byref(nf), 0)
    assert rc == 0
    h = rg.besselj_hess(torch.as_tensor(z, device=cuda), 3)
    ok = fail == 0
    assert np.array_equal(fail, h.fail.cpu().numpy())
    for a, b in ((J, h.J), (dz, h.dJdz), (d2, h.d2Jdz2)):
        assert np.array_equal(a[ok], b.cpu().numpy()[ok])


def test_ba_residuals_and_gmm_run_host(cuda):
    import sys
    import os
    sys.path.insert(0, os.path.dirname(__file__))
    from test_ba_gpu import ba_inputs
    from test_gmm_gpu import gmm_constants, inputs
    L = _native.lib()
    cams, X, w, feats, obs = ba_inputs(np.random.default_rng(5), 30, 200, 5000)
    err, fail, nf = np.empty((5000, 3)), np.empty(5000, np.uint8), ctypes.c_ulonglong()
    c = lambda a: np.ascontiguousarray(a)  # noqa: E731
    cams, X, w, feats, obs = c(cams), c(X), c(w), c(feats), c(obs.astype(np.int32))
    rc = L.rl_ba_residuals_f64_host(30, 200, 5000, _p(cams), _p(X), _p(w), _p(feats), _p(obs),
                                    1e-9, 1, _p(err), _p(fail), ctypes.byref(nf), 0)
    assert rc == 0
    t = lambda a: torch.as_tensor(a, device=cuda)  # noqa: E731
    r = rg.ba_residuals(t(cams), t(X), t(w), t(feats), t(obs))
    assert np.array_equal(err, r.out.cpu().numpy()) and np.array_equal(fail, r.fail.cpu().numpy())
    d, K, N = 20, 5, 700
    al, me, ic, x = (np.ascontiguousarray(v) for v in inputs(np.random.default_rng(6), d, K, N))
    cst = gmm_constants(d, K, N, 1.0, 0)
    for direction in (1, -1):
        e, nf, up = ctypes.c_double(), ctypes.c_ulonglong(), ctypes.c_ulonglong()
        rc = L.rl_gmm_run_f64_host(d, K, N, _p(al), _p(me), _p(ic), _p(x), 1.0, 0, cst, 2.5,
                                   1e-9, 1, direction, ctypes.byref(e), ctypes.byref(nf),
                                   ctypes.byref(up), 0)
        assert rc == 0 and nf.value == 0
        g = rg.gmm_run(t(al), t(me), t(ic), t(x), 1.0, 0, cst, err0=2.5, direction=direction)
        assert e.value == float(g.out.item()) and up.value == int(g.counters[0].item())


def test_gmm_grad_shard_host(cuda):
    """rl_gmm_grad_shard_f64_host (bench.py's N>1 e2e path): each shard equals
    the device shard entry bit for bit, and the shards' sum the whole
    gradient to rounding."""
    import sys
    import os
    sys.path.insert(0, os.path.dirname(__file__))
    from test_gmm_gpu import gmm_constants, inputs
    L = _native.lib()
    d, K, N = 16, 6, 1001
    al, me, ic, x = (np.ascontiguousarray(v) for v in inputs(np.random.default_rng(8), d, K, N))
    cst = gmm_constants(d, K, N, 1.0, 0)
    t = lambda a: torch.as_tensor(a, device=cuda)  # noqa: E731
    nout = 1 + K + K * d + K * d * (d + 1) // 2
    total = np.zeros(nout)
    for lo, hi in ((0, 400), (400, N)):
        out, nf = np.empty(nout), ctypes.c_ulonglong()
        xs = np.ascontiguousarray(x[lo:hi])
        rc = L.rl_gmm_grad_shard_f64_host(d, K, hi - lo, N, _p(al), _p(me), _p(ic), _p(xs), 1.0,
                                          0, cst, 1e-9, 1, int(lo == 0), _p(out),
                                          ctypes.byref(nf), 0)
        assert rc == 0 and nf.value == 0
        r = kernels.gmm_grad(t(al), t(me), t(ic), t(xs), 1.0, 0, cst, N_total=N,
                             add_param_terms=(lo == 0))
        assert np.array_equal(out, r.packed.cpu().numpy())
        total += out
    whole, nf = np.empty(nout), ctypes.c_ulonglong()
    assert L.rl_gmm_grad_f64_host(d, K, N, _p(al), _p(me), _p(ic), _p(x), 1.0, 0, cst, 1e-9, 1,
                                  _p(whole), ctypes.byref(nf), 0) == 0
    assert np.allclose(total, whole, rtol=1e-12, atol=1e-9)
