"""Edge cases across the newer entry points: empty batches, extreme orders
(the careful exp path: underflowing first terms), tiny/huge z, and the
shard/empty conventions of the CSR layout."""

import os

import numpy as np
import pytest
import torch

import paper_2003_04617_b200 as rg
from oracle import ERROR_NAMES

pytestmark = pytest.mark.gpu


def test_empty_batches(cuda):
    z = torch.zeros(0, dtype=torch.float64, device=cuda)
    assert rg.besselj_run(z, 2).out.numel() == 0
    assert rg.besselj_hess(z, 2).d2Jdz2.numel() == 0
    cams = torch.zeros((3, 11), dtype=torch.float64, device=cuda)
    X = torch.zeros((4, 3), dtype=torch.float64, device=cuda)
    w = torch.zeros(0, dtype=torch.float64, device=cuda)
    f = torch.zeros((0, 2), dtype=torch.float64, device=cuda)
    o = torch.zeros((0, 2), dtype=torch.int32, device=cuda)
    assert rg.ba_residuals(cams, X, w, f, o).out.shape == (0, 3)
    r = rg.ba_jacobian_csr(cams, X, w, f, o)
    torch.cuda.synchronize()
    assert r.rows.cpu().tolist() == [0] and r.cols.numel() == 0 and r.shape == (0, 33 + 12)
    h = rg.ba_jacobian_csr_host(cams.cpu().numpy(), X.cpu().numpy(), np.zeros(0),
                                np.zeros((0, 2)), np.zeros((0, 2), np.int32))
    assert h.rows.tolist() == [0] and h.vals.size == 0


@pytest.mark.parametrize("nu", [0, 1, 30, 600])
def test_extreme_orders_grad_run_hess(cuda, oracle, nu):
    z = np.array([1e-250, 1e-8, 0.3, 2.0, 9.5, 40.0, 150.0, 650.0])
    zt = torch.as_tensor(z, device=cuda)
    g = rg.besselj_grad(zt, nu)
    r = rg.besselj_run(zt, nu)
    h = rg.besselj_hess(zt, nu)
    torch.cuda.synchronize()
    J, dz, fail, _ = oracle.besselj_grad(nu, z)
    Jh, dzh, d2, failh, _ = oracle.besselj_hess(nu, z)
    names = [ERROR_NAMES[int(c)] for c in fail]
    for res in (g.fail, r.fail, h.fail):
        assert [ERROR_NAMES[int(c)] for c in res.cpu().numpy()] == names
    ok = fail == 0
    scale = np.maximum(np.abs(J), 1e-300)
    assert (np.abs(g.J.cpu().numpy()[ok] - J[ok]) <= 1e-9 * scale[ok] + 1e-13).all()
    assert np.array_equal(g.J.cpu().numpy()[ok], r.out.cpu().numpy()[ok])
    assert np.array_equal(g.J.cpu().numpy()[ok], h.J.cpu().numpy()[ok])
    assert np.array_equal(g.dJdz.cpu().numpy()[ok], h.dJdz.cpu().numpy()[ok])
    s2 = np.maximum(np.abs(d2), 1e-300)
    assert (np.abs(h.d2Jdz2.cpu().numpy()[ok] - d2[ok]) <= 1e-9 * s2[ok] + 1e-12).all()


def test_csr_odd_sizes_fall_back_correctly(cuda, oracle):
    """Block-tail and odd n_obs exercise the non-bulk store paths."""
    from test_ba_gpu import ba_inputs, to_dev
    rng = np.random.default_rng(11)
    for p in (1, 31, 33, 95, 1027):
        cams, X, w, feats, obs = ba_inputs(rng, 5, 9, p)
        r = rg.ba_jacobian_csr(*to_dev(cuda, cams, X, w, feats, obs))
        torch.cuda.synchronize()
        Jo, _, _ = oracle.ba_jac(cams, X, w, feats, obs)
        rows, cols, vals, shape = oracle.ba_sparse(5, 9, obs, Jo)
        assert np.array_equal(r.rows.cpu().numpy(), rows)
        assert np.array_equal(r.cols.cpu().numpy(), cols)
        v = r.vals.cpu().numpy()
        assert np.allclose(v, vals, rtol=1e-10, atol=1e-13 * np.abs(vals).max())


def test_out_buffers_and_devices_are_validated(cuda):
    z = torch.rand(100, dtype=torch.float64, device=cuda) + 0.1
    J = torch.empty(200, dtype=torch.float64, device=cuda)[::2]          # non-contiguous
    dz = torch.empty(100, dtype=torch.float64, device=cuda)
    fail = torch.empty(100, dtype=torch.uint8, device=cuda)
    with pytest.raises(rg.KindError):
        rg.besselj_grad(z, 2, out=(J, dz, fail))
    with pytest.raises(rg.KindError):
        rg.besselj_grad(z, 2, out=(dz, dz, fail.to(torch.int32)))
    ok = rg.besselj_grad(z, 2, out=(torch.empty_like(z), dz, fail))
    torch.cuda.synchronize()
    assert ok.dJdz is dz and not ok.fail.any()


def test_repeated_launches_are_bitwise_deterministic(cuda):
    """Every kernel family sums in a fixed order (no floating-point atomics):
    repeated launches on the same inputs give bitwise-equal outputs, including
    the GMM restoration replay (its side stream included)."""
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from test_ba_gpu import ba_inputs, to_dev
    from test_gmm_gpu import gmm_constants, inputs
    z = torch.as_tensor(np.random.default_rng(3).uniform(0.1, 12.0, 300001), device=cuda)
    a = rg.besselj_grad(z, 2)
    b = rg.besselj_grad(z, 2)
    assert torch.equal(a.J, b.J) and torch.equal(a.dJdz, b.dJdz) and torch.equal(a.fail, b.fail)
    args = to_dev(cuda, *ba_inputs(np.random.default_rng(4), 40, 300, 20000))
    p, q = rg.ba_jacobian(*args), rg.ba_jacobian(*args)
    assert torch.equal(p.J, q.J)
    d, K, N = 64, 25, 3000
    g = [torch.as_tensor(v, device=cuda) for v in inputs(np.random.default_rng(5), d, K, N)]
    cst = gmm_constants(d, K, N, 1.0, 0)
    r1 = rg.gmm_gradient(*g, 1.0, 0, cst)
    r2 = rg.gmm_gradient(*g, 1.0, 0, cst)
    assert torch.equal(r1.packed, r2.packed) and torch.equal(r1.resid, r2.resid)
