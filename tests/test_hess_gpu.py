"""Batched forward-over-reverse Hessian of besselj (rl_besselj_hess_f64,
SURVEY §8(f) rank 3) against the reference hessian goldens and the C oracle.

The Dual sweeps run the reference's operation sequence; the only
differences are exp (fexp, <= 1 ulp) and log(z) (libdevice), so d2J/dz2
is held to the Bessel gradient's tolerance scaled to the second
derivative's series: |gpu - ref| <= 1e-10 |ref| + 1e-13 (I_nu + I_nu' +
I_nu'').  J, dJ/dz, the failure classes and the trip counts are
bit-identical to the gradient kernel's."""

import numpy as np
import pytest
import torch

import paper_2003_04617_b200 as rg
from oracle import ERROR_NAMES

pytestmark = pytest.mark.gpu


def tol_d2(ref, z, nu):
    from scipy.special import iv, ivp
    scale = iv(nu, z) + np.abs(ivp(nu, z, 1)) + np.abs(ivp(nu, z, 2))
    return 1e-10 * np.abs(ref) + 1e-13 * scale


def test_hess_goldens(cuda, golden):
    g = golden("hess")
    for nu in np.unique(g["nu"]):
        m = g["nu"] == nu
        z = g["z"][m]
        r = rg.besselj_hess(torch.as_tensor(z, device=cuda), int(nu))
        torch.cuda.synchronize()
        names = np.array([ERROR_NAMES[int(f)] for f in r.fail.cpu().numpy()])
        assert np.array_equal(names, g["err"][m])
        ok = g["err"][m] == ""
        ref = g["H"][m][ok, 1, 1]
        d2 = r.d2Jdz2.cpu().numpy()[ok]
        assert (np.abs(d2 - ref) <= tol_d2(ref, z[ok], int(nu))).all()


def test_hess_primal_and_gradient_bit_identical_to_grad_kernel(cuda):
    z = torch.rand(300000, dtype=torch.float64, device=cuda) * 9.9 + 0.1
    h = rg.besselj_hess(z, 2)
    gr = rg.besselj_grad(z, 2)
    torch.cuda.synchronize()
    assert torch.equal(h.J, gr.J) and torch.equal(h.dJdz, gr.dJdz)
    assert torch.equal(h.fail, gr.fail)
    assert h.sum_trips == gr.sum_trips


def test_hess_vs_oracle_random(cuda, oracle):
    rng = np.random.default_rng(9)
    for nu in (0, 2, 7):
        z = rng.uniform(0.05, 12.0, 20000)
        r = rg.besselj_hess(torch.as_tensor(z, device=cuda), nu)
        torch.cuda.synchronize()
        J, dz, d2, fail, trips = oracle.besselj_hess(nu, z)
        assert np.array_equal(r.fail.cpu().numpy(), fail)
        ok = fail == 0
        assert (np.abs(r.d2Jdz2.cpu().numpy()[ok] - d2[ok]) <= tol_d2(d2[ok], z[ok], nu)).all()
        assert r.sum_trips == trips


def test_hess_edge_and_error_cases(cuda, oracle):
    z = np.array([1e-300, 1e-200, 1e-5, 300.0, 800.0, 0.0, -3.0, np.nan, np.inf, 5.0])
    r = rg.besselj_hess(torch.as_tensor(z, device=cuda), 2)
    torch.cuda.synchronize()
    J, dz, d2, fail, _ = oracle.besselj_hess(2, z)
    assert np.array_equal(r.fail.cpu().numpy(), fail)
    ok = fail == 0
    assert np.allclose(r.d2Jdz2.cpu().numpy()[ok], d2[ok], rtol=1e-10, atol=1e-300)


def test_dropin_hessian(cuda, golden):
    p = rg.load_example("besselj")
    res = rg.hessian(p, "besselj", [0.0, 2, 3.7])
    assert res.matrix.shape == (2, 2) and res.symmetry_error == 0.0
    assert res.matrix[0, 0] == res.matrix[0, 1] == res.matrix[1, 0] == 0.0
    assert abs(res.matrix[1, 1] - (-0.25515272541174533)) <= 1e-12      # reference value
    with pytest.raises(rg.DirtyAncilla):
        rg.hessian(p, "besselj", [0.0, 2, 25.0])
    # the registered ba functions' Hessians come from codegen's Dual kernel:
    # e! += 1.0; e! -= abs2(w) -> d2 e / dw2 = -2 (seed e!)
    res = rg.hessian(rg.load_example("ba_proj"), "ba_weight", [0.0, 0.7])
    assert np.array_equal(res.matrix, [[0.0, 0.0], [0.0, -2.0]])
