"""run / uncall / objective-only device kernels vs the
reference: golden run/uncall outputs made by the reference interpreter
(oracle/gen_golden.py gen_run), the gradient goldens' primal outputs, and the
round-trip property uncall(run(a)) == a."""

import numpy as np
import pytest
import torch

import paper_2003_04617_b200 as rg
from conftest import close_series
from oracle import ERROR_NAMES

pytestmark = pytest.mark.gpu


def test_besselj_run_uncall_goldens(cuda, golden):
    g = golden("run")
    z = torch.as_tensor(g["bj_z"], device=cuda)
    o0 = torch.as_tensor(g["bj_out0"], device=cuda)
    a = rg.besselj_run(z, 2, out_in=o0, direction=1)
    b = rg.besselj_run(z, 2, out_in=o0, direction=-1)
    torch.cuda.synchronize()
    names = np.array([ERROR_NAMES[int(f)] for f in a.fail.cpu().numpy()])
    assert np.array_equal(names, g["bj_err"])
    ok = g["bj_err"] == ""
    zz = g["bj_z"][ok]
    assert close_series(a.out.cpu().numpy()[ok], g["bj_run"][ok], 2, zz).all()
    assert close_series(b.out.cpu().numpy()[ok], g["bj_uncall"][ok], 2, zz).all()


def test_besselj_run_equals_gradient_primal(cuda, golden):
    g = golden("bessel")
    z = torch.as_tensor(g["z"][:1000], device=cuda)
    r = rg.besselj_run(z, 2)
    grad = rg.besselj_grad(z, 2)
    torch.cuda.synchronize()
    assert torch.equal(r.out, grad.J)                   # same primal arithmetic, bit for bit
    assert torch.equal(r.fail, grad.fail)


def test_besselj_round_trip(cuda):
    z = torch.rand(100000, dtype=torch.float64, device=cuda) * 9.9 + 0.1
    o0 = torch.randn(100000, dtype=torch.float64, device=cuda)
    mid = rg.besselj_run(z, 2, out_in=o0).out
    back = rg.besselj_run(z, 2, out_in=mid, direction=-1).out
    assert torch.max(torch.abs(back - o0)).item() <= 1e-9   # values_close(.., 1e-9)


def test_ba_residuals(cuda, golden):
    b = golden("ba")
    n = b["w"].size
    obs = np.stack([np.arange(n), np.arange(n)], 1).astype(np.int32)
    t = lambda a: torch.as_tensor(a, device=cuda)  # noqa: E731
    r = rg.ba_residuals(t(b["cams"]), t(b["X"]), t(b["w"]), t(b["feat"]), t(obs))
    torch.cuda.synchronize()
    e = r.out.cpu().numpy()
    assert not r.fail.any()
    assert np.allclose(e[:, :2], b["e"], rtol=1e-12, atol=1e-12)
    assert np.array_equal(e[:, 2], 1.0 - b["w"] * b["w"])
    g = golden("run")
    p = rg.load_example("ba_proj")
    for o in range(16):
        args = [float(g["ba_e_in"][o, 0]), float(g["ba_e_in"][o, 1]),
                rg.Array.vector(g["ba_cams"][o].tolist()), rg.Array.vector(g["ba_X"][o].tolist()),
                float(g["ba_w"][o]), float(g["ba_feat"][o, 0]), float(g["ba_feat"][o, 1])]
        assert np.allclose(rg.run(p, "ba_proj", args)[:2], g["ba_run"][o], rtol=1e-12, atol=1e-12)
        assert np.allclose(rg.uncall(p, "ba_proj", args)[:2], g["ba_uncall"][o], rtol=1e-12,
                           atol=1e-12)


def test_gmm_objective_matches_goldens_and_gradient(cuda, golden):
    G = golden("gmm")
    for ci in range(int(G["ncases"])):
        pre = f"c{ci}_"
        d, K, N, m = (int(v) for v in G[pre + "dims"])
        t = lambda a: torch.as_tensor(a, device=cuda)  # noqa: E731
        args = (t(G[pre + "alphas"]), t(G[pre + "means"]), t(G[pre + "icf"]), t(G[pre + "x"]),
                float(G[pre + "gamma"]), m, float(G[pre + "cst"]))
        r = rg.gmm_objective(*args)
        full = rg.gmm_grad(*args)
        torch.cuda.synchronize()
        e = float(r.out.item())
        assert abs(e - float(G[pre + "err"])) <= 1e-12 * abs(float(G[pre + "err"]))
        assert e == float(full.err.item())                 # same kernels up to the objective


def test_dropin_run_uncall_check(cuda):
    p = rg.load_example("besselj")
    a = [0.25, 2, 3.5]
    mid = rg.run(p, "besselj", a)
    back = rg.uncall(p, "besselj", mid)
    assert back[1:] == a[1:] and abs(back[0] - a[0]) <= 1e-15
    rep = rg.check_reversibility(p, "besselj", a)
    assert rep.ok and rep.max_deviation <= 1e-15
    bad = rg.check_reversibility(p, "besselj", [0.0, 2, -1.0])
    assert not bad.ok and "RevDomainError" in bad.error
    with pytest.raises(rg.DirtyAncilla):
        rg.run(p, "besselj", [0.0, 2, 30.0])
