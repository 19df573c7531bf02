"""The C oracle against golden vectors produced by the REFERENCE interpreter
(oracle/gen_golden.py imports /root/reference).  Bit-for-bit: the oracle
restates the reference's operation sequence with the same libm."""

import numpy as np

from oracle import ERROR_NAMES


def test_bessel_bitexact_all_orders_and_errors(oracle, golden):
    g = golden("bessel")
    for nu in np.unique(g["nu"]):
        m = g["nu"] == nu
        J, dz, fail, _ = oracle.besselj_grad(int(nu), g["z"][m])
        names = np.array([ERROR_NAMES[int(f)] for f in fail])
        assert np.array_equal(names, g["err"][m]), nu
        ok = g["err"][m] == ""
        assert np.array_equal(J[ok], g["J"][m][ok])
        assert np.array_equal(dz[ok], g["dJdz"][m][ok])


def test_bessel_config1_is_complete(golden):
    g = golden("bessel")
    m = g["nu"] == 2
    assert m.sum() >= 1000
    z1 = np.random.default_rng(0).uniform(0.1, 10.0, 1000)
    assert np.array_equal(g["z"][:1000], z1)  # configs[0]: 1,000 z, seed 0


def test_ba_bitexact(oracle, golden):
    b = golden("ba")
    n = b["w"].size
    obs = np.stack([np.arange(n), np.arange(n)], 1)
    J, err, fail = oracle.ba_jac(b["cams"], b["X"], b["w"], b["feat"], obs)
    assert not fail.any()
    want = np.concatenate([b["J"].reshape(n, 30), b["wjac"][:, None]], 1)
    assert np.array_equal(J, want)
    assert np.array_equal(err[:, :2], b["e"])


def test_ba_index_errors(oracle, golden):
    b = golden("ba")
    obs = np.array([[0, 0], [5, 0], [0, -1], [0, 1]], np.int32)
    J, err, fail = oracle.ba_jac(b["cams"][:2], b["X"][:2], b["w"][:4], b["feat"][:4], obs)
    assert list(fail) == [0, 8, 8, 0]


def test_gmm_bitexact(oracle, golden):
    G = golden("gmm")
    for ci in range(int(G["ncases"])):
        p = f"c{ci}_"
        d, K, N, m = (int(v) for v in G[p + "dims"])
        rc, e, ga, gm, gi = oracle.gmm_grad(G[p + "alphas"], G[p + "means"], G[p + "icf"],
                                            G[p + "x"], float(G[p + "gamma"]), m,
                                            float(G[p + "cst"]))
        assert rc == 0
        assert e == G[p + "err"]
        assert np.array_equal(ga, G[p + "g_alphas"])
        assert np.array_equal(gm, G[p + "g_means"])
        assert np.array_equal(gi, G[p + "g_icf"])


def test_bessel_known_values(oracle):
    # closed forms: J_nu and J_nu' from scipy agree to the series' accuracy
    import scipy.special as sp
    z = np.linspace(0.2, 9.5, 200)
    for nu in (0, 1, 2, 3):
        J, dz, fail, _ = oracle.besselj_grad(nu, z)
        assert not fail.any()
        assert np.max(np.abs(J - sp.jv(nu, z))) < 1e-12
        assert np.max(np.abs(dz - sp.jvp(nu, z))) < 1e-12


def test_bessel_checks_are_observers(oracle):
    z = np.random.default_rng(5).uniform(0.1, 10.0, 500)
    a = oracle.besselj_grad(2, z, invcheck=True)
    b = oracle.besselj_grad(2, z, invcheck=False)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_bessel_fuel(oracle):
    J, dz, fail, _ = oracle.besselj_grad(2, np.array([5.0]), max_trips=3)
    assert fail[0] == 6


def test_gmm_against_torch_autograd(oracle):
    """Independent cross-check of the program itself (not of the kernels)."""
    import math

    import torch
    rng = np.random.default_rng(7)
    d, K, N = 6, 3, 9
    alphas, means = rng.normal(size=K), rng.uniform(size=(K, d))
    icf, x = rng.normal(size=(K, d * (d + 1) // 2)) * 0.5, rng.uniform(size=(N, d))
    gamma, m = 1.0, 0
    n = d + m + 1
    C = n * d * (math.log(gamma) - 0.5 * math.log(2)) - (
        0.25 * d * (d - 1) * math.log(math.pi)
        + sum(math.lgamma(0.5 * n + 0.5 * (1 - j)) for j in range(1, d + 1)))
    cst = -N * d * 0.5 * math.log(2 * math.pi) - K * C
    rc, e, ga, gm, gi = oracle.gmm_grad(alphas, means, icf, x, gamma, m, cst)
    al = torch.tensor(alphas, requires_grad=True)
    me = torch.tensor(means, requires_grad=True)
    ic = torch.tensor(icf, requires_grad=True)
    qd = torch.exp(ic[:, :d])
    L = torch.zeros(K, d, d, dtype=torch.float64)
    for k in range(K):
        L[k] = torch.diag(qd[k])
        li = d
        for a in range(d):
            for b in range(a + 1, d):
                L[k, b, a] = ic[k, li]
                li += 1
    xc = torch.tensor(x)[:, None, :] - me[None]
    qx = torch.einsum("kba,nka->nkb", L, xc)
    mt = al[None] + ic[:, :d].sum(1)[None] - 0.5 * (qx ** 2).sum(-1)
    f = (torch.logsumexp(mt, 1).sum() - N * torch.logsumexp(al, 0)
         + 0.5 * gamma ** 2 * ((qd ** 2).sum() + (ic[:, d:] ** 2).sum())
         - m * ic[:, :d].sum() + cst)
    f.backward()
    assert rc == 0
    assert abs(e - f.item()) <= 1e-12 * abs(f.item())
    assert np.allclose(ga, al.grad.numpy(), rtol=1e-11, atol=1e-12)
    assert np.allclose(gm, me.grad.numpy(), rtol=1e-11, atol=1e-12)
    assert np.allclose(gi, ic.grad.numpy(), rtol=1e-11, atol=1e-12)


def test_oracle_hessian_bit_identical_to_reference(oracle, golden):
    """oracle.besselj_hess (C, Dual sweeps) against reference
    autodiff.hessian on 1,120 cases: H[z, z] bit for bit, the other entries
    zero, and the same error classes."""
    g = golden("hess")
    for nu in np.unique(g["nu"]):
        m = g["nu"] == nu
        z, H, err = g["z"][m], g["H"][m], g["err"][m]
        J, dz, d2, fail, _ = oracle.besselj_hess(int(nu), z)
        names = np.array([oracle.ERROR_NAMES[int(f)] for f in fail])
        assert np.array_equal(names, err)
        ok = err == ""
        assert np.array_equal(d2[ok], H[ok, 1, 1])                     # bit for bit
        assert (H[ok, 0, :] == 0).all() and (H[ok, :, 0] == 0).all()
        Jg, dzg, fg, _ = oracle.besselj_grad(int(nu), z)
        assert np.array_equal(J[ok], Jg[ok]) and np.array_equal(dz[ok], dzg[ok])


def test_bessel_fuel_formula_matches_reference_step_counts(oracle, golden):
    """The reference's statement count of one besselj sweep (read from its
    interpreter, bessel_fuel.npz) is 31 + 6 nu + 22 T for T series trips
    (the oracle's trip count): the exact fuel map kernels.bessel_trip_cap."""
    from paper_2003_04617_b200.kernels import bessel_trip_cap
    G = golden("bessel_fuel")
    for nu, z, steps in zip(G["nu"], G["z"], G["steps"]):
        _, _, f, trips = oracle.besselj_grad(int(nu), np.array([z]))
        assert f[0] == 0
        assert steps == 31 + 6 * int(nu) + 22 * int(trips)
        assert bessel_trip_cap(steps, int(nu)) == int(trips)
        assert bessel_trip_cap(steps - 1, int(nu)) == int(trips) - 1


def test_gmm_statement_count_formula(golden):
    """rl_gmm_statement_count against the reference's own counts
    (gmm_fuel.npz), with the argmax steps recomputed here in numpy."""
    from paper_2003_04617_b200.kernels import gmm_alpha_updates, gmm_statement_count
    G = golden("gmm_fuel")
    for ci in range(int(G["ncases"])):
        d, K, N = (int(v) for v in G[f"c{ci}_dims"])
        al, me = G[f"c{ci}_alphas"], G[f"c{ci}_means"].reshape(K, d)
        ic, x = G[f"c{ci}_icf"].reshape(K, -1), G[f"c{ci}_x"].reshape(N, d)
        U = 0
        for i in range(N):
            mt = []
            for k in range(K):
                L = np.diag(np.exp(ic[k, :d]))
                li = d
                for a in range(d):
                    for b in range(a + 1, d):
                        L[b, a] = ic[k, li]
                        li += 1
                q = L @ (x[i] - me[k])
                mt.append(al[k] + ic[k, :d].sum() - 0.5 * q @ q)
            best = 0
            for k in range(1, K):
                if mt[k] > mt[best]:
                    best, U = k, U + 1
        assert gmm_statement_count(d, K, N, U, gmm_alpha_updates(al)) == int(G["steps"][ci])
