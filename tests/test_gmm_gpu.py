"""GMM objective-gradient kernels (rl_gmm_grad_f64) vs the reference.

The device computes the per-point terms in parallel (fresh scratch per
point) and contracts products to FMA, so results match the sequential
reference to rounding: the bar is |gpu - ref| <= 1e-10 |ref| + 1e-12 max|ref|
per gradient array, and the objective to 1e-12 relative."""

import math

import numpy as np
import pytest
import torch

import paper_2003_04617_b200 as rg

pytestmark = pytest.mark.gpu


def arr_close(a, b, rtol=1e-10, floor=1e-12):
    a = np.asarray(a)
    b = np.asarray(b)
    return np.all(np.abs(a - b) <= rtol * np.abs(b) + floor * np.max(np.abs(b)))


def gmm_constants(d, K, N, gamma, m):
    n = d + m + 1
    lgd = 0.25 * d * (d - 1) * math.log(math.pi) + sum(
        math.lgamma(0.5 * n + 0.5 * (1 - j)) for j in range(1, d + 1))
    C = n * d * (math.log(gamma) - 0.5 * math.log(2.0)) - lgd
    return -N * d * 0.5 * math.log(2.0 * math.pi) - K * C


def inputs(rng, d, K, N):
    return (rng.normal(0.0, 1.0, K), rng.uniform(0.0, 1.0, (K, d)),
            rng.normal(0.0, 1.0, (K, d * (d + 1) // 2)) * 0.5, rng.uniform(0.0, 1.0, (N, d)))


def run_dev(dev, alphas, means, icf, x, gamma, m, cst, **kw):
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)  # noqa: E731
    r = rg.gmm_grad(t(alphas), t(means), t(icf), t(x), gamma, m, cst, **kw)
    torch.cuda.synchronize()
    return (float(r.err.item()), r.g_alphas.cpu().numpy(), r.g_means.cpu().numpy(),
            r.g_icf.cpu().numpy(), r.fail.cpu().numpy(), r)


def check_vs(ref, got):
    e, ga, gm, gi = ref
    assert abs(got[0] - e) <= 1e-12 * abs(e) + 1e-9
    assert arr_close(got[1], ga)
    assert arr_close(got[2], gm)
    assert arr_close(got[3], gi)


def test_golden_vectors(cuda, golden):
    G = golden("gmm")
    for ci in range(int(G["ncases"])):
        p = f"c{ci}_"
        d, K, N, m = (int(v) for v in G[p + "dims"])
        got = run_dev(cuda, G[p + "alphas"], G[p + "means"], G[p + "icf"], G[p + "x"],
                      float(G[p + "gamma"]), m, float(G[p + "cst"]))
        assert not got[4].any()
        check_vs((float(G[p + "err"]), G[p + "g_alphas"], G[p + "g_means"], G[p + "g_icf"]), got)


@pytest.mark.parametrize("d,K,N", [(7, 3, 50), (32, 4, 300), (33, 5, 129), (64, 6, 257),
                                   (100, 3, 70), (128, 2, 65)])
def test_random_shapes_vs_oracle(cuda, oracle, d, K, N):
    rng = np.random.default_rng(d * 1000 + K * 10 + N)
    alphas, means, icf, x = inputs(rng, d, K, N)
    gamma, m = 1.1, 1
    cst = gmm_constants(d, K, N, gamma, m)
    rc, e, ga, gm, gi = oracle.gmm_grad(alphas, means, icf, x, gamma, m, cst)
    assert rc == 0
    got = run_dev(cuda, alphas, means, icf, x, gamma, m, cst)
    assert not got[4].any()
    check_vs((e, ga, gm, gi), got)


def test_config3_full_size_vs_oracle(cuda, oracle):
    """configs[2]: d=64, K=25, N=10,000 (the oracle runs all 8 passes).

    At this size the reference's own final check — err! restored to 0.0
    within the default 1e-9 after 10^4 accumulate/uncompute steps — fails
    (RevError, oracle rc 5): the survey ran it with float_tolerance 1e-6,
    and so does this test."""
    d, K, N = 64, 25, 10000
    alphas, means, icf, x = inputs(np.random.default_rng(2), d, K, N)
    cst = gmm_constants(d, K, N, 1.0, 0)
    rc, e, ga, gm, gi = oracle.gmm_grad(alphas, means, icf, x, 1.0, 0, cst)
    assert rc == 5                                   # RevError at tol 1e-9, as the reference
    rc, e, ga, gm, gi = oracle.gmm_grad(alphas, means, icf, x, 1.0, 0, cst, tol=1e-6)
    assert rc == 0
    got = run_dev(cuda, alphas, means, icf, x, 1.0, 0, cst)
    assert not got[4].any() and got[5].n_failed == 0
    check_vs((e, ga, gm, gi), got)


def test_shards_sum_to_the_whole(cuda):
    """The data-parallel split used by the multi-GPU path: per-point terms of
    each shard + parameter terms once == the unsharded result."""
    d, K, N = 40, 5, 1000
    alphas, means, icf, x = inputs(np.random.default_rng(9), d, K, N)
    cst = gmm_constants(d, K, N, 1.0, 0)
    whole = run_dev(cuda, alphas, means, icf, x, 1.0, 0, cst)[5].packed.cpu().numpy()
    parts = []
    for r, (lo, hi) in enumerate(((0, 337), (337, 1000))):
        res = run_dev(cuda, alphas, means, icf, x[lo:hi], 1.0, 0, cst, N_total=N,
                      add_param_terms=(r == 0))[5]
        parts.append(res.packed.cpu().numpy())
    summed = parts[0] + parts[1]
    assert arr_close(summed, whole, rtol=1e-12, floor=1e-13)


def test_no_points_gives_parameter_terms_only(cuda, oracle):
    d, K = 5, 3
    alphas, means, icf, _ = inputs(np.random.default_rng(4), d, K, 1)
    x = np.zeros((0, d))
    rc, e, ga, gm, gi = oracle.gmm_grad(alphas, means, icf, x, 1.0, 0, 2.5)
    got = run_dev(cuda, alphas, means, icf, x, 1.0, 0, 2.5)
    check_vs((e, ga, gm, gi), got)


def test_against_torch_autograd_at_scale(cuda):
    """configs[4] shape class (d=128, K=200) on 4,000 points, vs torch FP64
    autograd on the GPU (an independent implementation of the objective)."""
    d, K, N = 128, 200, 4000
    rng = np.random.default_rng(4)
    alphas, means, icf, x = inputs(rng, d, K, N)
    gamma, m = 1.0, 0
    cst = gmm_constants(d, K, N, gamma, m)
    got = run_dev(cuda, alphas, means, icf, x, gamma, m, cst)
    dev = cuda
    al = torch.tensor(alphas, device=dev, requires_grad=True)
    me = torch.tensor(means, device=dev, requires_grad=True)
    ic = torch.tensor(icf, device=dev, requires_grad=True)
    qd = torch.exp(ic[:, :d])
    rows, cols = np.tril_indices(d, -1)
    order = np.lexsort((rows, cols))           # column-major strict lower triangle
    L = torch.zeros(K, d, d, dtype=torch.float64, device=dev)
    L[:, torch.arange(d), torch.arange(d)] = qd
    L[:, torch.as_tensor(rows[order], device=dev), torch.as_tensor(cols[order], device=dev)] = ic[:, d:]
    xt = torch.tensor(x, device=dev)
    xc = xt[:, None, :] - me[None]
    qx = torch.einsum("kba,nka->nkb", L, xc)
    mt = al[None] + ic[:, :d].sum(1)[None] - 0.5 * (qx ** 2).sum(-1)
    f = (torch.logsumexp(mt, 1).sum() - N * torch.logsumexp(al, 0)
         + 0.5 * gamma ** 2 * ((qd ** 2).sum() + (ic[:, d:] ** 2).sum()) - m * ic[:, :d].sum()
         + cst)
    f.backward()
    assert abs(got[0] - f.item()) <= 1e-11 * abs(f.item())
    assert arr_close(got[1], al.grad.cpu().numpy(), rtol=1e-9, floor=1e-11)
    assert arr_close(got[2], me.grad.cpu().numpy(), rtol=1e-9, floor=1e-11)
    assert arr_close(got[3], ic.grad.cpu().numpy(), rtol=1e-9, floor=1e-11)


def test_dropin_gradient(cuda, golden):
    G = golden("gmm")
    p = rg.load_example("gmm")
    pre = "c1_"
    d, K, N, m = (int(v) for v in G[pre + "dims"])
    A = lambda a: rg.Array.matrix(a.tolist()) if a.ndim == 2 else rg.Array.vector(a.tolist())  # noqa
    Z = lambda *s: A(np.zeros(s))  # noqa: E731
    args = [0.0, A(G[pre + "alphas"]), A(G[pre + "means"]), A(G[pre + "icf"]), A(G[pre + "x"]),
            Z(K, d), Z(K), Z(d), Z(d), Z(K), Z(K), float(G[pre + "gamma"]), m,
            float(G[pre + "cst"])]
    primal, g = rg.gradient(p, rg.GradRequest("gmm", args, wrt=["alphas", "means", "icf"]))
    assert abs(primal[0] - float(G[pre + "err"])) <= 1e-12 * abs(float(G[pre + "err"]))
    assert arr_close(np.array(g["icf"].data).reshape(K, -1), G[pre + "g_icf"])
    bad = list(args)
    bad[7] = rg.Array.vector([1.0] + [0.0] * (d - 1))
    with pytest.raises(rg.KindError):
        rg.gradient(p, rg.GradRequest("gmm", bad))
