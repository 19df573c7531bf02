"""Multi-process host logic on CPU (gloo, world_size 2): sharding ranges and
the GMM packed-partial allreduce (the one collective of the path).  The
per-rank partial is computed here with torch autograd on CPU — a stand-in
for the CUDA kernel, which the GPU tests cover (test_gmm_gpu
::test_shards_sum_to_the_whole) — and the result is checked against the
oracle."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2003_04617_b200 import parallel
from paper_2003_04617_b200.kernels import GMMResult, gmm_packed_size


def test_shard_range_covers_exactly():
    for n in (0, 1, 7, 1000, 2 ** 26 + 3):
        for world in (1, 2, 3, 8):
            parts = [parallel.shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        parallel.shard_range(10, 2, 2)


def gmm_constants(d, K, N, gamma, m):
    n = d + m + 1
    lgd = 0.25 * d * (d - 1) * math.log(math.pi) + sum(
        math.lgamma(0.5 * n + 0.5 * (1 - j)) for j in range(1, d + 1))
    C = n * d * (math.log(gamma) - 0.5 * math.log(2.0)) - lgd
    return -N * d * 0.5 * math.log(2.0 * math.pi) - K * C


def torch_partial(alphas, means, icf, x, gamma, m, cst, N_total, add_param_terms, **kw):
    K, d = means.shape
    al = alphas.clone().requires_grad_(True)
    me = means.clone().requires_grad_(True)
    ic = icf.clone().requires_grad_(True)
    qd = torch.exp(ic[:, :d])
    L = torch.zeros(K, d, d, dtype=torch.float64)
    for k in range(K):
        L[k] = torch.diag(qd[k])
        li = d
        for a in range(d):
            for b in range(a + 1, d):
                L[k, b, a] = ic[k, li]
                li += 1
    xc = x[:, None, :] - me[None]
    qx = torch.einsum("kba,nka->nkb", L, xc)
    mt = al[None] + ic[:, :d].sum(1)[None] - 0.5 * (qx ** 2).sum(-1)
    f = torch.logsumexp(mt, 1).sum()
    if add_param_terms:
        f = f + (-N_total * torch.logsumexp(al, 0)
                 + 0.5 * gamma ** 2 * ((qd ** 2).sum() + (ic[:, d:] ** 2).sum())
                 - m * ic[:, :d].sum() + cst)
    f.backward()
    packed = torch.cat([f.detach().reshape(1), al.grad, me.grad.reshape(-1), ic.grad.reshape(-1)])
    assert packed.numel() == gmm_packed_size(d, K)
    return GMMResult(None, None, None, None, torch.zeros(x.shape[0], dtype=torch.uint8),
                     torch.zeros(2, dtype=torch.int64), packed)


def _worker(rank, world, port, data, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    alphas, means, icf, x, gamma, m, cst = data
    N = x.shape[0]
    lo, hi = parallel.shard_range(N, rank, world)
    t = torch.from_numpy
    res = parallel.gmm_grad_distributed(t(alphas), t(means), t(icf), t(x[lo:hi]), gamma, m, cst,
                                        N, local_fn=torch_partial)
    out_q.put((rank, res.packed.numpy().copy()))
    # the timing helper used by bench.py: max over ranks
    assert parallel.allreduce_max(float(rank)) == world - 1
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gmm_allreduce_world2_matches_oracle(oracle):
    rng = np.random.default_rng(31)
    d, K, N = 4, 3, 23
    alphas, means = rng.normal(size=K), rng.uniform(size=(K, d))
    icf, x = rng.normal(size=(K, d * (d + 1) // 2)) * 0.5, rng.uniform(size=(N, d))
    gamma, m = 1.0, 0
    cst = gmm_constants(d, K, N, gamma, m)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, (alphas, means, icf, x, gamma, m, cst), q))
             for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rc, e, ga, gm, gi = oracle.gmm_grad(alphas, means, icf, x, gamma, m, cst)
    want = np.concatenate([[e], ga, gm.ravel(), gi.ravel()])
    for r in (0, 1):
        np.testing.assert_allclose(results[r], want, rtol=1e-11, atol=1e-11)
    assert np.array_equal(results[0], results[1])
