"""rl_seq_sum_f64: the reference's sequential binary64 accumulation chain
(`acc += t` statement by statement, numerics.py:296-339), evaluated in
parallel by one CTA, must be BIT-EXACT against the plain sequential loop —
on sequences chosen to break the parallel path's predictions: binade
crossings, zero crossings, round-half-even ties, mixed magnitudes,
subnormals, infinities.  The GMM restoration replay (k_gmm_restore) is this
evaluation over err!'s terms."""

import struct

import numpy as np
import pytest
import torch

import paper_2003_04617_b200 as rg

pytestmark = pytest.mark.gpu


def bits(x):
    return struct.unpack("<q", struct.pack("<d", x))[0]


def seq_py(t, e0, mark):
    """The definition: Python floats are IEEE binary64 (as the reference's)."""
    e = e0
    em = e0 if mark == 0 else None
    for j, v in enumerate(t):
        e = e + v
        if j + 1 == mark:
            em = e
    return em, e


def gmm_like(rng, n):
    a = rng.uniform(-420.0, -280.0, n)      # log(se_i) + ... scale of configs[2]
    b = rng.uniform(-60.0, 0.0, n)
    fwd = np.stack([a, b], 1).ravel()
    p = np.array([-123456.789, 9876.54321, -0.0, 1.25e5])
    return np.concatenate([fwd, p, -p[::-1], -fwd[::-1]])


def cases():
    rng = np.random.default_rng(7)
    yield "gmm_like", gmm_like(rng, 20000), 0.0, True
    yield "gmm_like_err0", gmm_like(rng, 3000), 1234.5678, True
    yield "normal", rng.normal(0, 1, 100003), 0.0, True
    yield "mixed_magnitudes", rng.normal(0, 1, 50000) * 10.0 ** rng.uniform(-30, 30, 50000), 0.0, False
    yield "zero_walk", rng.choice([-1.0, 1.0], 40000) * rng.uniform(0.5, 1.5, 40000), 0.0, False
    # at 2^53 the grid is 2: integer and half-integer steps round half to even
    ties = rng.integers(-3, 4, 30000).astype(np.float64) + 0.5 * (rng.random(30000) < 0.5)
    yield "ties", ties, 2.0 ** 53, False
    yield "positive_growth", rng.uniform(0, 1e3, 60000), 0.0, True
    yield "subnormal", rng.normal(0, 1, 5000) * 2.0 ** -1060, 0.0, False
    yield "cancel_to_zero", np.concatenate([np.full(1000, 0.1), np.full(1000, -0.1)]), 0.0, False
    t = rng.normal(0, 1, 3000)
    t[1500] = np.inf
    yield "infinity", t, 0.0, False
    for m in (0, 1, 2, 31, 511, 512, 513, 1025):
        yield f"small_{m}", rng.normal(0, 100, m), 0.5, False


@pytest.mark.parametrize("name,t,e0,expect_fast", list(cases()), ids=[c[0] for c in cases()])
def test_parallel_chain_is_bit_exact(cuda, name, t, e0, expect_fast):
    dev = torch.as_tensor(np.ascontiguousarray(t, dtype=np.float64), device=cuda)
    M = t.shape[0]
    rng = np.random.default_rng(M)
    for mark in sorted({0, M, M // 2, int(rng.integers(0, M + 1))}):
        em_p, ef_p, ver = rg.seq_sum(dev, e0, mark)
        em_s, ef_s, ver_s = rg.seq_sum(dev, e0, mark, force_serial=True)
        assert not ver_s
        em_r, ef_r = seq_py(t.tolist(), e0, mark)
        assert bits(ef_s) == bits(ef_r) and bits(em_s) == bits(em_r), name
        assert bits(ef_p) == bits(ef_r), (name, mark, ef_p, ef_r)
        assert bits(em_p) == bits(em_r), (name, mark, em_p, em_r)
        if expect_fast:
            assert ver, f"{name}: the parallel path should verify"


def test_residual_is_the_rounding_of_the_chain(cuda):
    """A forward-then-inverse chain over GMM-scale terms does not return to
    exactly 0 in binary64; the device residual is the sequential one."""
    t = gmm_like(np.random.default_rng(3), 10000)
    _, resid, ver = rg.seq_sum(torch.as_tensor(t, device=cuda), 0.0)
    assert ver
    assert resid == seq_py(t.tolist(), 0.0, len(t))[1]
    assert resid != 0.0


def test_invalid_arguments(cuda):
    from paper_2003_04617_b200 import _native
    L = _native.lib()
    assert L.rl_seq_sum_f64(None, 5, 0.0, 0, 0, None, None, None) == _native.RL_ERR_INVALID
    t = torch.zeros(4, dtype=torch.float64, device=cuda)
    with pytest.raises(rg.NativeLibraryError):
        rg.seq_sum(t, 0.0, 7)
