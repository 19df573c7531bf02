import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100) device")


@pytest.fixture(scope="session")
def oracle():
    import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name + ".npz"))
    return load


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test on a host without CUDA")  # fail loudly, never skip silently
    from paper_2003_04617_b200 import _native
    _native.lib()
    return torch.device("cuda", 0)


def close(a, b, rtol=1e-10, atol=1e-12):
    """FP64 parity bar: |a - b| <= rtol |b| + atol (atol covers outputs that
    cancel to ~0, e.g. J_2 near its zeros where the terms are O(10))."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) <= rtol * np.abs(b) + atol


def close_series(a, b, nu, z, rtol=1e-12, ftol=5e-14):
    """Bessel parity bar: 1e-12 relative plus an absolute floor of 5e-14 x
    the series' absolute scale I_nu(z) + I_nu'(z) (the sum of |terms| and of
    |d term/dz|): cancellation in the alternating series makes the absolute
    error of ANY binary64 evaluation — the reference's included — scale with
    it, and a 1-ulp difference in log(z) moves every term by ~(2k+nu) ulp.
    Measured (profiles/r02/parity_stats.json, 1.2M elements over nu 0-12,
    z to 60, random thr / seed): |err| <= 5.2e-16 scale for J and 6.7e-15
    scale for dJ/dz; relative error <= 1.4e-14 wherever |ref| > 1e-2 scale."""
    import scipy.special as sp
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    z = np.asarray(z, np.float64)
    scale = sp.iv(nu, z) + np.abs(sp.ivp(nu, z))
    return np.abs(a - b) <= rtol * np.abs(b) + ftol * scale
