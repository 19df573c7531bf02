"""Generic .rnl -> CUDA compilation (codegen.py) against
reference gradient() goldens (tests/golden/codegen.npz, made by
oracle/gen_golden.py codegen) and, for besselj.rnl compiled by the generic
path, against the reference Bessel goldens.  Arithmetic-only programs are
bit-identical; transcendental ones differ only through libdevice vs the host
libm (<= 2 ulp per call), held to 1e-12 relative."""

import os

import numpy as np
import pytest
import torch

from conftest import REPO, close_series
from oracle import ERROR_NAMES
from paper_2003_04617_b200 import codegen

pytestmark = pytest.mark.gpu

CASES = {"mul_acc": (["y!", "a", "b"], {}, True), "sink": (["out!", "x", "y"], {"n": 3}, False),
         "wloop": (["acc!", "x"], {"n": 5}, True),
         "prims": (["a!", "b!", "c!", "th"], {"n!": 3}, False),
         "loose": (["y!", "x"], {}, True),
         "xorfold": (["y!", "x"], {"n": 5, "m!": 6}, True)}


def src(name):
    return open(os.path.join(REPO, "tests", "golden", "codegen", name + ".rnl")).read()


@pytest.mark.parametrize("fn", list(CASES))
def test_generated_kernel_matches_reference(cuda, golden, fn):
    floats, ints, exact = CASES[fn]
    g = golden("codegen")
    X, P, G, E = g[fn + "_x"], g[fn + "_primal"], g[fn + "_grad"], g[fn + "_err"]
    k = codegen.compile_function(src(fn), fn, int_params=tuple(ints))
    assert k.floats == floats
    inputs = {nm: torch.as_tensor(X[:, j].copy(), device=cuda) for j, nm in enumerate(floats)}
    inputs.update(ints)
    primal, grads, fail = k.gradient(inputs)
    torch.cuda.synchronize()
    names = np.array([ERROR_NAMES[int(c)] for c in fail.cpu().numpy()])
    assert np.array_equal(names, E)
    ok = E == ""
    for j, nm in enumerate(floats):
        p = primal[nm].cpu().numpy()[ok]
        d = grads[nm].cpu().numpy()[ok]
        if exact:
            assert np.array_equal(p, P[ok, j]) and np.array_equal(d, G[ok, j]), nm
        else:
            assert np.allclose(p, P[ok, j], rtol=1e-12, atol=1e-13), nm
            assert np.allclose(d, G[ok, j], rtol=1e-12, atol=1e-13), nm


def test_generic_besselj_matches_reference_and_handwritten(cuda, golden):
    """programs/besselj.rnl through the generic compiler: the reference's J
    and dJ/dz (and the hand-written kernel's) on configs[0]'s 1,000 z."""
    import paper_2003_04617_b200 as rg
    g = golden("bessel")
    m = g["nu"] == 2
    z = g["z"][m]
    k = codegen.compile_function(open(os.path.join(REPO, "paper_2003_04617_b200", "programs",
                                                   "besselj.rnl")).read(),
                                 "besselj", int_params=("nu",))
    zt = torch.as_tensor(z, device=cuda)
    primal, grads, fail = k.gradient({"out!": 0.0, "z": zt, "nu": 2})
    hw = rg.besselj_grad(zt, 2)
    torch.cuda.synchronize()
    names = np.array([ERROR_NAMES[int(c)] for c in fail.cpu().numpy()])
    assert np.array_equal(names, g["err"][m])
    ok = g["err"][m] == ""
    J, dz = primal["out!"].cpu().numpy()[ok], grads["z"].cpu().numpy()[ok]
    assert close_series(J, g["J"][m][ok], 2, z[ok]).all()
    assert close_series(dz, g["dJdz"][m][ok], 2, z[ok]).all()
    assert close_series(J, hw.J.cpu().numpy()[ok], 2, z[ok]).all()


def test_generated_kernel_checks(cuda):
    """A reversibility failure is reported, not raised: a routine whose
    ancilla cannot be released (the release check is the reference's)."""
    bad = "fn leak(y!, x)\n    t <- 0.0\n    t += x\n    y! += t\n    t -> 0.0\nend\n"
    k = codegen.compile_function(bad, "leak")
    x = torch.tensor([0.0, 0.5], dtype=torch.float64, device=cuda)
    _, _, fail = k.gradient({"y!": 0.0, "x": x})
    torch.cuda.synchronize()
    assert fail.cpu().tolist() == [0, 2]                 # x = 0 releases cleanly; DirtyAncilla


@pytest.mark.parametrize("fn", list(CASES))
def test_generated_hessian_matches_reference(cuda, golden, fn):
    """The same generated code over Dual numbers: reference hessian()
    (forward-over-reverse) for every program, one launch per direction."""
    floats, ints, exact = CASES[fn]
    g = golden("codegen")
    X, H, E = g[fn + "_x"], g[fn + "_hess"], g[fn + "_hess_err"]
    k = codegen.compile_function(src(fn), fn, int_params=tuple(ints))
    inputs = {nm: torch.as_tensor(X[:, j].copy(), device=cuda) for j, nm in enumerate(floats)}
    inputs.update(ints)
    Hg, fail = k.hessian(inputs)
    torch.cuda.synchronize()
    names = np.array([ERROR_NAMES[int(c)] for c in fail.cpu().numpy()])
    assert np.array_equal(names, E)
    ok = E == ""
    Hd = Hg.cpu().numpy()[ok]
    if exact:
        assert np.array_equal(Hd, H[ok])
    else:
        assert np.allclose(Hd, H[ok], rtol=1e-11, atol=1e-12)


def test_generic_besselj_hessian_matches_reference(cuda, golden):
    from test_hess_gpu import tol_d2
    g = golden("hess")
    m = g["nu"] == 2
    z = g["z"][m][:200]
    k = codegen.compile_function(open(os.path.join(REPO, "paper_2003_04617_b200", "programs",
                                                   "besselj.rnl")).read(),
                                 "besselj", int_params=("nu",))
    Hg, fail = k.hessian({"out!": 0.0, "z": torch.as_tensor(z, device=cuda), "nu": 2})
    torch.cuda.synchronize()
    err = g["err"][m][:200]
    assert np.array_equal(np.array([ERROR_NAMES[int(c)] for c in fail.cpu().numpy()]), err)
    ok = err == ""
    ref = g["H"][m][:200][ok]
    Hd = Hg.cpu().numpy()[ok]
    assert (Hd[:, 0, :] == 0).all() and (Hd[:, :, 0] == 0).all()
    assert (np.abs(Hd[:, 1, 1] - ref[:, 1, 1]) <= tol_d2(ref[:, 1, 1], z[ok], 2)).all()
