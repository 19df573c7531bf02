"""Generic .rnl -> CUDA over fixed-shape Float array parameters (codegen.py,
SURVEY §8(f) rank 4): indexed views as targets and operands, length/size,
@safe assert, the run-time bounds and alias checks, explicit leaf-path seeds
and the Hessian over every leaf, against reference gradient() / hessian()
goldens (tests/golden/codegen_arrays.npz, oracle/gen_golden.py
codegen_arrays).  Arithmetic-only programs: bit-identical."""

import numpy as np
import pytest
import torch

from oracle import ERROR_NAMES
from paper_2003_04617_b200 import codegen
from paper_2003_04617_b200.errors import KindError
from test_codegen_gpu import src

pytestmark = pytest.mark.gpu

QUAD = {"r!": (3,), "A": (3, 3), "u": (3,)}
XSEED = [("x", (("idx", (1,)),), 1.0), ("x", (("idx", (3,)),), -0.5)]


def _inputs(k, X, cuda):
    out, b = {}, 0
    for p in k.floats:
        shp = k.shapes.get(p, ())
        m = int(np.prod(shp)) if shp else 1
        out[p] = torch.as_tensor(X[:, b:b + m].reshape((X.shape[0],) + shp).copy(), device=cuda)
        b += m
    return out


def _leaves(k, d):
    n = next(iter(d.values())).shape[0]
    return np.concatenate([d[p].reshape(n, -1).cpu().numpy() for p in k.floats], 1)


def _check(k, g, case, cuda, seeds=None, ints=None):
    X, P, G, E = (g[case + s] for s in ("_x", "_primal", "_grad", "_err"))
    inputs = _inputs(k, X, cuda)
    inputs.update(ints or {})
    primal, grads, fail = k.gradient(inputs, seeds=seeds)
    torch.cuda.synchronize()
    names = np.array([ERROR_NAMES[int(c)] for c in fail.cpu().numpy()])
    assert np.array_equal(names, E), case
    ok = E == ""
    assert np.array_equal(_leaves(k, primal)[ok], P[ok]), case
    assert np.array_equal(_leaves(k, grads)[ok], G[ok]), case
    return inputs


def test_quad_gradient_and_hessian(cuda, golden):
    g = golden("codegen_arrays")
    k = codegen.compile_function(src("quad"), "quad", array_shapes=QUAD)
    assert len(k.leaves) == 16 and k.leaves[4] == ("A", (("idx", (1, 1)),))
    inputs = _check(k, g, "quad", cuda)
    H, fail = k.hessian(inputs)
    torch.cuda.synchronize()
    assert not fail.any()
    assert np.array_equal(H.cpu().numpy(), g["quad_hess"])


def test_quad_shape_mismatch_fails_the_assert(cuda, golden):
    g = golden("codegen_arrays")
    k = codegen.compile_function(src("quad"), "quad",
                                 array_shapes={"r!": 2, "A": (3, 2), "u": 2})
    _check(k, g, "quad_bad", cuda)                       # AssertFailed for every row


def test_quad_broadcast_array_input(cuda):
    """An array given once (shape `shape`) is shared by every element."""
    k = codegen.compile_function(src("quad"), "quad", array_shapes=QUAD)
    A = np.arange(9.0).reshape(3, 3) / 10
    u = torch.rand(5, 3, dtype=torch.float64, device=cuda)
    primal, grads, fail = k.gradient({"q!": 0.0, "r!": np.zeros(3), "A": A, "u": u})
    torch.cuda.synchronize()
    At = torch.as_tensor(A, device=cuda)
    q = torch.einsum("ni,ij,nj->n", u, At, u)
    assert not fail.any() and torch.allclose(primal["q!"], q, rtol=1e-14, atol=1e-15)
    assert torch.allclose(grads["u"], u @ (At + At.T), rtol=1e-14, atol=1e-15)
    assert grads["A"].shape == (5, 3, 3)


@pytest.mark.parametrize("km", ["12", "33", "51", "24"])
def test_mix_fwd_alias_and_bounds(cuda, golden, km):
    g = golden("codegen_arrays")
    k = codegen.compile_function(src("mix"), "mix_fwd", int_params=("k", "m"),
                                 array_shapes={"x": 4})
    _check(k, g, "mix_fwd_" + km, cuda, seeds=XSEED, ints={"k": int(km[0]), "m": int(km[1])})


@pytest.mark.parametrize("km", ["12", "33", "01"])
def test_mix_grad_shared_reads(cuda, golden, km):
    """k == m passes the forward run and fails only under differentiation."""
    g = golden("codegen_arrays")
    k = codegen.compile_function(src("mix"), "mix_grad", int_params=("k", "m"),
                                 array_shapes={"x": 4})
    ints = {"k": int(km[0]), "m": int(km[1])}
    inputs = _check(k, g, "mix_grad_" + km, cuda, ints=ints)
    H, fail = k.hessian(inputs)
    torch.cuda.synchronize()
    E = g["mix_grad_" + km + "_hess_err"]
    assert np.array_equal(np.array([ERROR_NAMES[int(c)] for c in fail.cpu().numpy()]), E)
    ok = E == ""
    assert np.array_equal(H.cpu().numpy()[ok], g["mix_grad_" + km + "_hess"][ok])


def test_mix_wrong_index_count(cuda, golden):
    g = golden("codegen_arrays")
    k = codegen.compile_function(src("mix"), "mix_arity", int_params=("k",),
                                 array_shapes={"x": 4})
    _check(k, g, "mix_arity", cuda, ints={"k": 1})


def test_array_seeds_and_defaults(cuda):
    k = codegen.compile_function(src("mix"), "mix_fwd", int_params=("k", "m"),
                                 array_shapes={"x": 4})
    x = torch.rand(3, 4, dtype=torch.float64, device=cuda)
    with pytest.raises(KindError):                       # first argument is not scalar
        k.gradient({"x": x, "k": 1, "m": 2})
    with pytest.raises(KindError):
        k.gradient({"x": x, "k": 1, "m": 2}, seeds=[("x", (("idx", (9,)),), 1.0)])
    _, grads, fail = k.gradient({"x": x, "k": 1, "m": 2}, seeds=[("x", (("idx", (1,)),), 1.0)])
    torch.cuda.synchronize()
    # x[1] += x[2]: d x1_out / d x = e1 + e2
    assert not fail.any()
    assert torch.equal(grads["x"], torch.tensor([[1.0, 1.0, 0, 0]] * 3, dtype=torch.float64,
                                                device=cuda))
