"""The reference's own known-answer tests (pkg/tests/test_autodiff.py), run
through the drop-in API on programs written for this repository (the
generic path: codegen.py via generic.py).  Each test cites the reference
test it mirrors; the expected values are the reference tests' analytic ones."""

import math
import os
import random

import numpy as np
import pytest

import paper_2003_04617_b200 as rg
from conftest import REPO

pytestmark = pytest.mark.gpu


def src(name):
    return open(os.path.join(REPO, "tests", "golden", "codegen", name + ".rnl")).read()


def test_product_rule(cuda):
    """test_autodiff.py:21-25 (multiplier) and :68-72 (explicit wrt)."""
    primal, g = rg.gradient(src("mul_acc"), rg.GradRequest("mul_acc", [0.0, 3.0, 5.0]))
    assert primal == [15.0, 3.0, 5.0]
    assert g["a"] == 5.0 and g["b"] == 3.0 and g["y!"] == 1.0
    _, g = rg.gradient(src("mul_acc"), rg.GradRequest("mul_acc", [0.0, 3.0, 5.0], wrt=["a"]))
    assert list(g) == ["a"]


def test_jacobian_rows_and_swap_permutation(cuda):
    """test_autodiff.py:76-86."""
    J = rg.jacobian(src("mul_acc"), "mul_acc", [0.0, 3.0, 5.0])
    assert np.allclose(J, [[1, 5, 3], [0, 1, 0], [0, 0, 1]])
    J = rg.jacobian("fn f(a, b)\nSWAP(a, b)\nend\n", "f", [1.0, 2.0])
    assert np.array_equal(J, [[0, 1], [1, 0]])


def test_shared_reads_rejected_under_differentiation(cuda):
    """test_autodiff.py:51-58."""
    with pytest.raises(rg.AliasedArguments):
        rg.gradient("fn f(y, x)\ny += x * x\nend\n", rg.GradRequest("f", [0.0, 3.0]))
    _, g = rg.gradient("fn f(y, x)\ny += x ^ 2\nend\n", rg.GradRequest("f", [0.0, 3.0]))
    assert g["x"] == 6.0


def test_norm_gradient_analytic(cuda):
    """test_autodiff.py:27-34: d|x|/dx = x / |x| within 1e-9 at n = 1000."""
    rng = random.Random(2)
    x = rg.Array.vector([rng.uniform(-1, 1) for _ in range(1000)])
    before = list(x.data)
    _, g = rg.gradient(src("vlen"), rg.GradRequest("vlen", [0.0, 0.0, x]))
    nrm = math.sqrt(sum(v * v for v in x.data))
    assert max(abs(gv - xv / nrm) for gv, xv in zip(g["v"].data, x.data)) <= 1e-9
    assert x.data == before                              # the caller's Array is untouched


def test_hessians_analytic(cuda):
    """test_autodiff.py:117-140: bilinear, square, and the norm's
    (I - x^ x^T) / |x| within 1e-6 with symmetry error <= 1e-6."""
    res = rg.hessian("fn f(y, a, b)\ny += a * b\nend\n", "f", [0.0, 3.0, 5.0])
    want = np.zeros((3, 3))
    want[1, 2] = want[2, 1] = 1.0
    assert np.allclose(res.matrix, want, atol=1e-9) and res.symmetry_error <= 1e-9
    res = rg.hessian("fn f(y, x)\ny += x ^ 2\nend\n", "f", [0.0, 2.0])
    assert res.matrix[1, 1] == pytest.approx(2.0)
    rng = random.Random(5)
    x = rg.Array.vector([rng.uniform(-1, 1) for _ in range(10)])
    res = rg.hessian(src("vlen"), "vlen", [0.0, 0.0, x])
    xs = np.array(x.data)
    nrm = float(np.linalg.norm(xs))
    xh = xs / nrm
    want = (np.eye(10) - np.outer(xh, xh)) / nrm
    assert np.max(np.abs(res.matrix[2:, 2:] - want)) <= 1e-6
    assert res.symmetry_error <= 1e-6


def test_adjoint_unit_rules(cuda):
    """test_numerics.py:146-160 at the program level: out -= sqrt(x) with
    out.g = 1 gives x.g = 1/6 at x = 9; y -= a * b gives a.g = b, b.g = a."""
    _, g = rg.gradient("fn f(out!, x)\nout! += sqrt(x)\nend\n", rg.GradRequest("f", [3.0, 9.0]))
    assert g["x"] == pytest.approx(1.0 / 6.0, rel=1e-15)
    _, g = rg.gradient("fn f(y!, a, b)\ny! += a * b\nend\n", rg.GradRequest("f", [1.0, 6.0, 10.0]))
    assert g["a"] == 10.0 and g["b"] == 6.0


def _worst(g, f):
    """test_acceptance.py _compare_grad_structure: |g - f| / max(|f|, 1e-2)."""
    w = 0.0
    for p, fv in f.items():
        if fv is None or g.get(p) is None:
            continue
        a = np.ravel(np.asarray(g[p].data if hasattr(g[p], "data") else g[p], float))
        b = np.ravel(np.asarray(fv.data if hasattr(fv, "data") else fv, float))
        w = max(w, float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-2))))
    return w


@pytest.mark.parametrize("name", ["mul_acc", "sink", "wloop", "prims", "quad", "vlen"])
def test_gradient_matches_central_differences(cuda, golden, name):
    """test_acceptance.py:131-150 (criterion 4: gradient vs central
    differences, h = 1e-6, rel err < 1e-5 on 20 points) and :184-196
    (criterion 7: the arguments are untouched by every gradient call)."""
    g = golden("codegen")
    rng = np.random.default_rng(7)
    ints = {"sink": [3], "wloop": [5], "prims": [3]}.get(name, [])
    worst = 0.0
    for trial in range(20):
        if name == "quad":
            args = [float(rng.uniform(-1, 1)), rg.Array.vector(rng.uniform(-1, 1, 3).tolist()),
                    rg.Array.matrix(rng.uniform(-1, 1, (3, 3)).tolist()),
                    rg.Array.vector(rng.uniform(-1, 1, 3).tolist())]
        elif name == "vlen":
            args = [0.0, 0.0, rg.Array.vector(rng.uniform(-1, 1, 7).tolist())]
        else:
            ok = np.nonzero(g[name + "_err"] == "")[0]
            args = [float(v) for v in g[name + "_x"][ok[trial % len(ok)]]] + ints
        before = [list(a.data) if hasattr(a, "data") else a for a in args]
        _, grads = rg.gradient(src(name), rg.GradRequest(name, args))
        fd = rg.finite_difference(src(name), name, args, 1e-6)
        worst = max(worst, _worst(grads, fd))
        assert [list(a.data) if hasattr(a, "data") else a for a in args] == before
    assert worst < 1e-5, worst


def test_finite_difference_registered_programs(cuda):
    """The same check on a registered (hand-written) kernel: besselj."""
    p = rg.load_example("besselj")
    args = [0.0, 2, 3.7]
    _, g = rg.gradient(p, rg.GradRequest("besselj", args))
    fd = rg.finite_difference(p, "besselj", args, 1e-6)
    assert fd["nu"] is None and abs(g["z"] - fd["z"]) <= 1e-5 * max(abs(fd["z"]), 1e-2)
    with pytest.raises(rg.KindError):
        rg.finite_difference(p, "besselj", args, 0.0)
