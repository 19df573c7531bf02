"""The drop-in API on functions WITHOUT a hand-written kernel: gradient,
gradient_batch, jacobian, hessian, run, uncall and check_reversibility
(reference autodiff.py / interpreter.py signatures) compile the function with
codegen.py (generic.py) and run it on the device.  Against the reference
interpreter's own outputs on the same calls (tests/golden/codegen*.npz,
oracle/gen_golden.py codegen / codegen_arrays / codegen_dropin)."""

import os

import numpy as np
import pytest
import torch

import paper_2003_04617_b200 as rg
from conftest import REPO
from oracle import ERROR_NAMES

pytestmark = pytest.mark.gpu


def src(name):
    return open(os.path.join(REPO, "tests", "golden", "codegen", name + ".rnl")).read()


def close(a, b, rel=1e-12, floor=1e-14):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.all(np.abs(a - b) <= rel * np.abs(b) + floor)


def test_gradient_and_jacobian_of_an_unregistered_program(cuda, golden):
    g = golden("codegen")
    prog = rg.parse_program(src("prims"))
    assert prog.functions["prims"].kernel is None
    for i in range(8):
        args = [float(v) for v in g["prims_x"][i]] + [3]
        primal, grads = rg.gradient(prog, rg.GradRequest("prims", args))
        assert close(primal[:4], g["prims_primal"][i]) and primal[4] == 3
        assert close([grads[p] for p in ("a!", "b!", "c!", "th")], g["prims_grad"][i])
        assert grads["n!"] is None                          # Int leaves carry no cotangent
    d = golden("codegen_dropin")
    J = rg.jacobian(prog, "prims", [float(v) for v in d["prims_x"][0]] + [3])
    assert close(J, d["prims_jac"])


def test_run_uncall_check_reversibility(cuda, golden):
    d = golden("codegen_dropin")
    prog = rg.parse_program(src("prims"))
    for i, row in enumerate(d["prims_x"]):
        args = [float(v) for v in row] + [3]
        mid = rg.run(prog, "prims", args)
        assert close(mid[:4], d["prims_run"][i]) and mid[4] == 3
        assert close(rg.uncall(prog, "prims", args)[:4], d["prims_uncall"][i])
        rep = rg.check_reversibility(prog, "prims", args)
        assert rep.ok and rep.max_deviation <= 1e-12


def test_arrays_through_the_public_api(cuda, golden):
    ga = golden("codegen_arrays")
    row = ga["quad_x"][0]
    args = [float(row[0]), rg.Array.vector(row[1:4].tolist()),
            rg.Array.matrix(row[4:13].reshape(3, 3).tolist()), rg.Array.vector(row[13:16].tolist())]
    primal, grads = rg.gradient(src("quad"), rg.GradRequest("quad", args))
    flat = lambda vs: [vs[0]] + [x for v in vs[1:] for x in v.data]  # noqa: E731
    assert flat(primal) == list(ga["quad_primal"][0])                  # arithmetic only: exact
    assert flat([grads[p] for p in ("q!", "r!", "A", "u")]) == list(ga["quad_grad"][0])
    assert isinstance(grads["A"], rg.Array) and grads["A"].shape == (3, 3)
    assert flat(rg.run(src("quad"), "quad", args)) == list(golden("codegen_dropin")["quad_run"])
    H = rg.hessian(src("quad"), "quad", args)
    assert np.array_equal(H.matrix, ga["quad_hess"][0]) and H.symmetry_error >= 0.0


def test_device_errors_raise_the_reference_classes(cuda):
    x = rg.Array.vector([0.5, 1.5, -0.25, 2.0])
    seeds = [("x", (("idx", (1,)),), 1.0)]
    with pytest.raises(rg.AliasedArguments):
        rg.gradient(src("mix"), rg.GradRequest("mix_fwd", [x, 3, 3], seeds=seeds))
    with pytest.raises(rg.IndexOutOfBounds):
        rg.run(src("mix"), "mix_fwd", [x, 5, 1])
    with pytest.raises(rg.KindError):                  # default seed: x is not scalar
        rg.gradient(src("mix"), rg.GradRequest("mix_fwd", [x, 1, 2]))
    out = rg.run(src("mix"), "mix_fwd", [x, 1, 2])
    assert out[0].data == [2.0, 1.5, -0.25, 2.0] and out[1:] == [1, 2]
    # the shared-read alias fires only under differentiation
    y = rg.run(src("mix"), "mix_grad", [0.0, x, 3, 3])
    assert y[0] == 0.0625
    with pytest.raises(rg.AliasedArguments):
        rg.gradient(src("mix"), rg.GradRequest("mix_grad", [0.0, x, 3, 3]))


def test_gradient_batch_generic(cuda, golden):
    g = golden("codegen")
    X, P, G, E = g["prims_x"], g["prims_primal"], g["prims_grad"], g["prims_err"]
    names = ["a!", "b!", "c!", "th"]
    inputs = {nm: torch.as_tensor(X[:, j].copy(), device=cuda) for j, nm in enumerate(names)}
    inputs["n!"] = 3
    primal, grads, restored, codes = rg.gradient_batch(src("prims"), "prims", inputs,
                                                       return_codes=True)
    torch.cuda.synchronize()
    assert np.array_equal(np.array([ERROR_NAMES[int(c)] for c in codes.cpu().numpy()]), E)
    ok = restored.cpu().numpy()
    assert ok.all() == (E == "").all()
    for j, nm in enumerate(names):
        assert close(primal[nm].cpu().numpy()[ok], P[ok, j])
        assert close(grads[nm].cpu().numpy()[ok], G[ok, j])
    assert "n!" not in grads


def test_readme_rotation_example(cuda):
    """ROT's adjoint (numerics.py _rot_adjoint) against the analytic
    derivatives of p' = p cos t - q sin t, seeded on p!."""
    import math
    src_ = "fn turn(p!, q!, ang)\n    ROT(p!, q!, ang)\nend\n"
    p, q, t = 1.0, 0.5, 0.3
    out, g = rg.gradient(src_, rg.GradRequest("turn", [p, q, t]))
    assert abs(out[0] - (p * math.cos(t) - q * math.sin(t))) <= 1e-15
    assert abs(out[1] - (p * math.sin(t) + q * math.cos(t))) <= 1e-15
    assert abs(g["p!"] - math.cos(t)) <= 1e-15 and abs(g["q!"] + math.sin(t)) <= 1e-15
    assert abs(g["ang"] - (-p * math.sin(t) - q * math.cos(t))) <= 1e-15
    k = rg.compile_function(src_, "turn")
    z = torch.linspace(0.1, 2.0, 64, dtype=torch.float64, device=cuda)
    primal, grads, fail = k.gradient({"p!": z, "q!": q, "ang": t})
    torch.cuda.synchronize()
    assert not fail.any()
    assert torch.allclose(grads["ang"], -z * math.sin(t) - q * math.cos(t), rtol=1e-14, atol=0)


def test_gradient_batch_generic_arrays(cuda, golden):
    """Batched array inputs: (n, *shape) tensors, one row per call, against
    the reference's per-row gradient() of quad.rnl (bit-exact)."""
    ga = golden("codegen_arrays")
    X = ga["quad_x"]
    n = X.shape[0]
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=cuda)  # noqa: E731
    inputs = {"q!": t(X[:, 0]), "r!": t(X[:, 1:4]), "A": t(X[:, 4:13].reshape(n, 3, 3)),
              "u": t(X[:, 13:16])}
    primal, grads, restored = rg.gradient_batch(src("quad"), "quad", inputs)
    torch.cuda.synchronize()
    assert restored.all()
    flat = lambda d: torch.cat([d[p].reshape(n, -1) for p in ("q!", "r!", "A", "u")], 1)  # noqa
    assert np.array_equal(flat(primal).cpu().numpy(), ga["quad_primal"])
    assert np.array_equal(flat(grads).cpu().numpy(), ga["quad_grad"])


def test_gmm_wider_than_the_tiles_goes_generic(cuda, oracle):
    """d > 128 is beyond the hand-written GMM tiles (gmm.cu): the drop-in
    gradient runs the generic compiler's kernel of the same program and
    matches the oracle (the reference takes any d)."""
    d, K, N = 130, 2, 3
    rng = np.random.default_rng(5)
    alphas, means = rng.normal(0, 1, K), rng.uniform(0, 1, (K, d))
    icf, x = rng.normal(0, 0.3, (K, d * (d + 1) // 2)), rng.uniform(0, 1, (N, d))
    rc, e, ga, gm, gi = oracle.gmm_grad(alphas, means, icf, x, 1.0, 0, 0.5)
    assert rc == 0
    A = lambda a: rg.Array.matrix(a.tolist()) if a.ndim == 2 else rg.Array.vector(a.tolist())  # noqa
    Z = lambda *s: A(np.zeros(s))  # noqa: E731
    args = [0.0, A(alphas), A(means), A(icf), A(x), Z(K, d), Z(K), Z(d), Z(d), Z(K),
            rg.Array.vector([0] * K), 1.0, 0, 0.5]
    primal, g = rg.gradient(rg.load_example("gmm"), rg.GradRequest("gmm", args,
                                                                    wrt=["alphas", "icf"]))
    assert abs(primal[0] - e) <= 1e-12 * abs(e)
    assert np.allclose(np.array(g["alphas"].data), ga, rtol=1e-10, atol=1e-12)
    assert np.allclose(np.array(g["icf"].data).reshape(K, -1), gi, rtol=1e-9,
                       atol=1e-12 * np.max(np.abs(gi)))
