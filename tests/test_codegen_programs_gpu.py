"""The paper's three benchmark programs through the GENERIC compiler
(codegen.py): programs/ba.rnl (calls rodrigues —
inlined — over Float array parameters), programs/gmm.rnl (Int array scratch,
INC, argmax branches, routines in loops) and programs/besselj.rnl (in
test_codegen_gpu.py), compiled from their .rnl source with no hand-written
kernel, against the reference's own gradient() goldens (tests/golden/ba.npz,
gmm.npz) and hessian() goldens (codegen_programs.npz).  Transcendental
programs: libdevice vs host libm (<= 1-2 ulp per call), so tolerances as the
hand-written kernels' parity tests."""

import os

import numpy as np
import pytest
import torch

from conftest import REPO
from paper_2003_04617_b200 import codegen

pytestmark = pytest.mark.gpu


def prog(name):
    return open(os.path.join(REPO, "paper_2003_04617_b200", "programs", name + ".rnl")).read()


def close(a, b, rel, floor):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b) <= rel * np.abs(b) + floor * max(np.abs(b).max(), 1e-300)


def gmm_case(G, ci, n=1):
    pre = f"c{ci}_"
    d, K, N, m = (int(v) for v in G[pre + "dims"])
    P = d * (d + 1) // 2
    shapes = {"alphas": K, "means": (K, d), "icf": (K, P), "x": (N, d), "qd!": (K, d), "sq!": K,
              "xc!": d, "qxc!": d, "mt!": K, "dm!": K}
    inputs = {"err!": 0.0, "alphas": G[pre + "alphas"], "means": G[pre + "means"],
              "icf": G[pre + "icf"], "qd!": np.zeros((K, d)), "sq!": np.zeros(K),
              "xc!": np.zeros(d), "qxc!": np.zeros(d), "mt!": np.zeros(K),
              "dm!": np.zeros(K, np.int64), "ga": float(G[pre + "gamma"]), "wm": m,
              "cst": float(G[pre + "cst"])}
    x = torch.as_tensor(G[pre + "x"], device="cuda")
    inputs["x"] = x.expand(n, N, d).contiguous() if n > 1 else G[pre + "x"]
    return shapes, inputs


@pytest.mark.parametrize("ci", range(8))
def test_generic_gmm_matches_reference(cuda, golden, ci):
    G = golden("gmm")
    shapes, inputs = gmm_case(G, ci, n=2)
    k = codegen.compile_function(prog("gmm"), "gmm", int_params=("dm!", "wm"),
                                 array_shapes=shapes)
    primal, grads, fail = k.gradient(inputs)
    torch.cuda.synchronize()
    assert not fail.any()
    pre = f"c{ci}_"
    err = primal["err!"].cpu().numpy()
    assert close(err, np.full(2, float(G[pre + "err"])), 1e-12, 0).all()
    for nm in ("alphas", "means", "icf"):
        g = grads[nm].cpu().numpy()
        for r in range(2):
            assert close(g[r], G[pre + "g_" + nm], 1e-10, 1e-12).all(), nm
    # the scratch comes back zero up to round-off (the routines uncompute it,
    # as in the reference) and x is untouched
    assert primal["mt!"].abs().max().item() <= 1e-12 and torch.equal(primal["x"], inputs["x"])


def test_generic_gmm_hessian(cuda, golden):
    G = golden("gmm")
    shapes, inputs = gmm_case(G, 5)
    k = codegen.compile_function(prog("gmm"), "gmm", int_params=("dm!", "wm"),
                                 array_shapes=shapes)
    assert len(k.leaves) == 27
    H, fail = k.hessian(inputs)
    torch.cuda.synchronize()
    assert not fail.any()
    ref = golden("codegen_programs")["gmm_c5_hess"]
    assert close(H[0].cpu().numpy(), ref, 1e-10, 1e-12).all()


def _ba_inputs(B, cuda, rows=slice(None)):
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a[rows]), device=cuda)  # noqa: E731
    return {"e1!": 0.0, "e2!": 0.0, "cam": t(B["cams"]), "X": t(B["X"]), "w": t(B["w"]),
            "f1": t(B["feat"][:, 0]), "f2": t(B["feat"][:, 1])}


def test_generic_ba_jacobian_matches_reference(cuda, golden):
    B = golden("ba")
    k = codegen.compile_function(prog("ba"), "ba_proj", array_shapes={"cam": 11, "X": 3})
    inputs = _ba_inputs(B, cuda)
    for r, seed in enumerate(("e1!", "e2!")):
        primal, grads, fail = k.gradient(inputs, seeds=[(seed, (), 1.0)])
        torch.cuda.synchronize()
        assert not fail.any()
        J = torch.cat([grads["cam"], grads["X"], grads["w"][:, None]], 1).cpu().numpy()
        ref = B["J"][:, r, :]
        for o in range(J.shape[0]):
            assert close(J[o], ref[o], 1e-11, 1e-13).all(), (seed, o)
        e = primal[seed].cpu().numpy()
        assert close(e, B["e"][:, r], 1e-12, 1e-14).all()
    kw = codegen.compile_function(prog("ba"), "ba_weight")
    _, g, fail = kw.gradient({"e!": 0.0, "w": inputs["w"]})
    torch.cuda.synchronize()
    assert not fail.any() and np.array_equal(g["w"].cpu().numpy(), B["wjac"])


def test_generic_ba_hessian(cuda, golden):
    B = golden("ba")
    k = codegen.compile_function(prog("ba"), "ba_proj", array_shapes={"cam": 11, "X": 3})
    H, fail = k.hessian(_ba_inputs(B, cuda, slice(0, 4)))
    torch.cuda.synchronize()
    assert not fail.any()
    ref = golden("codegen_programs")["ba_hess"]
    for o in range(4):
        assert close(H[o].cpu().numpy(), ref[o], 1e-9, 1e-11).all(), o


def test_nbody_nested_calls_bit_exact(cuda, golden):
    """tests/golden/codegen/nbody.rnl: kick -> pull calls whose view
    arguments vel![a, c] are indexed by the loop variable a passed alongside
    (inlined: pull never writes a), 2-d arrays, a routine in the callee.
    Only + - * / sqrt: correctly rounded on both sides, so the batched
    gradient, run and uncall equal the reference interpreter bit for bit."""
    from test_codegen_gpu import src
    g = golden("codegen_nbody")
    X = g["x"]
    n = X.shape[0]
    k = codegen.compile_function(src("nbody"), "nbody", int_params=("steps",),
                                 array_shapes={"pos!": (4, 3), "vel!": (4, 3), "mass": 4})
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=cuda)  # noqa: E731
    inputs = {"pos!": t(X[:, :12].reshape(n, 4, 3)), "vel!": t(X[:, 12:24].reshape(n, 4, 3)),
              "mass": t(X[:, 24:28]), "h": t(X[:, 28]), "steps": 3}
    seeds = [("pos!", (("idx", (1, 1)),), 1.0), ("vel!", (("idx", (2, 3)),), 0.5)]
    primal, grads, fail = k.gradient(inputs, seeds=seeds)
    out, rfail = k.run(inputs, 1)
    back, ufail = k.run(inputs, -1)
    torch.cuda.synchronize()
    assert not fail.any() and not rfail.any() and not ufail.any()
    flat = lambda d, names: torch.cat([d[p].reshape(n, -1) for p in names], 1).cpu().numpy()  # noqa
    assert np.array_equal(flat(primal, ["pos!", "vel!"]), g["primal"])
    assert np.array_equal(flat(grads, ["pos!", "vel!", "mass", "h"]), g["grad"])
    assert np.array_equal(flat(out, ["pos!", "vel!"]), g["run"])
    assert np.array_equal(flat(back, ["pos!", "vel!"]), g["uncall"])


def test_random_programs_against_the_reference(cuda, golden):
    """Differential test: 80 random reversible programs (oracle/gen_golden.py
    random_program: instructions over distinct operands, counted loops,
    branches with SAME postconditions, ancilla blocks, SWAP / ROT; half with
    log-domain ancillas and counted while loops) compiled
    by codegen.py, against the reference's gradient() on 6 inputs each:
    error classes exact, values within 1e-12 (libdevice sin/cos/sqrt ulps)."""
    from oracle import ERROR_NAMES
    g = golden("codegen_random")
    X, P, G, E = g["x"], g["primal"], g["grad"], g["err"]
    for q, text in enumerate(g["texts"]):
        k = codegen.compile_function(str(text), f"r{q}", int_params=("n",))
        for r in range(6 * q, 6 * q + 6):          # n varies per row: one launch per row
            inputs = {nm: float(X[r, j]) for j, nm in enumerate(("y!", "a", "b", "c"))}
            inputs["n"] = int(X[r, 4])
            primal, grads, fail = k.gradient(inputs)
            name = ERROR_NAMES[int(fail[0].item())]
            assert name == E[r], (q, r, text)
            if name:
                continue
            got_p = [primal[c][0].item() for c in ("y!", "a", "b", "c")]
            got_g = [grads[c][0].item() for c in ("y!", "a", "b", "c")]
            assert close(got_p, P[r], 1e-12, 1e-14).all(), (q, r, text)
            assert close(got_g, G[r], 1e-12, 1e-14).all(), (q, r, text)


def test_registered_programs_full_jacobian_and_hessian(cuda, golden):
    """The drop-in jacobian / hessian of the registered gmm and ba_proj
    functions: their hand-written kernels do not produce these, the generic
    compiler does (reference hessian() goldens: codegen_programs.npz)."""
    import paper_2003_04617_b200 as rg
    G = golden("gmm")
    pre = "c5_"
    d, K, N, m = (int(v) for v in G[pre + "dims"])
    A = lambda a: rg.Array.matrix(a.tolist()) if a.ndim == 2 else rg.Array.vector(a.tolist())  # noqa
    Z = lambda *s: A(np.zeros(s))  # noqa: E731
    args = [0.0, A(G[pre + "alphas"]), A(G[pre + "means"]), A(G[pre + "icf"]), A(G[pre + "x"]),
            Z(K, d), Z(K), Z(d), Z(d), Z(K), rg.Array.vector([0] * K), float(G[pre + "gamma"]), m,
            float(G[pre + "cst"])]
    p = rg.load_example("gmm")
    res = rg.hessian(p, "gmm", args)
    assert close(res.matrix, golden("codegen_programs")["gmm_c5_hess"], 1e-10, 1e-12).all()
    J = rg.jacobian(p, "gmm", args)
    assert J.shape == (27, 27)
    # row 0 (seed err!) restricted to alphas / means / icf is the gradient
    assert close(J[0, 1:1 + K], G[pre + "g_alphas"], 1e-10, 1e-12).all()
    B = golden("ba")
    o = 0
    bargs = [0.0, 0.0, rg.Array.vector(B["cams"][o].tolist()), rg.Array.vector(B["X"][o].tolist()),
             float(B["w"][o]), float(B["feat"][o, 0]), float(B["feat"][o, 1])]
    res = rg.hessian(rg.load_example("ba_proj"), "ba_proj", bargs)
    assert close(res.matrix, golden("codegen_programs")["ba_hess"][o], 1e-9, 1e-11).all()


def test_gradient_batch_of_gmm_problems(cuda, golden):
    """gradient_batch on the registered gmm: a batch of independent problems
    (here the reference case c0, twice, with x perturbed in the second row)
    through the generic kernel; row 0 equals the reference's gradient()."""
    import paper_2003_04617_b200 as rg
    G = golden("gmm")
    pre = "c0_"
    d, K, N, m = (int(v) for v in G[pre + "dims"])
    P = d * (d + 1) // 2
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=cuda)  # noqa: E731
    x2 = np.stack([G[pre + "x"], G[pre + "x"] * 0.9])
    inputs = {"err!": t(np.zeros(2)), "alphas": G[pre + "alphas"], "means": G[pre + "means"],
              "icf": G[pre + "icf"], "x": t(x2), "qd!": np.zeros((K, d)), "sq!": np.zeros(K),
              "xc!": np.zeros(d), "qxc!": np.zeros(d), "mt!": np.zeros(K),
              "dm!": np.zeros(K, np.int64), "ga": float(G[pre + "gamma"]), "wm": m,
              "cst": float(G[pre + "cst"])}
    primal, grads, restored = rg.gradient_batch(rg.load_example("gmm"), "gmm", inputs,
                                                wrt=["alphas", "means", "icf"])
    torch.cuda.synchronize()
    assert restored.all() and grads["icf"].shape == (2, K, P)
    assert close(primal["err!"].cpu().numpy()[:1], [float(G[pre + "err"])], 1e-12, 0).all()
    for nm in ("alphas", "means", "icf"):
        assert close(grads[nm][0].cpu().numpy(), G[pre + "g_" + nm], 1e-10, 1e-12).all()
    assert not torch.equal(grads["means"][0], grads["means"][1])


def test_complex_parameters_against_the_reference(cuda, golden):
    """tests/golden/codegen/polar.rnl: Complex parameters (two Float leaves),
    field views as targets / operands / a ROT angle, abs2 and angle of a
    Complex operand; batched gradient with seeds on y!.re and y!.im, and the
    Hessian, against the reference (codegen_complex.npz)."""
    from oracle import ERROR_NAMES
    from test_codegen_gpu import src
    g = golden("codegen_complex")
    X = g["x"]
    k = codegen.compile_function(src("polar"), "polar", complex_params=("y!", "x"))
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=cuda)  # noqa: E731
    inputs = {"y!": t(X[:, 0] + 1j * X[:, 1]), "x": t(X[:, 2] + 1j * X[:, 3]),
              "p!": t(X[:, 4]), "q!": t(X[:, 5])}
    for tag in ("re", "im"):
        primal, grads, fail = k.gradient(inputs, seeds=[("y!", (("field", tag),), 1.0)])
        torch.cuda.synchronize()
        names = np.array([ERROR_NAMES[int(c)] for c in fail.cpu().numpy()])
        assert np.array_equal(names, g["err_" + tag])
        ok = names == ""
        P = torch.stack([primal["y!"].real, primal["y!"].imag, primal["x"].real,
                         primal["x"].imag, primal["p!"], primal["q!"]], 1).cpu().numpy()
        G = torch.stack([grads["y!"].real, grads["y!"].imag, grads["x"].real, grads["x"].imag,
                         grads["p!"], grads["q!"]], 1).cpu().numpy()
        for r in np.nonzero(ok)[0]:
            assert close(P[r], g["primal_" + tag][r], 1e-12, 1e-14).all(), (tag, r)
            assert close(G[r], g["grad_" + tag][r], 1e-12, 1e-14).all(), (tag, r)
    H, fail = k.hessian(inputs)
    torch.cuda.synchronize()
    for r in range(X.shape[0]):
        if g["hess_err"][r] == "":
            assert fail[r].item() == 0
            assert close(H[r].cpu().numpy(), g["hess"][r], 1e-10, 1e-12).all(), r
        else:
            assert fail[r].item() != 0                  # the reference raised too


def test_complex_through_the_dropin_api(cuda, golden):
    """gradient() with the reference's own Complex values round-trips the
    Complex containers (default seed: the real part of the first argument)."""
    import sys
    import paper_2003_04617_b200 as rg
    from test_codegen_gpu import src

    class Complex:                                      # the reference's container shape
        def __init__(self, re, im):
            self.re, self.im = re, im
    g = golden("codegen_complex")
    row = g["x"][0]
    args = [Complex(row[0], row[1]), Complex(row[2], row[3]), float(row[4]), float(row[5])]
    primal, grads = rg.gradient(src("polar"), rg.GradRequest("polar", args))
    assert isinstance(primal[0], Complex) and isinstance(grads["x"], Complex)
    got = [grads["y!"].re, grads["y!"].im, grads["x"].re, grads["x"].im, grads["p!"], grads["q!"]]
    assert close(got, g["grad_re"][0], 1e-12, 1e-14).all()
    del sys


def test_complex_finite_difference_against_the_reference(cuda, golden):
    """finite_difference() with Complex arguments (re / im leaves, default
    seed y!.re, explicit y!.im seed) against the reference's own
    finite_difference (codegen_complex_fd.npz, h = 1e-6).  Both difference
    the same binary64 program at the same steps; the device's libdevice
    sin / cos / log differ from the host libm by <= 1-2 ulp, amplified by
    1 / (2h) = 5e5: the bar is 1e-8 absolute + 1e-8 relative."""
    import paper_2003_04617_b200 as rg
    from test_codegen_gpu import src

    class Complex:
        def __init__(self, re, im):
            self.re, self.im = re, im
    g = golden("codegen_complex")
    f = golden("codegen_complex_fd")
    for j, i in enumerate(f["rows"]):
        row = g["x"][i]
        args = [Complex(row[0], row[1]), Complex(row[2], row[3]), float(row[4]), float(row[5])]
        for tag, seeds in (("re", None), ("im", [("y!", (("field", "im"),), 1.0)])):
            fd = rg.finite_difference(src("polar"), "polar", args, float(f["h"]), seeds=seeds)
            assert isinstance(fd["x"], Complex)
            got = [fd["y!"].re, fd["y!"].im, fd["x"].re, fd["x"].im, fd["p!"], fd["q!"]]
            assert close(got, f["fd_" + tag][j], 1e-8, 1e-8).all(), (tag, i, got)
