"""gradient_batch: row i equals gradient(program,
GradRequest(fname, args_i, seeds, wrt)) bit for bit (same kernels), failing
rows are flagged in `restored` with the revlang error code, never raised."""

import numpy as np
import pytest
import torch

import paper_2003_04617_b200 as rg
from paper_2003_04617_b200.errors import error_for_code
from paper_2003_04617_b200.values import to_numpy

pytestmark = pytest.mark.gpu


def test_besselj_rows_match_gradient(cuda):
    p = rg.load_example("besselj")
    rng = np.random.default_rng(3)
    z = rng.uniform(0.1, 10.0, 64)
    z[5], z[9] = -1.0, 25.0                               # RevDomainError, DirtyAncilla
    out0 = rng.normal(size=64)
    for seeds in (None, [("out!", (), 2.5), ("z", (), 0.25)]):
        primal, grads, restored, code = rg.gradient_batch(
            p, "besselj", {"out!": torch.as_tensor(out0, device=cuda), "nu": 2,
                           "z": torch.as_tensor(z, device=cuda)}, seeds=seeds, return_codes=True)
        assert set(grads) == {"out!", "z"}
        for i in range(64):
            args = [float(out0[i]), 2, float(z[i])]
            try:
                pr, g = rg.gradient(p, rg.GradRequest("besselj", args, seeds=seeds))
            except rg.RevLangError as err:
                assert not bool(restored[i])
                assert type(error_for_code(int(code[i]), "")) is type(err)
                continue
            assert bool(restored[i])
            assert float(primal["out!"][i]) == pr[0]
            assert float(grads["z"][i]) == g["z"] and float(grads["out!"][i]) == g["out!"]


def test_ba_rows_match_gradient(cuda):
    from test_ba_gpu import ba_inputs
    p = rg.load_example("ba_proj")
    rng = np.random.default_rng(4)
    cams, X, w, feats, obs = ba_inputs(rng, 40, 40, 40, shuffle=False)
    t = lambda a: torch.as_tensor(a, device=cuda)        # noqa: E731
    inp = {"cam": t(cams), "X": t(X), "w": t(w), "f1": t(feats[:, 0]), "f2": t(feats[:, 1])}
    for seeds in (None, [("e2!", (), 1.0)]):
        primal, grads, restored = rg.gradient_batch(p, "ba_proj", inp, seeds=seeds,
                                                    wrt=["cam", "X", "w"])
        assert restored.all()
        for i in range(0, 40, 7):
            args = [0.0, 0.0, rg.Array.vector(cams[i].tolist()), rg.Array.vector(X[i].tolist()),
                    float(w[i]), float(feats[i, 0]), float(feats[i, 1])]
            pr, g = rg.gradient(p, rg.GradRequest("ba_proj", args, seeds=seeds,
                                                  wrt=["cam", "X", "w"]))
            assert np.array_equal(grads["cam"][i].cpu().numpy(), to_numpy(g["cam"], "cam"))
            assert np.array_equal(grads["X"][i].cpu().numpy(), to_numpy(g["X"], "X"))
            assert float(grads["w"][i]) == g["w"]
            assert float(primal["e1!"][i]) == pr[0] and float(primal["e2!"][i]) == pr[1]
    pw, gw, rw = rg.gradient_batch(p, "ba_weight", {"w": t(w)})
    for i in range(0, 40, 9):
        pr, g = rg.gradient(p, rg.GradRequest("ba_weight", [0.0, float(w[i])]))
        assert float(gw["w"][i]) == g["w"] and float(pw["e!"][i]) == pr[0]


def test_gmm_is_rejected(cuda):
    with pytest.raises(rg.KindError):
        rg.gradient_batch(rg.load_example("gmm"), "gmm", {})
