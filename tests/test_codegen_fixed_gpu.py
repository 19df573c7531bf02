"""Fixed (Q31.32) cells in generated kernels (codegen.py kind "x"): the
reference's Fixed semantics (values.py:28-86, numerics.py:305-306, 419-428)
— raw int64 cells, + / - wrapping mod 2^64, from_real rounding half-even,
Fixed cotangents quantized at every accumulation — on tests/golden/codegen/
fxmix.rnl against the reference (codegen_fixed.npz: run, uncall, gradient
with the default Fixed seed and a Float seed, finite_difference with the
measured Fixed step), through the drop-in API with the package's own Fixed.

Bit-exact: every Fixed raw value, Float and finite difference equals the
reference's (tools/fixed_parity_count.py counts them; the device exp / log
reproduce the host libm on these arguments)."""
import numpy as np
import pytest

import paper_2003_04617_b200 as rg

pytestmark = pytest.mark.gpu


def src():
    import os
    return open(os.path.join(os.path.dirname(__file__), "golden", "codegen", "fxmix.rnl")).read()


def f64(bits):
    return float(np.int64(bits).view(np.float64))


def fclose(a, b):
    return a == b


def case_args(g, r):
    a0, y0, b = g["cases"][r]
    return [rg.Fixed.from_real(a0), float(y0), rg.Fixed.from_real(b), int(g["k"][r])]


def call(fn):
    try:
        return fn(), ""
    except Exception as err:  # noqa: BLE001
        return None, type(err).__name__


def test_fixed_run_and_uncall_against_the_reference(cuda, golden):
    g = golden("codegen_fixed")
    exact = 0
    for tag, fn in (("run", rg.run), ("uncall", rg.uncall)):
        for r in range(len(g["k"])):
            out, err = call(lambda: fn(src(), "fxmix", case_args(g, r)))
            assert err == g[tag + "_err"][r], (tag, r, err)
            if err:
                continue
            acc, y, b = g[tag][r]
            assert isinstance(out[0], rg.Fixed) and isinstance(out[2], rg.Fixed)
            assert out[2].raw == b and out[3] == int(g["k"][r])
            assert out[0].raw == acc, (tag, r, out[0].raw, acc)
            assert fclose(out[1], f64(y)), (tag, r)
            exact += 1
    assert exact >= 60


def test_fixed_gradient_against_the_reference(cuda, golden):
    g = golden("codegen_fixed")
    for tag, seeds in (("gacc", None), ("gy", [("y!", (), 1.0)])):
        for r in range(len(g["k"])):
            res, err = call(lambda: rg.gradient(src(), rg.GradRequest("fxmix", case_args(g, r),
                                                                      seeds=seeds)))
            assert err == g[tag + "_err"][r], (tag, r, err)
            if err:
                continue
            prim, grads = res
            acc, y, b, ga, gy, gb = g[tag][r]
            assert prim[0].raw == acc and prim[2].raw == b
            assert fclose(prim[1], f64(y))
            assert isinstance(grads["acc!"], rg.Fixed) and isinstance(grads["b"], rg.Fixed)
            assert grads["acc!"].raw == ga and grads["k"] is None
            assert fclose(grads["y!"], f64(gy))
            assert grads["b"].raw == gb, (tag, r, grads["b"].raw, gb)


def test_fixed_finite_difference_against_the_reference(cuda, golden):
    """finite_difference over a Fixed leaf divides by the step actually taken
    after Q31.32 quantization (autodiff.py:299-301)."""
    g = golden("codegen_fixed")
    for r in range(len(g["k"])):
        fd, err = call(lambda: rg.finite_difference(src(), "fxmix", case_args(g, r), 1e-6))
        assert err == g["fd_err"][r], (r, err)
        if err:
            continue
        for got, want in zip((fd["acc!"], fd["y!"], fd["b"]), g["fd"][r]):
            assert got == want, (r, got, want)
