"""Recursion and bijector-view call arguments in generated kernels
(codegen.py: recursive calls inlined level by level up to
REVGPU_CODEGEN_DEPTH, `x |> addconst(c)` / `mulconst` / `neg` arguments
copied in through the bijector and written back through its inverse,
interpreter.py:565-583, 960-989) on tests/golden/codegen/countdown.rnl,
bit-exact against the reference's run / uncall (codegen_recursion.npz)."""
import os

import numpy as np
import pytest

import paper_2003_04617_b200 as rg

pytestmark = pytest.mark.gpu


def src():
    return open(os.path.join(os.path.dirname(__file__), "golden", "codegen",
                             "countdown.rnl")).read()


def test_recursion_through_bijector_views_against_the_reference(cuda, golden):
    g = golden("codegen_recursion")
    for i, n in enumerate(g["n"]):
        assert rg.run(src(), "chain", [0, int(n)]) == list(g["chain_run"][i])
        assert rg.uncall(src(), "chain", [100, int(n)]) == list(g["chain_uncall"][i])
    for i, k in enumerate(g["k"]):
        assert rg.run(src(), "tri", [7, int(k)]) == list(g["tri_run"][i])


def test_recursion_past_the_inlined_depth_is_a_recursion_error(cuda):
    """tri(k) recurses k levels: past the compiled depth (24 by default) the
    generated kernel reports Python's RecursionError instead of a result."""
    with pytest.raises(RecursionError):
        rg.run(src(), "tri", [0, 40])


def test_bijector_write_back_that_does_not_divide_is_a_kind_error(cuda):
    """numerics._div_const: an Int write-back through mulconst must divide."""
    text = ("fn bump(a)\n    a += 1\nend\n\n"
            "fn f(x)\n    bump(x |> mulconst(2))\nend\n")
    with pytest.raises(rg.KindError):
        rg.run(text, "f", [3])
