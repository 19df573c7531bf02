"""codegen front end on CPU: parsing, the reverser's inversion (an
involution), routine expansion, and compile-time rejection of what the
subset does not cover."""

import os

import pytest

from conftest import REPO
from paper_2003_04617_b200 import codegen
from paper_2003_04617_b200.errors import AliasedArguments, UnsupportedProgram


def src(name):
    return open(os.path.join(REPO, "tests", "golden", "codegen", name + ".rnl")).read()


@pytest.mark.parametrize("name", ["mul_acc", "sink", "wloop"])
def test_inversion_is_an_involution(name):
    fns = codegen._Parser(src(name)).program()
    (params, body), = fns.values()
    assert codegen._invert_list(codegen._invert_list(body)) == body


def test_besselj_parses_and_expands():
    text = open(os.path.join(REPO, "paper_2003_04617_b200", "programs", "besselj.rnl")).read()
    (params, body), = codegen._Parser(text).program().values()
    assert params == ("out!", "nu", "z")
    fwd = codegen._expand(body)
    # the routine opens, the middle runs, the routine closes inverted
    assert isinstance(fwd[0], codegen.Alloc) and isinstance(fwd[-1], codegen.Dealloc)
    assert any(isinstance(s, codegen.While) for s in fwd)


def test_unsupported_constructs_are_rejected():
    for text in ("fn f(y!::array, x)\n y![1] += x\nend\n",
                 "fn f(y!, x)\n g(y!, x)\nend\n",
                 "fn f(y!, x)\n y! += 1.0fx\nend\n"):
        with pytest.raises(UnsupportedProgram):
            codegen.generate(text, "f")


def test_static_aliasing_is_rejected():
    with pytest.raises(AliasedArguments):
        codegen.generate("fn f(y!, x)\n y! += x * x\nend\n", "f")
    with pytest.raises(AliasedArguments):
        codegen.generate("fn f(y!, x)\n y! += y! * x\nend\n", "f")


def test_generated_source_compiles_for_sm100a(tmp_path, monkeypatch):
    monkeypatch.setenv("REVGPU_CODEGEN_CACHE", str(tmp_path))
    source, floats, ints = codegen.generate(src("sink"), "sink", ("n",))
    assert floats == ["out!", "x", "y"] and ints == ["n"]
    so = codegen.build(source)
    assert os.path.exists(so)
