"""codegen front end on CPU: parsing, the reverser's inversion (an
involution), routine expansion, and compile-time rejection of what the
subset does not cover."""

import os

import pytest

from conftest import REPO
from paper_2003_04617_b200 import codegen
from paper_2003_04617_b200.errors import KindError, UnsupportedProgram


def src(name):
    return open(os.path.join(REPO, "tests", "golden", "codegen", name + ".rnl")).read()


@pytest.mark.parametrize("name", ["mul_acc", "sink", "wloop", "quad", "mix", "prims", "vlen", "loose", "xorfold",
                                  "polar"])
def test_inversion_is_an_involution(name):
    for params, body in codegen._Parser(src(name)).program().values():
        assert codegen._invert_list(codegen._invert_list(body)) == body


def test_besselj_parses_and_expands():
    text = open(os.path.join(REPO, "paper_2003_04617_b200", "programs", "besselj.rnl")).read()
    (params, body), = codegen._Parser(text).program().values()
    assert params == ("out!", "nu", "z")
    fwd = codegen._expand(body)
    # the routine opens, the middle runs, the routine closes inverted
    assert isinstance(fwd[0], codegen.Alloc) and isinstance(fwd[-1], codegen.Dealloc)
    assert any(isinstance(s, codegen.While) for s in fwd)


def test_calls_are_inlined_with_fresh_locals():
    """programs/ba.rnl calls rodrigues inside a routine: four inlined copies
    (forward, routine close, and both again in the gradient sweep)."""
    text = open(os.path.join(REPO, "paper_2003_04617_b200", "programs", "ba.rnl")).read()
    source = codegen.generate(text, "ba_proj", array_shapes={"cam": 11, "X": 3})[0]
    for j in range(1, 5):
        assert f"v_th__rodrigues{j}" in source
    # recursion is inlined level by level; past REVGPU_CODEGEN_DEPTH the kernel
    # reports the interpreter's RecursionError (an endless self-call here)
    assert "code = RC_DEPTH" in codegen.generate("fn f(y!, x)\n f(y!, x)\nend\n", "f")[0]
    with pytest.raises(UnsupportedProgram):               # two self-calls per level: 2^24 copies
        codegen.generate("fn f(y!, x)\n f(y!, x)\n f(y!, x)\nend\n", "f")
    with pytest.raises(UnsupportedProgram):                 # leaks an ancilla (DirtyAncilla)
        codegen.generate("fn g(y!)\n t <- 0.0\nend\nfn f(y!)\n g(y!)\nend\n", "f")


def test_unsupported_constructs_are_rejected():
    for text in ("fn f(y!, x)\n g(y!, x)\nend\n",
                 "fn f(y!, x)\n h(y!, x |> mulconst(2.5))\nend\nfn h(a!, b)\n a! += b\nend\n",
                 "fn f(y!, x)\n y! += 1.0im\nend\n",
                 "fn f(y!, x)\n y!.rec += x\nend\n",
                 "fn f(y!, x)\n @safe print(x)\nend\n"):
        with pytest.raises(UnsupportedProgram):
            codegen.generate(text, "f")


def test_complex_field_views():
    with pytest.raises(KindError):                      # y! is not declared Complex
        codegen.generate("fn f(y!, x)\n y!.re += x\nend\n", "f")
    src_, floats, ints, leaves = codegen.generate("fn f(y!, x)\n y!.re += x\nend\n", "f",
                                                  complex_params=("y!",))
    assert leaves == [("y!", (("field", "re"),)), ("y!", (("field", "im"),)), ("x", ())]


def test_array_shapes_are_required_and_checked():
    text = "fn f(y!::array, x)\n y![1] += x\nend\n"
    with pytest.raises(KindError):                      # ::array without a shape
        codegen.generate(text, "f")
    with pytest.raises(KindError):
        codegen.generate(text, "f", array_shapes={"y!": (2, 2, 2)})
    with pytest.raises(KindError):                      # whole array as an operand
        codegen.generate("fn f(y!, x::array)\n y! += x\nend\n", "f", array_shapes={"x": 3})
    src_, floats, ints, leaves = codegen.generate(text, "f", array_shapes={"y!": (2, 3)})
    assert floats == ["y!", "x"] and ints == []
    assert leaves[:2] == [("y!", (("idx", (1, 1)),)), ("y!", (("idx", (1, 2)),))]
    assert leaves[-1] == ("x", ()) and len(leaves) == 7


def test_aliasing_is_checked_at_run_time():
    """interpreter.py:624-657: same-root operands raise AliasedArguments when
    the instruction runs (a branch never taken never raises), so the checks
    are emitted into the kernel rather than rejected at compile time."""
    src_ = codegen.generate("fn f(y!, x)\n y! += x * x\nend\n", "f")[0]
    fwd, grad = src_.split("uncall_function")
    assert "RC_ALIAS" not in fwd.split("run_function")[1] and "RC_ALIAS" in grad
    src_ = codegen.generate("fn f(y!, x)\n y! += y! * x\nend\n", "f")[0]
    assert "RC_ALIAS" in src_.split("run_function")[1].split("uncall_function")[0]
    src_ = codegen.generate(src("mix"), "mix_fwd", ("k", "m"), array_shapes={"x": 4})[0]
    assert "if (o1 == o2 && !code) code = RC_ALIAS;" in src_


def test_generated_source_compiles_for_sm100a(tmp_path, monkeypatch):
    monkeypatch.setenv("REVGPU_CODEGEN_CACHE", str(tmp_path))
    source, floats, ints, _ = codegen.generate(src("sink"), "sink", ("n",))
    assert floats == ["out!", "x", "y"] and ints == ["n"]
    so = codegen.build(source)
    assert os.path.exists(so)
    source = codegen.generate(src("quad"), "quad", array_shapes={"r!": 3, "A": (3, 3), "u": 3},
                              mode="hess")[0]
    assert os.path.exists(codegen.build(source))


def test_view_argument_indexed_by_another_argument():
    """kick_pair-style calls: a view argument indexed by a scalar that is
    also passed is inlined when the callee never writes that parameter."""
    text = src("nbody")
    codegen.generate(text, "nbody", ("steps",),
                     array_shapes={"pos!": (4, 3), "vel!": (4, 3), "mass": 4})
    bad = ("fn g(y!, k)\n    y! += 1.0\n    k += 1\nend\n"
           "fn f(x::array, k)\n    g(x[k], k)\nend\n")
    with pytest.raises(UnsupportedProgram):
        codegen.generate(bad, "f", ("k",), array_shapes={"x": 3})


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"),
                    reason="the reference is only present in the build container")
def test_reference_catalog_programs_in_the_subset_compile(tmp_path, monkeypatch):
    """The reference's own catalog (stdlib.CATALOG), pretty-printed by the
    reference and compiled here: every program whose argument kinds are in
    the subset generates and builds for sm_100a: all ten, the Complex and
    Fixed ones and the recursive bijector-view program (rrfib) included."""
    import random
    import sys
    monkeypatch.setenv("REVGPU_CODEGEN_CACHE", str(tmp_path))
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        from revlang.parser import pretty_print
        from revlang.stdlib import CATALOG, entry_function, load_example, sample_args
    finally:
        sys.path.pop(0)
    from paper_2003_04617_b200 import generic
    built, rejected = [], []
    for name in CATALOG:
        p, fn = load_example(name), entry_function(name)
        args = sample_args(name, random.Random(1))
        try:
            kinds = {nm: generic._kind(v, nm) for nm, v in zip(p.get(fn).param_names(), args)}
            ints = tuple(k for k, (kk, _) in kinds.items() if kk in ("i", "ai"))
            shapes = {k: s for k, (kk, s) in kinds.items() if kk in ("a", "ai")}
            cplx = tuple(k for k, (kk, _) in kinds.items() if kk == "c")
            fixed = tuple(k for k, (kk, _) in kinds.items() if kk == "x")
            codegen.build(codegen.generate(pretty_print(p), fn, ints, array_shapes=shapes,
                                           complex_params=cplx, fixed_params=fixed)[0])
            built.append(name)
        except UnsupportedProgram:
            rejected.append(name)
    assert {"multiplier", "i_affine", "i_umm", "r_norm", "leapfrog_clean",
            "leapfrog_cumulative", "complex_log", "complex_log_ccu", "mypower_log",
            "rrfib_corrected"} <= set(built), \
        (built, rejected)


def test_fixed_literals_and_rounding():
    """Q31.32 from_real: round half to even, wrapped mod 2^64 (values.py:23-41);
    the package's Fixed and the compiler's literal conversion agree."""
    import paper_2003_04617_b200 as rg
    assert codegen._fx_from_real(1.5) == 3 << 31
    assert codegen._fx_from_real(2.5 / 2 ** 32) == 2          # half to even
    assert codegen._fx_from_real(3.5 / 2 ** 32) == 4
    assert codegen._fx_from_real(2.0 ** 31) == -(1 << 63)     # wraps
    assert codegen._fx_from_real(-2.0 ** 31) == -(1 << 63)
    for v in (0.0, -1.25, 1e9, -3e9, 1.3, 7.1e-10):
        assert rg.Fixed.from_real(v).raw == codegen._fx_from_real(v)
    toks = codegen._tokenize("x != 0fx + 2.25fx")
    assert toks[2] == ("num", codegen.FixLit(0)) and toks[4] == ("num", codegen.FixLit(9 << 30))


def test_fixed_program_generates_and_builds(tmp_path, monkeypatch):
    """tests/golden/codegen/fxmix.rnl: Fixed parameters, literals, a Fixed
    ancilla, Fixed += Float, Float += f(Fixed): all modes generate and build."""
    monkeypatch.setenv("REVGPU_CODEGEN_CACHE", str(tmp_path))
    text = open(os.path.join(os.path.dirname(__file__), "golden", "codegen", "fxmix.rnl")).read()
    for mode in ("grad", "run", "uncall"):
        code, floats, ints, leaves = codegen.generate(text, "fxmix", ("k",), mode=mode,
                                                      fixed_params=("acc!", "b"))
        assert "rl_fx_from" in code and floats == ["acc!", "y!", "b"] and ints == ["k"]
        codegen.build(code)
    with pytest.raises(UnsupportedProgram):
        codegen.generate(text, "fxmix", ("k",), mode="hess", fixed_params=("acc!", "b"))
