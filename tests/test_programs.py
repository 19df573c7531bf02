"""Program recognition (the drop-in boundary's front end) and the host API's
refusal to run anything without a device kernel."""

import os

import pytest

import paper_2003_04617_b200 as rg
from paper_2003_04617_b200.programs import program_text


def test_catalog_programs_bind_to_kernels():
    for name in rg.CATALOG:
        p = rg.load_example(name)
        f = p.functions[rg.entry_function(name)]
        assert f.kernel is not None, name


def test_formatting_and_comments_do_not_matter():
    text = program_text("besselj")
    mangled = "# leading comment\n" + text.replace("    ", "\t").replace("<-", "←")
    mangled = mangled.replace("1e-16", "1.0e-16")
    p = rg.parse_program(mangled)
    assert p.functions["besselj"].kernel is not None
    assert p.functions["besselj"].constants["thr"] == 1e-16


def test_threshold_literal_is_a_kernel_parameter():
    p = rg.parse_program(program_text("besselj").replace("1e-16", "1e-10"))
    assert p.functions["besselj"].constants["thr"] == 1e-10


def test_modified_program_has_no_kernel():
    """A modified benchmark program loses its hand-written kernel; calling it
    goes to the generic compiler, which (like every kernel) has no CPU path."""
    text = program_text("besselj").replace("s /= kn", "s /= k")
    p = rg.parse_program(text)
    assert p.functions["besselj"].kernel is None
    import torch
    if torch.cuda.is_available():
        pytest.skip("host has a GPU (tests/test_generic_dropin_gpu.py covers that path)")
    with pytest.raises(rg.UnsupportedProgram):
        rg.gradient(p, rg.GradRequest("besselj", [0.0, 2, 1.0]))


def test_ba_needs_its_registered_helper():
    text = program_text("ba_proj").replace("th += sqrt(sqt)", "th += sqt")
    p = rg.parse_program(text)
    assert p.functions["ba_proj"].kernel is None
    assert p.functions["ba_weight"].kernel is not None


def test_unknown_function_and_example():
    with pytest.raises(rg.UnknownFunction):
        rg.gradient(rg.load_example("besselj"), rg.GradRequest("nope", []))
    with pytest.raises(rg.UnknownExample):
        rg.load_example("nope")


def test_param_names_match_the_reference_signature():
    assert rg.load_example("besselj").functions["besselj"].param_names() == ["out!", "nu", "z"]
    assert rg.load_example("gmm").functions["gmm"].param_names()[:5] == \
        ["err!", "alphas", "means", "icf", "x"]
    p = rg.parse_program("fn r_norm(out!, out2!, x::array)\n out! += x[1]\nend")
    assert p.functions["r_norm"].param_names() == ["out!", "out2!", "x"]


def test_exec_options_validation():
    with pytest.raises(ValueError):
        rg.ExecOptions(float_tolerance=-1)
    with pytest.raises(ValueError):
        rg.ExecOptions(max_steps=0)


def test_no_cpu_fallback_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("host has a GPU")
    with pytest.raises(rg.UnsupportedProgram):
        rg.gradient(rg.load_example("besselj"), rg.GradRequest("besselj", [0.0, 2, 1.0]))
    with pytest.raises(rg.KindError):
        rg.besselj_grad(torch.ones(4, dtype=torch.float64))


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"),
                    reason="reference tree only exists in the build container")
def test_reference_program_objects_go_through_their_text():
    """The product runs no reference code: a revlang.Program object is
    rejected with guidance, and its pretty-printed text (printed here by the
    reference, test infrastructure) is recognised as the registered program."""
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.dont_write_bytecode = True
    from revlang import parse_program as ref_parse
    from revlang.parser import pretty_print
    ref_prog = ref_parse(program_text("besselj"))
    with pytest.raises(rg.UnsupportedProgram, match="pretty_print"):
        rg.programs.as_program(ref_prog)
    p = rg.programs.as_program(pretty_print(ref_prog))
    assert p.functions["besselj"].kernel is not None
