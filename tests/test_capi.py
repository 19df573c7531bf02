"""The C-ABI boundary: librevgpu.so loads and exports exactly what
include/revgpu.h declares (no compute calls here: CPU host)."""

import ctypes
import os
import re
import subprocess

from conftest import REPO

HEADER = os.path.join(REPO, "include", "revgpu.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int64_t|int|size_t|const char \*)\s*(rl_\w+)\(", text, re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("rl_besselj_grad_f64", "rl_besselj_grad_f64_host", "rl_ba_jac_f64",
              "rl_ba_jac_f64_host", "rl_gmm_grad_f64", "rl_gmm_grad_f64_host",
              "rl_gmm_workspace_bytes", "rl_strerror", "rl_abi_version", "rl_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2003_04617_b200 import _native
    L = _native.lib()
    for s in declared_symbols():
        assert hasattr(L, s), s
    out = subprocess.check_output(["nm", "-D", "--defined-only", _native.LIB_PATH], text=True)
    exported = set(re.findall(r"\bT (rl_\w+)", out))
    assert set(declared_symbols()) <= exported
    # the python binding describes every declared symbol
    assert set(declared_symbols()) == set(_native.exported_symbols())


def test_abi_and_status_strings():
    from paper_2003_04617_b200 import _native
    L = _native.lib()
    assert L.rl_abi_version() == 1
    names = {1: b"PostconditionMismatch", 2: b"DirtyAncilla", 3: b"RevDomainError",
             4: b"LoopIteratorMutated", 5: b"RevError", 6: b"FuelExhausted", 7: b"KindError",
             8: b"IndexOutOfBounds", 9: b"OverflowError"}
    for code, nm in names.items():
        assert L.rl_strerror(code) == nm
    from paper_2003_04617_b200.errors import CODE_NAMES
    for code, nm in names.items():
        assert CODE_NAMES[code] == nm.decode()


def test_library_is_sm100a_only():
    from paper_2003_04617_b200 import _native
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                                   _native.LIB_PATH], text=True)
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_gmm_workspace_query_is_pure():
    from paper_2003_04617_b200 import _native
    L = _native.lib()
    assert L.rl_gmm_workspace_bytes(64, 25, 10000) >= 0


def test_invalid_arguments_rejected_before_any_device_work():
    from paper_2003_04617_b200 import _native
    L = _native.lib()
    rc = L.rl_besselj_grad_f64(2, None, -5, 1e-16, 1e-9, 1.0, 100, 1, None, None, None, None,
                               None)
    assert rc == _native.RL_ERR_INVALID
    assert b"bad argument" in L.rl_last_error()
