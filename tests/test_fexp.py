"""csrc/fexp.cuh (the series kernels' exp) on the host, against the C
library exp that CPython's math.exp (the reference's s_exp) calls."""

import os
import subprocess

from conftest import REPO


def test_fexp_within_one_ulp_and_mostly_bit_identical(tmp_path):
    exe = str(tmp_path / "fexp_test")
    subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-o", exe,
                           os.path.join(REPO, "tools", "fexp_test.cpp")])
    for tab in ("64", "256", "1024"):                      # fexp_core / fexp1024_core (the kernel's)
        for lo, hi, seed in ((-40.0, 10.0, 1), (-707.0, 707.0, 2), (-1e-3, 1e-3, 3)):
            n, eq, maxulp = subprocess.check_output(
                [exe, "2000000", str(lo), str(hi), str(seed), tab], text=True).split()
            assert float(maxulp) <= 1.0
            assert int(eq) / int(n) > 0.995
