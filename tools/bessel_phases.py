"""Cycle split of k_besselj<1> over its per-chunk phases, summed over warps
(timing-only -DBJ_PHASES variant through REVGPU_LIB; tools/build_variants.sh)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2003_04617_b200 import _native, kernels  # noqa: E402

n = 1 << 24
g = torch.Generator(device="cuda")
g.manual_seed(1)
z = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(0.1, 10.0, generator=g)
lib = _native.lib()
out = (ctypes.c_ulonglong * 16)()
kernels.besselj_grad(z, 2)
torch.cuda.synchronize()
lib.rl_debug_bj_phases(out)
kernels.besselj_grad(z, 2)
torch.cuda.synchronize()
lib.rl_debug_bj_phases(out)
names = {0: "hist (+cp.async wait)", 1: "scan", 2: "scatter", 4: "round-end barrier",
         5: "stores", 6: "element prologue", 7: "forward loops", 8: "reverse loops",
         9: "element epilogue", 3: "round loop other"}
tot = sum(out[i] for i in names)
for i, nm in sorted(names.items()):
    print(f"{nm:24s} {100 * out[i] / tot:5.1f}%")
