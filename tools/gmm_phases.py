"""Cycle split of k_gmm_fwd at configs[2] over its per-tile phases, summed
over warps (timing-only -DGMM_PHASES variant through REVGPU_LIB)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2003_04617_b200 as rg  # noqa: E402
from paper_2003_04617_b200 import _native  # noqa: E402
from test_gmm_gpu import gmm_constants, inputs  # noqa: E402

d, K, N = 64, 25, 10000
a, me, ic, x = (torch.as_tensor(v, device="cuda") for v in inputs(np.random.default_rng(2), d, K, N))
cst = gmm_constants(d, K, N, 1.0, 0)
lib = _native.lib()
out = (ctypes.c_ulonglong * 32)()
for rep in range(2):
    rg.gmm_gradient(a, me, ic, x, 1.0, 0, cst)
    torch.cuda.synchronize()
    lib.rl_debug_gmm_phases(out)
names = {0: "prologue", 1: "x wait (+prefetch issue)", 2: "sync 1", 3: "center", 4: "sync 2",
         5: "MMA issue", 6: "sqn epilogue (MMA drain)", 7: "sync 3", 8: "mt stores"}
tot = sum(out[i] for i in names)
for i, nm in sorted(names.items()):
    print(f"fwd {nm:26s} {100 * out[i] / tot:5.1f}%")
rnames = {0: "prologue", 1: "x wait + top sync", 2: "prefetch issue + cg", 3: "center",
          4: "sync B", 5: "Z MMA issue", 6: "G epilogue (MMA drain)", 7: "sync C",
          8: "M-product"}
tot = sum(out[16 + i] for i in rnames)
for i, nm in sorted(rnames.items()):
    print(f"rev {nm:26s} {100 * out[16 + i] / tot:5.1f}%")
