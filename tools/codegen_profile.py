"""Run the generically compiled besselj.rnl gradient on 2^22 elements (for
ncu: the generated kernel is rlg_kernel)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_04617_b200 import codegen  # noqa: E402

src = open(os.path.join(os.path.dirname(__file__), "..", "paper_2003_04617_b200", "programs",
                        "besselj.rnl")).read()
k = codegen.compile_function(src, "besselj", int_params=("nu",))
g = torch.Generator(device="cuda").manual_seed(1)
z = torch.empty(1 << 22, dtype=torch.float64, device="cuda").uniform_(0.1, 10.0, generator=g)
for _ in range(2):
    primal, grads, fail = k.gradient({"out!": 0.0, "z": z, "nu": 2})
torch.cuda.synchronize()
print("ok", int(fail.sum()))
