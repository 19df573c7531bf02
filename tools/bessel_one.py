"""A few rl_besselj_grad_f64 launches over n z ~ U(0.1, 10) (ncu target).
usage: python tools/bessel_one.py [log2 n] [launches]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2003_04617_b200 import kernels  # noqa: E402

n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 24)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = torch.Generator(device="cuda")
g.manual_seed(1)
z = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(0.1, 10.0, generator=g)
J, dz = torch.empty_like(z), torch.empty_like(z)
fail = torch.empty(n, dtype=torch.uint8, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(reps):
    a.record()
    kernels.besselj_grad(z, 2, out=(J, dz, fail))
    b.record()
    torch.cuda.synchronize()
    print(f"launch {i}: {a.elapsed_time(b):.4f} ms ({n} z)")
