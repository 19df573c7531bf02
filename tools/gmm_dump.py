"""Dump one GMM gradient evaluation (packed [err, g_alphas, g_means, g_icf],
fail flags, counters) for bitwise comparison of library variants:
REVGPU_LIB=... python tools/gmm_dump.py out.npz [d K N]."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2003_04617_b200 import kernels  # noqa: E402

d, K, N = (int(v) for v in (sys.argv[2:5] if len(sys.argv) > 4 else (64, 25, 10000)))
g = torch.Generator(device="cuda").manual_seed(5)
dev = "cuda"
alphas = torch.randn(K, dtype=torch.float64, device=dev, generator=g)
means = torch.rand(K, d, dtype=torch.float64, device=dev, generator=g)
icf = torch.randn(K, d * (d + 1) // 2, dtype=torch.float64, device=dev, generator=g) * 0.5
x = torch.rand(N, d, dtype=torch.float64, device=dev, generator=g)
r = kernels.gmm_grad(alphas, means, icf, x, 1.0, 0, 0.0)
torch.cuda.synchronize()
np.savez(sys.argv[1], packed=r.packed.cpu().numpy(), fail=r.fail.cpu().numpy(),
         counters=r.counters.cpu().numpy())
print("dumped", sys.argv[1], float(r.packed[0]))
