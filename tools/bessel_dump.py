"""Dump one Bessel gradient / run batch (J, dJ/dz, fail, trips) for bitwise
comparison of library variants: REVGPU_LIB=... python tools/bessel_dump.py out.npz."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2003_04617_b200 import kernels  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(3)
z = torch.empty(1 << 22, dtype=torch.float64, device="cuda").uniform_(0.1, 10.0, generator=g)
z[::1001] = -1.0
z[5::777] = 650.0                           # CAREFUL re-run path
r = kernels.besselj_grad(z, 2)
q = kernels.besselj_grad(z, 5, seed=0.37)   # non-unit seed, other order
u = kernels.besselj_run(z, 2)
h = kernels.besselj_hess(z, 2)
h3 = kernels.besselj_hess(z, 3, seed=0.37)
torch.cuda.synchronize()
np.savez(sys.argv[1], J=r.J.cpu().numpy(), dz=r.dJdz.cpu().numpy(), f=r.fail.cpu().numpy(),
         t=np.array([r.sum_trips]), J5=q.J.cpu().numpy(), dz5=q.dJdz.cpu().numpy(),
         run=u.out.cpu().numpy(), runf=u.fail.cpu().numpy(), hJ=h.J.cpu().numpy(),
         hdz=h.dJdz.cpu().numpy(), hd2=h.d2Jdz2.cpu().numpy(), hf=h.fail.cpu().numpy(),
         ht=np.array([h.sum_trips]), h3d2=h3.d2Jdz2.cpu().numpy(), h3f=h3.fail.cpu().numpy())
print("dumped", sys.argv[1])
