"""Small runs of every kernel family, an extended smoke (compute-sanitizer is
not available on the GPU pool): Bessel gradient / run / Hessian and the host
entry (with failing elements: the status-list path), BA dense and CSR, GMM
gradient (lse with 4 lanes, and K > 96), a generated kernel (arrays, calls)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2003_04617_b200 as rg  # noqa: E402
from paper_2003_04617_b200 import codegen, kernels  # noqa: E402

dev = "cuda"
rng = np.random.default_rng(0)
z = rng.uniform(0.1, 10.0, 5000)
z[::97] = -1.0
zt = torch.as_tensor(z, device=dev)
rg.besselj_grad(zt, 2)
rg.besselj_run(zt, 2)
rg.besselj_hess(zt[:1000], 2)
kernels.besselj_grad_host(z, 2)
cams = np.concatenate([rng.normal(0, 0.3, (8, 3)), rng.normal(0, 1, (8, 3)),
                       rng.uniform(500, 600, (8, 1)), rng.uniform(0, 1, (8, 2)),
                       rng.normal(0, 0.01, (8, 2))], 1)
X = rng.normal(0, 1, (16, 3))
X[:, 2] += 10
w, f = rng.uniform(0, 1, 300), rng.uniform(0, 100, (300, 2))
obs = np.stack([np.arange(300) % 8, np.arange(300) % 16], 1).astype(np.int32)
t = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
rg.ba_jacobian(t(cams), t(X), t(w), t(f), t(obs))
rg.ba_jacobian_csr(t(cams), t(X), t(w), t(f), t(obs))
for d, K, N in ((8, 5, 700), (4, 120, 90)):
    P = d * (d + 1) // 2
    rg.gmm_grad(t(rng.normal(size=K)), t(rng.uniform(size=(K, d))), t(rng.normal(0, .5, (K, P))),
                t(rng.uniform(size=(N, d))), 1.0, 0, 0.0)
src = open("tests/golden/codegen/nbody.rnl").read()
k = codegen.compile_function(src, "nbody", int_params=("steps",),
                             array_shapes={"pos!": (4, 3), "vel!": (4, 3), "mass": 4})
k.gradient({"pos!": t(rng.uniform(-1, 1, (64, 4, 3))), "vel!": t(rng.uniform(-.2, .2, (64, 4, 3))),
            "mass": t(rng.uniform(.5, 1.5, (64, 4))), "h": 0.01, "steps": 2},
           seeds=[("pos!", (("idx", (1, 1)),), 1.0)])
torch.cuda.synchronize()
print("sanitize run ok")
