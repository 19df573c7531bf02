"""Where the GMM drop-in host-buffer call's time goes at configs[2]: the full
rl_gmm_gradient_f64_host call, the device step alone (inputs resident), and
the pinned H2D of x / D2H of the gradient alone."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2003_04617_b200 as rg  # noqa: E402
from paper_2003_04617_b200 import _native  # noqa: E402
from test_gmm_gpu import gmm_constants, inputs  # noqa: E402

d, K, N = 64, 25, 10000
al, me, ic, x = inputs(np.random.default_rng(2), d, K, N)
cst = gmm_constants(d, K, N, 1.0, 0)
L = _native.lib()
pin = lambda a: torch.as_tensor(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
ha, hm, hi, hx = pin(al), pin(me), pin(ic), pin(x)
nout = 1 + K + K * d + K * d * (d + 1) // 2
out = torch.empty(nout, dtype=torch.float64).pin_memory()
nf, resid = ctypes.c_ulonglong(), ctypes.c_double()


def call():
    L.rl_gmm_gradient_f64_host(d, K, N, ha.data_ptr(), hm.data_ptr(), hi.data_ptr(), hx.data_ptr(),
                               1.0, 0, cst, 0.0, 1e-9, 1, out.data_ptr(), ctypes.byref(resid),
                               ctypes.byref(nf), 0)


def wall(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


print(f"host entry call        {wall(call):.4f} ms")
dev = torch.device("cuda")
da, dm, di, dx = (t.to(dev) for t in (ha, hm, hi, hx))
ws = torch.empty(L.rl_gmm_workspace_bytes(d, K, N), dtype=torch.uint8, device=dev)
print(f"device step (no copies) {wall(lambda: rg.gmm_gradient(da, dm, di, dx, 1.0, 0, cst, workspace=ws)):.4f} ms")
buf = torch.empty_like(dx)
print(f"H2D x pinned ({hx.numel() * 8 / 1e6:.1f} MB) {wall(lambda: buf.copy_(hx, non_blocking=True)):.4f} ms")
dout = torch.empty(nout, dtype=torch.float64, device=dev)
print(f"D2H gradient ({nout * 8 / 1e6:.2f} MB) {wall(lambda: out.copy_(dout, non_blocking=True)):.4f} ms")
