"""One GMM-sized rl_seq_sum_f64 problem, launched a few times (ncu target).
usage: python tools/seq_one.py N   (M = 4N + 8 terms)"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_2003_04617_b200 import _native  # noqa: E402
from test_seqsum_gpu import gmm_like  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
L = _native.lib()
d = torch.as_tensor(gmm_like(np.random.default_rng(7), N), device="cuda")
out = torch.zeros(2, dtype=torch.float64, device="cuda")
for _ in range(3):
    L.rl_seq_sum_f64(ctypes.c_void_p(d.data_ptr()), d.numel(), 0.0, d.numel(), 0,
                     ctypes.c_void_p(out.data_ptr()), None, None)
torch.cuda.synchronize()
print(out.cpu())
