"""Phase timestamps of rl_seq_sum_f64 (needs a -DSEQ_DIAG build via REVGPU_LIB)."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_2003_04617_b200 import _native  # noqa: E402
from test_seqsum_gpu import gmm_like  # noqa: E402
L = _native.lib()
for N in (10000, 1000000):
    d = torch.as_tensor(gmm_like(np.random.default_rng(7), N), device="cuda")
    out = torch.zeros(2 + 16, dtype=torch.float64, device="cuda")
    for _ in range(3):
        L.rl_seq_sum_f64(ctypes.c_void_p(d.data_ptr()), d.numel(), 0.0, d.numel(), 0,
                         ctypes.c_void_p(out.data_ptr()), None, None)
    torch.cuda.synchronize()
    o = out.cpu().numpy()[2:]
    ph = np.diff(o[:7])
    print(N, "phases (cycles):", dict(zip(["walk1", "scans", "walk2", "compact", "fold", "walk3"],
                                           ph.astype(int))), "nmk+1000ntot", o[8])
