"""Probe rl_seq_sum_f64: verified flag and device time per call (CUDA
events over back-to-back launches) on GMM-like and other sequences."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2003_04617_b200 as rg  # noqa: E402
from paper_2003_04617_b200 import _native  # noqa: E402
from test_seqsum_gpu import gmm_like  # noqa: E402

L = _native.lib()
for name, t in [("gmm_c3", gmm_like(np.random.default_rng(7), 10000)),
                ("gmm_c5", gmm_like(np.random.default_rng(7), 1000000)),
                ("normal", np.random.default_rng(1).normal(0, 1, 100003)),
                ("growth", np.random.default_rng(2).uniform(0, 1e3, 60000))]:
    d = torch.as_tensor(t, device="cuda")
    print(name, len(t), rg.seq_sum(d, 0.0))
    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    args = (ctypes.c_void_p(d.data_ptr()), d.numel(), 0.0, d.numel(), 0,
            ctypes.c_void_p(out.data_ptr()), None, ctypes.c_void_p(st))
    for _ in range(3):
        L.rl_seq_sum_f64(*args)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        L.rl_seq_sum_f64(*args)
    b.record()
    torch.cuda.synchronize()
    print(name, "kernel us/call", a.elapsed_time(b) / 20 * 1e3)
