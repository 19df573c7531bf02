"""A few drop-in GMM gradient evaluations (rl_gmm_gradient_f64) at a BASELINE
config (ncu target).  usage: python tools/gmm_one.py [c3|c5|N] [reps] [--flush]
(--flush: a 256 MiB L2 eviction before every evaluation, as bench.py does; with
`ncu --cache-control none` the DRAM counters then show one evaluation's real
traffic: caches are not flushed between its kernels)"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2003_04617_b200 as rg  # noqa: E402
from test_gmm_gpu import gmm_constants, inputs  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
d, K, N = (64, 25, 10000) if which == "c3" else (128, 200, int(which) if which.isdigit() else 100000)
a, me, ic, x = (torch.as_tensor(v, device="cuda") for v in inputs(np.random.default_rng(2), d, K, N))
cst = gmm_constants(d, K, N, 1.0, 0)
ws = torch.empty(rg.kernels._native.lib().rl_gmm_workspace_bytes(d, K, N), dtype=torch.uint8,
                 device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
# --flush evicts L2 by READING 256 MiB (clean lines: no write-back of the
# eviction buffer lands in the measured kernels' DRAM-write counters)
flush = torch.ones(32 << 20, dtype=torch.float64, device="cuda") if "--flush" in sys.argv else None
torch.cuda.synchronize()
for i in range(reps):
    if flush is not None:
        flush.sum()                # evict L2 between evaluations (bench.py writes instead)
    ev[0].record()
    r = rg.gmm_gradient(a, me, ic, x, 1.0, 0, cst, workspace=ws)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"eval {i}: {ev[0].elapsed_time(ev[1]):.4f} ms, E={r.err.item():.6f}")
