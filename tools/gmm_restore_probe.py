"""Cost of the in-order err! replay (k_gmm_restore on a side stream beside
k_gmm_rev): device time per evaluation of rl_gmm_grad_f64 (tree-summed
objective, no restoration verdict) vs rl_gmm_gradient_f64 (the drop-in
gradient() with the replay), direct launches and CUDA-graph replays."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2003_04617_b200 as rg  # noqa: E402
from test_gmm_gpu import gmm_constants, inputs  # noqa: E402


def timeit(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for (d, K, N) in [(64, 25, 10000), (128, 200, 100000)]:
    al, me, ic, x = (torch.as_tensor(v, device="cuda") for v in inputs(np.random.default_rng(2), d, K, N))
    cst = gmm_constants(d, K, N, 1.0, 0)
    L = rg._native.lib() if hasattr(rg, "_native") else None
    ws = torch.empty(int(rg.kernels._native.lib().rl_gmm_workspace_bytes(d, K, N)), dtype=torch.uint8, device="cuda")
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    f_tree = lambda: rg.gmm_grad(al, me, ic, x, 1.0, 0, cst, workspace=ws, counters=cnt)  # noqa: E731
    f_seq = lambda: rg.gmm_gradient(al, me, ic, x, 1.0, 0, cst, tol=1e-6, workspace=ws, counters=cnt)  # noqa: E731
    t_tree, t_seq = timeit(f_tree), timeit(f_seq)
    res = {}
    for nm, fn in (("tree", f_tree), ("seq", f_seq)):
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                fn()
        res[nm] = timeit(g.replay)
    r = f_seq()
    torch.cuda.synchronize()
    print(f"d={d} K={K} N={N}: direct tree {t_tree:.4f} ms, seq {t_seq:.4f} ms; "
          f"graph tree {res['tree']:.4f} ms, seq {res['seq']:.4f} ms; E={r.err.item():.6f} "
          f"resid={r.resid.item():.3e} code={int(r.restore_code.item())}")
