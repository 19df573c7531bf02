"""Generic .rnl -> CUDA Bessel gradient vs the hand-written kernel on the
configs[1] batch: device ms per launch, and agreement on the full batch."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2003_04617_b200 import codegen, kernels  # noqa: E402

n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 26)
g = torch.Generator(device="cuda")
g.manual_seed(1)
z = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(0.1, 10.0, generator=g)
ck = codegen.compile_function(open("paper_2003_04617_b200/programs/besselj.rnl").read(),
                              "besselj", int_params=("nu",))


def timed(fn, reps=8, rounds=3):
    """best of `rounds` means over `reps` back-to-back launches"""
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(rounds):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            r = fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best, r


tg, (primal, grads, fail) = timed(lambda: ck.gradient({"out!": 0.0, "z": z, "nu": 2}))
th, hw = timed(lambda: kernels.besselj_grad(z, 2))
J, dz = primal["out!"], grads["z"]
ok = (fail == 0) & (hw.fail == 0)
print(f"n={n}: generic {tg:.3f} ms, hand-written {th:.3f} ms, ratio {tg / th:.2f}; "
      f"codes equal {bool(torch.equal(fail, hw.fail))}; J bit-equal frac "
      f"{(J[ok] == hw.J[ok]).double().mean().item():.4f}, max |dJ| "
      f"{(J[ok] - hw.J[ok]).abs().max().item():.3e}, max |d dz| "
      f"{(dz[ok] - hw.dJdz[ok]).abs().max().item():.3e}")
