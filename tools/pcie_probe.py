"""Pinned host <-> device copy bandwidth vs transfer size (one B200)."""
import time

import torch

dev = torch.device("cuda", 0)
for mb in (0.5, 2, 5, 20, 80, 320):
    n = int(mb * (1 << 20)) // 8
    h = torch.rand(n, dtype=torch.float64).pin_memory()
    d = torch.empty(n, dtype=torch.float64, device=dev)
    for name, f in (("H2D", lambda: d.copy_(h, non_blocking=True)),
                    ("D2H", lambda: h.copy_(d, non_blocking=True))):
        f()
        torch.cuda.synchronize()
        reps = 10
        t0 = time.perf_counter()
        for _ in range(reps):
            f()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        f()
        ev1.record()
        torch.cuda.synchronize()
        print(f"{name} {mb:6.1f} MB  wall {dt * 1e3:7.3f} ms  {n * 8 / dt / 1e9:6.1f} GB/s   "
              f"event {ev0.elapsed_time(ev1):7.3f} ms")
