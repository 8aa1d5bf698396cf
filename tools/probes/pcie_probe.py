"""Pinned host <-> device copy bandwidth on the GPU box (context for e2e)."""
import time

import torch

n = 192 * 1024 * 1024 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"{name}: {n * 8 / dt / 1e9:.1f} GB/s ({dt * 1e3:.2f} ms per 192 MiB)")
