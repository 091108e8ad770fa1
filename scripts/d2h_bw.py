"""Host link bandwidth (pinned D2H / H2D) on this box: the e2e ceiling."""
import time

import torch

n = 2 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8).pin_memory()
for name, dst, src in (("D2H", h, d), ("H2D", d, h)):
    for _ in range(2):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"{name}: {n / dt / 1e9:.1f} GB/s ({n / 1e9:.2f} GB in {1e3 * dt:.1f} ms)")
