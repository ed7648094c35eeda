"""Pinned D2H bandwidth: one stream vs two / four concurrent streams (dev probe)."""
import time

import torch

dev = torch.device("cuda", 0)
n = 1 << 28  # 1 GiB of float32
src = torch.empty(n, dtype=torch.float32, device=dev).fill_(1.0)
dst = torch.empty(n, dtype=torch.float32).pin_memory()
for k in (1, 2, 4):
    streams = [torch.cuda.Stream(dev) for _ in range(k)]
    part = n // k
    best = 0.0
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dst[i * part:(i + 1) * part].copy_(src[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
        best = max(best, 4 * n / (time.perf_counter() - t0) / 1e9)
    print(f"{k} stream(s): {best:.1f} GB/s")
