"""e2e HostStream throughput vs slots / part size on config 5 (dev probe; 8192 rooms)."""
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_2304_08052_b200 import engine, workloads  # noqa: E402

dev = torch.device('cuda', 0)
w = workloads.build(5, 8192)
for slots, part in ((2, 1024), (3, 1024), (4, 512), (2, 2048), (3, 512)):
    hs = engine.HostStream(w.sample_rate, w.jobs, w.mics, part_jobs=part, include_early=True, slots=slots, device=dev)
    hs.run()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hs.run()
    s = time.perf_counter() - t0
    t0 = time.perf_counter()
    hs.run(revalidate=False)
    s2 = time.perf_counter() - t0
    print(f"slots {slots} part {part}: {8192 / s:.0f} RIR/s ({hs.d2h_bytes / s / 1e9:.1f} GB/s), no revalidate {8192 / s2:.0f} RIR/s")
    del hs
    torch.cuda.empty_cache()
