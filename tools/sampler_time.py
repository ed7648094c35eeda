"""Time DeviceSceneSampler.render (dev tool)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_08052_b200 import mixture as MX  # noqa: E402
from paper_2304_08052_b200.sampler import DeviceSceneSampler  # noqa: E402

smp = DeviceSceneSampler(MX.MixtureSpec())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
smp.render(seed=1, first=0, count=n)
torch.cuda.synchronize()
for r in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    smp.render(seed=2 + r, first=0, count=n)
    e1.record()
    torch.cuda.synchronize()
    print(f"count={n} event_ms={e0.elapsed_time(e1):.2f} wall_ms={(time.perf_counter() - t0) * 1e3:.2f}", flush=True)
