"""sha256 of the rendered outputs of a few workloads (dev tool): run under two
builds / settings and compare the digests to prove bit-identical results."""
import hashlib
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_08052_b200 import engine, workloads  # noqa: E402

for cfg, rooms in ((2, 1024), (3, 64), (4, 8), (5, 512)):
    w = workloads.build(cfg, rooms)
    res = engine.simulate_jobs(w.sample_rate, w.jobs, w.mics, include_early=True)
    torch.cuda.synchronize()
    h = hashlib.sha256()
    for t in (res.full, res.early, res.direct_index):
        h.update(t.cpu().numpy().tobytes())
    print(f"cfg{cfg} {h.hexdigest()[:24]}")
