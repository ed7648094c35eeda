"""Small end-to-end run for compute-sanitizer (dev tool): golden cases in both
modes plus a few rooms of every BASELINE config, full + early."""

import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2304_08052_b200 import engine, workloads  # noqa: E402

G = ROOT / "tests" / "golden"
cases = np.load(G / "cases.npz")
meta = json.loads((G / "cases.json").read_text())
for ci, m in enumerate(meta):
    mics = cases[f"c{ci}_mics"]
    jobs = engine.new_jobs(1)
    jobs["room"] = m["room"]
    jobs["center"] = mics.mean(axis=0)
    jobs["d0"], jobs["az"], jobs["el"] = m["source"]
    jobs["t60"], jobs["seed"], jobs["n_images"], jobs["n_mics"] = m["t60"], m["seed"], m["num_images"], len(mics)
    for early in (True, False):
        engine.simulate_jobs(m["fs"], jobs, mics, include_early=early)
for cfg, n in ((2, 3), (3, 1), (4, 1), (5, 1), (5, 384)):  # (5, 384): 12,288 channels, the early pass
    w = workloads.build(cfg, n)
    if n == 384:
        w.jobs["n_images"][7] = 8192  # the longest register-staged sort rows (8,193)
    engine.simulate_jobs(w.sample_rate, w.jobs, w.mics, include_early=True, padded=(cfg == 3))
torch.cuda.synchronize()
from paper_2304_08052_b200 import _abi  # noqa: E402

line = _abi.lib().frir_debug_status()
print("sanitize run ok; first failed bounds check at line", line)
sys.exit(1 if line else 0)
