"""Run a config batch a few times (profiling driver; not a benchmark)."""

import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_08052_b200 import engine, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--rooms", type=int, default=None)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--no-early", action="store_true")
    a = ap.parse_args()
    w = workloads.build(a.cfg, a.rooms)
    db = engine.DeviceBatch(engine.prepare(w.sample_rate, w.jobs, w.mics))
    full, early, direct = db.alloc_outputs(not a.no_early)
    for _ in range(a.iters):
        db.launch(full, early, direct)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    db.launch(full, early, direct)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"cfg{a.cfg} rirs={w.n_rirs} ms={ms:.3f} rir_per_s={w.n_rirs / ms * 1e3:.0f}")


if __name__ == "__main__":
    main()
