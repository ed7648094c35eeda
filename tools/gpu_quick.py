"""Quick GPU parity probe against the committed goldens (dev tool)."""

import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2304_08052_b200 import engine, workloads  # noqa: E402
from paper_2304_08052_b200.scene import linear_array  # noqa: E402

G = ROOT / "tests" / "golden"


def rel(a, b, peak):
    return float(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)).max() / peak)


def main():
    c1 = np.load(G / "cfg1.npz")
    w = workloads.config1()
    for mode in ("native", "oracle"):
        draws = None
        if mode == "oracle":
            draws = (c1["dist"], c1["az"], c1["el"], c1["refl"])
        res = engine.simulate_jobs(16000, w.jobs, w.mics, include_early=True, draws=draws)
        torch.cuda.synchronize()
        full = res.job_view(0).cpu().numpy()
        early = res.job_view(0, "early").cpu().numpy()
        ef = max(rel(full[m], c1["full"][m], c1["full_peak"][m]) for m in range(4))
        ee = max(rel(early[m], c1["early"][m], c1["early_peak"][m]) for m in range(4))
        print(f"cfg1 {mode}: full {ef:.3e} early {ee:.3e} direct {res.direct_index.cpu().numpy()} vs {c1['direct']}")
    cases = np.load(G / "cases.npz")
    meta = json.loads((G / "cases.json").read_text())
    for ci, mcase in enumerate(meta):
        pre = f"c{ci}_"
        mics = cases[pre + "mics"]
        jobs = engine.new_jobs(1)
        jobs["room"] = mcase["room"]
        jobs["center"] = mics.mean(axis=0)
        jobs["d0"], jobs["az"], jobs["el"] = mcase["source"]
        jobs["t60"] = mcase["t60"]
        jobs["seed"] = mcase["seed"]
        jobs["n_images"] = mcase["num_images"]
        jobs["n_mics"] = len(mics)
        for mode in ("native", "oracle"):
            draws = None
            if mode == "oracle":
                draws = tuple(cases[pre + k] for k in ("dist", "az", "el", "refl"))
            res = engine.simulate_jobs(mcase["fs"], jobs, mics, include_early=True, draws=draws)
            full = res.job_view(0).cpu().numpy()
            early = res.job_view(0, "early").cpu().numpy()
            pk = cases[pre + "peak"]
            print(f"case {ci} fs={mcase['fs']} t60={mcase['t60']} I={mcase['num_images']} {mode}: "
                  f"full {rel(full, cases[pre + 'full'], pk[0]):.3e} early {rel(early, cases[pre + 'early'], pk[1]):.3e} "
                  f"direct ok {np.array_equal(res.direct_index.cpu().numpy(), cases[pre + 'direct'])}")
    # throughput probe on config 2
    w2 = workloads.config2(1024)
    pb = engine.prepare(16000, w2.jobs, w2.mics)
    db = engine.DeviceBatch(pb)
    full, early, direct = db.alloc_outputs(True)
    for _ in range(3):
        db.launch(full, early, direct)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 10
    for _ in range(n):
        db.launch(full, early, direct)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"cfg2 1024 rooms: {ms:.3f} ms/batch -> {1024 / ms * 1e3:.0f} RIR/s")


if __name__ == "__main__":
    main()
