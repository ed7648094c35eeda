"""Render time vs image count on config-2 rooms (dev tool): separates the
per-item cost from the per-window/per-channel overhead."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_08052_b200 import engine, workloads  # noqa: E402


def t_ms(db, full, early, stages, reps=9):
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        db.launch(full, early, direct=None, stages=stages) if False else db.launch(full, early, db_direct, stages=stages)
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return sorted(out)[reps // 2]


for early_on in (True, False):
    for n in (256, 1024, 2048, 4096):
        w = workloads.config2()
        w.jobs["n_images"] = n
        db = engine.DeviceBatch(engine.prepare(w.sample_rate, w.jobs, w.mics))
        full, early, db_direct = db.alloc_outputs(early_on)
        db.launch(full, early, db_direct)
        torch.cuda.synchronize()
        tr = t_ms(db, full, early, 4)
        items = int((w.jobs["n_images"] + 1).astype("int64").dot(w.jobs["n_mics"]))
        print(f"early={early_on} I={n} items={items} render_us={tr*1e3:.0f} ns_per_item={tr*1e6/items:.2f}", flush=True)
