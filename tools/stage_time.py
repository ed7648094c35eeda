"""Per-stage device times of one config (dev tool; not a benchmark).

Times GEOM, GEOM+DELAY and ALL with CUDA events (best of N) and prints the
differences, so two builds can be compared with FRIR_LIB=... .
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_08052_b200 import _abi, engine, workloads  # noqa: E402


def best_ms(fn, reps):
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    out.sort()
    return out[len(out) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--rooms", type=int, default=None)
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--no-early", action="store_true")
    ap.add_argument("--ism", type=int, default=0, help="ISM rows of bench_rows.py (this many rooms x 3 sources)")
    a = ap.parse_args()
    if a.ism:
        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        import bench_rows
        from paper_2304_08052_b200 import ism

        fs, jobs, mics, draws, _ = ism.ism_prepare(bench_rows.ism_configs(a.ism))
        db = engine.DeviceBatch(engine.prepare(fs, jobs, mics, draws=draws))
        a.no_early = True
        a.cfg = f"-ism{a.ism}"
        n_rirs = len(jobs)
    else:
        w = workloads.build(a.cfg, a.rooms)
        db = engine.DeviceBatch(engine.prepare(w.sample_rate, w.jobs, w.mics))
        n_rirs = w.n_rirs
    full, early, direct = db.alloc_outputs(not a.no_early)
    for _ in range(3):
        db.launch(full, early, direct)
    torch.cuda.synchronize()
    t = {}
    for name, st in (("geom", 1), ("geom+sort", 3), ("all", 7)):
        t[name] = best_ms(lambda: db.launch(full, early, direct, stages=st), a.reps)
    print(f"lib={_abi.LIB_PATH if 'FRIR_LIB' not in __import__('os').environ else __import__('os').environ['FRIR_LIB']} "
          f"cfg{a.cfg} rirs={n_rirs} geom={t['geom']*1e3:.0f}us sort={(t['geom+sort']-t['geom'])*1e3:.0f}us "
          f"render={(t['all']-t['geom+sort'])*1e3:.0f}us total={t['all']*1e3:.0f}us "
          f"rir/s={n_rirs / t['all'] * 1e3:.0f}", flush=True)


if __name__ == "__main__":
    main()
