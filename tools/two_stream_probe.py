"""Does splitting a batch over two streams overlap one half's geom/sort/tail
with the other half's render tail? (dev tool)"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_08052_b200 import engine, workloads  # noqa: E402


def timed(fn, reps=7):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return sorted(out)[reps // 2]


n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
parts = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = workloads.config2(n)
one = engine.DeviceBatch(engine.prepare(16000, w.jobs, w.mics))
o1 = one.alloc_outputs(True)
subs, outs, streams = [], [], []
for p in range(parts):
    lo, hi = n * p // parts, n * (p + 1) // parts
    jb = w.jobs[lo:hi]
    db = engine.DeviceBatch(engine.prepare(16000, jb, w.mics))
    subs.append(db)
    outs.append(db.alloc_outputs(True))
    streams.append(torch.cuda.Stream())


def run_one():
    one.launch(*o1)


def run_split():
    main = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(main)
    for db, o, s in zip(subs, outs, streams):
        s.wait_event(ev)
        db.launch(*o, stream=s)
    for s in streams:
        e = torch.cuda.Event()
        e.record(s)
        main.wait_event(e)


for _ in range(3):
    run_one()
    run_split()
t1 = timed(run_one)
t2 = timed(run_split)
print(f"rooms={n} one={t1 * 1e3:.0f}us split{parts}={t2 * 1e3:.0f}us rir/s one={n / t1 * 1e3:.0f} split={n / t2 * 1e3:.0f}")
