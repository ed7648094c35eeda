"""Throughput of K back-to-back batches: one stream vs two streams with
double-buffered workspaces (dev tool)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_08052_b200 import engine, workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
depth = int(sys.argv[3]) if len(sys.argv) > 3 else 2
w = workloads.config2(n)
pb = engine.prepare(16000, w.jobs, w.mics)
dbs = [engine.DeviceBatch(pb) for _ in range(depth)]
outs = [db.alloc_outputs(True) for db in dbs]
streams = [torch.cuda.Stream() for _ in range(depth)]


def run(serial):
    main = torch.cuda.current_stream()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for s in streams:
        s.wait_event(e0)
    for k in range(K):
        i = 0 if serial else k % depth
        dbs[i].launch(*outs[i], stream=streams[0] if serial else streams[i])
    for s in streams:
        ev = torch.cuda.Event()
        ev.record(s)
        main.wait_event(ev)
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for _ in range(2):
    run(True)
    run(False)
ts, tp = run(True), run(False)
print(f"rooms={n} K={K} depth={depth} serial={ts / K * 1e3:.0f}us/step pipelined={tp / K * 1e3:.0f}us/step "
      f"rir/s serial={n * K / ts * 1e3:.0f} pipelined={n * K / tp * 1e3:.0f}")
