import sys, time, torch
sys.path.insert(0, '.')
from paper_2304_08052_b200 import engine, workloads
dev = torch.device('cuda', 0)
w = workloads.build(2, 1024, start=0)
for chunks in (4, 8, 16):
    pipe = engine.HostPipeline(w.sample_rate, w.jobs, w.mics, include_early=True, chunks=chunks, device=dev)
    pipe.run(); torch.cuda.synchronize()
    ts = []
    for _ in range(6):
        t0 = time.perf_counter(); pipe.run(); ts.append(time.perf_counter() - t0)
    ts2 = []
    for _ in range(6):
        t0 = time.perf_counter(); pipe.run(revalidate=False); ts2.append(time.perf_counter() - t0)
    print(chunks, 'ms', round(1e3 * min(ts), 3), round(1e3 * sorted(ts)[3], 3), 'noreval', round(1e3 * min(ts2), 3), 'MB', pipe.d2h_bytes / 1e6)
