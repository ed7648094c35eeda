"""Where a drop-in simulate_rir call spends its time (dev tool): cProfile of
200 config-1 calls on the GPU."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2304_08052_b200 as F  # noqa: E402

params = F.SimParams(t60=0.5, num_images=2048, seed=0)
scene = F.Scene(room_dims=(6.0, 5.0, 3.0), mic_positions=F.linear_array([0.05, 0.05, 0.05]),
                sources=[(1.4456832294801, 2.356194490192345, 0.20903329903452)])
for _ in range(10):
    F.simulate_rir(params, scene)
t0 = time.perf_counter()
for _ in range(200):
    F.simulate_rir(params, scene)
print("ms per call", (time.perf_counter() - t0) * 5)
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    F.simulate_rir(params, scene)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
