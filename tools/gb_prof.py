import sys, time, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2304_08052_b200 import mixture as MX
spec = MX.MixtureSpec()
cores = len(os.sched_getaffinity(0))
MX.generate_batch(64, spec, seed=1, workers=cores)
torch.cuda.synchronize()
import cProfile, pstats
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
res = MX.generate_batch(64, spec, seed=2, workers=cores)
torch.cuda.synchronize()
pr.disable()
print('wall', time.perf_counter() - t0)
pstats.Stats(pr).sort_stats('cumulative').print_stats(25)
