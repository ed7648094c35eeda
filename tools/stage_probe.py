"""Run the three stages separately with a sync after each (dev tool)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_08052_b200 import engine, workloads, _abi  # noqa: E402
print("lib", _abi.LIB_PATH, flush=True)
w = workloads.config1()
db = engine.DeviceBatch(engine.prepare(16000, w.jobs, w.mics))
full, early, direct = db.alloc_outputs(True)
for st in (1, 2, 4):
    db.launch(full, early, direct, stages=st)
    try:
        torch.cuda.synchronize()
        print("stage", st, "ok; check line", _abi.lib().frir_debug_status(), flush=True)
    except Exception as e:
        print("stage", st, "FAILED", str(e)[:200], flush=True)
        break
