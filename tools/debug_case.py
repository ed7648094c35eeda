"""Dev tool: where does one random scene's GPU output deviate from the oracle."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from oracle import framrir_port as P  # noqa: E402
from paper_2304_08052_b200 import engine  # noqa: E402

def _random_job(rng):
    fs = int(rng.choice([8000, 11025, 16000, 22050, 24000, 32000, 44100, 48000]))
    t60 = float(rng.uniform(0.05, 0.35))
    m = int(rng.integers(1, 6))
    room = rng.uniform([3.0, 3.0, 2.4], [9.0, 9.0, 4.0])
    mics = rng.uniform(-0.12, 0.12, size=(m, 3))
    center = mics.mean(axis=0)
    r = P.wall_reflection(room, t60)
    d_min = max(0.02, 343.0 * t60 / (1000.0 * r) * 1.05)
    d0 = float(rng.uniform(d_min, d_min + 2.5))
    n = int(rng.choice([0, 1, 7, 64, 333, 1024, 2500]))
    return P.Job(room=tuple(room), mics=mics, center=center,
                 source=(d0, float(rng.uniform(0, 2 * np.pi)), float(rng.uniform(-1.2, 1.2))),
                 t60=t60, sample_rate=fs, num_images=n, seed=int(rng.integers(2**63)),
                 source_index=int(rng.integers(0, 3)))

job = _random_job(np.random.default_rng(int(sys.argv[1])))
full_o, early_o, _ = P.render(job)
jobs = engine.new_jobs(1)
jobs["room"] = job.room; jobs["center"] = job.center
jobs["d0"], jobs["az"], jobs["el"] = job.source
jobs["t60"] = job.t60; jobs["seed"] = job.seed; jobs["source_index"] = job.source_index
jobs["n_images"] = job.num_images; jobs["n_mics"] = len(job.mics)
res = engine.simulate_jobs(job.sample_rate, jobs, job.mics, include_early=True)
early = res.job_view(0, "early").cpu().numpy()
full = res.job_view(0).cpu().numpy()
for m in range(len(job.mics)):
    for name, a, b in (("full", full[m], full_o[m]), ("early", early[m], early_o[m])):
        err = np.abs(a - b) / np.abs(b).max()
        bad = np.flatnonzero(err > 1e-6)
        print(m, name, "max", err.max(), "n2", len(b), "bad idx", bad[:5], bad[-5:] if len(bad) else "", "count", len(bad))
