"""Where does a segmented channel differ from the oracle? (dev tool)

Renders one long-row job (rows > kSegRows, so the render splits its
channels into segments joined by the seam kernel) and prints, per channel and
variant, the max relative error and the sample where it occurs.
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import framrir_port as P  # noqa: E402
from paper_2304_08052_b200 import engine  # noqa: E402


def main():
    fs, t60, n = (int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (48000, 0.05, 17000)
    mics = np.array([[0.0, 0.0, 0.0], [0.1, 0.0, 0.0]])
    jobs = engine.new_jobs(1)
    jobs["room"] = (4.0, 4.0, 3.0)
    jobs["center"] = mics.mean(axis=0)
    jobs["d0"], jobs["az"], jobs["el"] = 0.9, 1.0, 0.1
    jobs["t60"] = t60
    jobs["seed"] = 5
    jobs["n_images"] = n
    jobs["n_mics"] = 2
    res = engine.simulate_jobs(fs, jobs, mics)
    job = P.Job(room=(4.0, 4.0, 3.0), mics=mics, center=mics.mean(axis=0), source=(0.9, 1.0, 0.1),
                t60=t60, sample_rate=fs, num_images=n, seed=5)
    full_o, early_o, _ = P.render(job)
    for name, ours, ref in (("full", res.job_view(0).cpu().numpy(), full_o),
                            ("early", res.job_view(0, "early").cpu().numpy(), early_o)):
        for m in range(2):
            d = np.abs(ours[m] - ref[m]) / np.abs(ref[m]).max()
            i = int(d.argmax())
            big = np.nonzero(d > 1e-6)[0]
            print(f"{name} m={m} n2={ref.shape[1]} max_rel={d.max():.3e} at {i} (window {(i + 32) // 32}); "
                  f">1e-6 at {big[:5].tolist()}..{big[-3:].tolist() if len(big) else []} ({len(big)} samples)")


if __name__ == "__main__":
    main()
