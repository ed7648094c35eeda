"""Seeded BASELINE workloads: ranges, determinism, and that every
generated job passes the reference's validation (frir_jobs_prepare)."""

import numpy as np
import pytest

from paper_2304_08052_b200 import engine, workloads


@pytest.mark.parametrize("cfg,rooms", [(2, 300), (3, 100), (4, 60), (5, 200)])
def test_workload_valid_and_in_range(cfg, rooms):
    w = workloads.build(cfg, rooms)
    pb = engine.prepare(w.sample_rate, w.jobs, w.mics)  # raises on any invalid job
    j = pb.jobs
    lo, hi = {2: (1024, 4096), 3: (1024, 4096), 4: (8192, 16384), 5: (1024, 8192)}[cfg]
    assert j["n_images"].min() >= lo and j["n_images"].max() <= hi
    t60 = {2: (0.1, 0.7), 3: (0.2, 1.0), 4: (1.0, 1.5), 5: (0.1, 0.7)}[cfg]
    assert j["t60"].min() >= t60[0] and j["t60"].max() <= t60[1]
    m = {2: 6, 3: 8, 4: 16, 5: 32}[cfg]
    assert (j["n_mics"] == m).all()
    assert (j["rr_max"] >= 1.0).all()
    assert (j["d0"] >= {2: 0.3, 3: 1.0, 4: 0.6, 5: 0.3}[cfg] - 1e-9).all()
    # n2 == ceil(T60 * fs)
    assert np.array_equal(j["n2"], np.ceil(j["t60"] * w.sample_rate).astype(np.int64))


def test_config1_is_the_reference_scene(golden):
    w = workloads.config1()
    g = golden["cfg1"]
    assert np.allclose(w.mics, g["mics"])
    assert np.allclose([w.jobs[0]["d0"], w.jobs[0]["az"], w.jobs[0]["el"]], g["source"][0], rtol=0, atol=0)


def test_deterministic():
    a, b = workloads.config3(5), workloads.config3(5)
    assert a.jobs.tobytes() == b.jobs.tobytes() and a.mics.tobytes() == b.mics.tobytes()
