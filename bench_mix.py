"""Benchmark of the spatialise-and-mix consumer.

One step = B on-the-fly training utterances with the reference's default
MixtureSpec (2 speakers + point noise, 4-mic linear array, 4 s at 16 kHz,
2048 images, T60 ~ U[0.1, 0.7]): render the (2 + 1) x 4-channel full + early
RIRs on the GPU, then convolve, scale and mix on the GPU.  Dry signals and
scenes are seeded synthetic inputs resident in HBM before the timed region.
Prints one JSON line; ``mix_only_ms`` times the mixing half alone.

cpu_baseline: the reference algorithm on the host cores -- oracle/framrir_port
(RIRs) + oracle/mixture_port (scipy FP64 fftconvolve mixing) over a bounded
sample of the same utterances, one process per core.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def make_workload(n_items: int, seed: int = 0):
    """Scenes drawn like mixture.sample_scene (reference mixture.py:171-213) and
    seeded dry signals; returns (spec, scenes, params, dry (B,S,N), noise (B,N))."""
    from paper_2304_08052_b200 import mixture as MX

    spec = MX.MixtureSpec()
    scenes, params = [], []
    for i in range(n_items):
        rng = np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, i))))
        sc, pr = MX.sample_scene(spec, rng)
        scenes.append(sc)
        params.append(pr)
    n = int(spec.utterance_seconds * spec.sample_rate)
    g = np.random.default_rng(seed + 1)
    dry = g.standard_normal((n_items, spec.n_speakers, n)).astype(np.float32)
    noise = g.standard_normal((n_items, n)).astype(np.float32)
    return spec, scenes, params, dry, noise


def _cpu_item(args):
    from oracle import framrir_port as P
    from oracle import mixture_port as MP

    spec_dict, scene, prm, dry, noise, offsets, sir, snr = args
    from paper_2304_08052_b200 import mixture as MX  # the same host material generator

    pool = MX.SyntheticPool()
    rng = np.random.default_rng(0)
    for _ in range(len(dry) + 1):
        pool.draw(rng, len(noise), 16000)
    rirs_f, rirs_e = [], []
    for job in P.jobs_from_scene(prm, scene):
        full, early, _ = P.render(job)
        rirs_f.append(full)
        rirs_e.append(early)
    MP.mix([d.astype(float) for d in dry], noise.astype(float), rirs_f, rirs_e[:-1], offsets, sir, snr)
    return 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--items", type=int, default=64)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu-items", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    a = ap.parse_args()

    import torch

    from paper_2304_08052_b200 import engine
    from paper_2304_08052_b200 import mixture as MX

    dev = torch.device("cuda", 0)
    spec, scenes, params, dry_h, noise_h = make_workload(a.items)
    B, S, N = dry_h.shape
    # per-item offsets / SIR / SNR drawn as the reference does (mixture.py:245-263)
    rng = np.random.default_rng(7)
    offsets, sir, snr = [], [], []
    for b in range(B):
        offsets.append(MX._draw_offsets([dry_h[b, k] for k in range(S)], spec, rng))
        sir.append([float(rng.uniform(*spec.sir_db)) for _ in range(S - 1)])
        snr.append(float(rng.uniform(*spec.snr_db)))
    jobs, mics = MX.scene_batch_jobs(scenes, params)
    pb = engine.prepare(spec.sample_rate, jobs, mics, padded=True)
    db = engine.DeviceBatch(pb, device=dev)
    full, early, direct = db.alloc_outputs(True)
    M = len(scenes[0].mic_positions)
    stride = int(pb.jobs[0]["out_stride"])
    rir_len = pb.jobs["n2"].reshape(B, S + 1)[:, 0]
    dry = torch.as_tensor(dry_h, device=dev)
    noise = torch.as_tensor(noise_h, device=dev)

    def step(mix_only=False):
        if not mix_only:
            db.launch(full, early, direct)
        rf = full.view(B, S + 1, M, stride)
        re = early.view(B, S + 1, M, stride)
        return MX.mix_device(dry, [[N] * S] * B, offsets, noise, [N] * B, rf, re, rir_len, sir, snr)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    for e0, e1 in ev:
        e0.record()
        step()
        e1.record()
    torch.cuda.synchronize()
    ms = float(np.median([e0.elapsed_time(e1) for e0, e1 in ev]))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        step(mix_only=True)
    e1.record()
    torch.cuda.synchronize()
    mix_ms = e0.elapsed_time(e1) / a.steps

    line = {
        "metric": "on-the-fly training mixtures/sec (RIRs + spatialise-and-mix), 1 B200",
        "value": B / ms * 1e3, "unit": "mixtures/s", "n_gpus": 1, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms, "mix_only_ms": mix_ms, "higher_is_better": True, "dtype": "f32 (FP64 powers/gains)",
        "data": "synthetic: MixtureSpec() scenes (sample_scene draws), seeded Gaussian dry signals",
        "config": {"workload": f"{B} utterances: 2 speakers + noise, 4 mics, 4 s @ 16 kHz, 2048 images, "
                               "full+early RIRs, frir_mix_convolve (own 8192-point partitioned FFT convolution) + frir_mix_* kernels"},
    }
    # device scene sampler: rooms drawn on the GPU straight
    # into render jobs, then all their RIRs in one launch
    from paper_2304_08052_b200.sampler import DeviceSceneSampler

    smp = DeviceSceneSampler(spec)
    nroom = 1024
    smp.render(seed=11, first=0, count=nroom)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for r in range(3):
        smp.render(seed=12 + r, first=0, count=nroom)
    s1.record()
    torch.cuda.synchronize()
    ms_s = s0.elapsed_time(s1) / 3
    line["device_sampler"] = {"value": nroom * (S + 1) / ms_s * 1e3, "unit": "RIR/s",
                              "ms_per_batch": ms_s,
                              "workload": f"{nroom} sample_scene draws on the device -> {nroom * (S + 1)} "
                                          f"{M}-channel full+early RIRs (2048 images), one launch"}
    # e2e: the public drop-in generate_batch -- host draws in the reference's
    # order on all host cores (threads), RIRs + mix on the device, results
    # copied back to host numpy arrays -- wall clock per batch
    cores = len(os.sched_getaffinity(0))
    MX.generate_batch(B, spec, seed=1, workers=cores)  # warm-up (pinned host blocks get cached)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = MX.generate_batch(B, spec, seed=2, workers=cores)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    d2h = sum(r.mixture.nbytes + sum(x.nbytes for x in r.sources) + sum(x.nbytes for x in r.early_sources)
              + r.noise.nbytes for r in res)
    h2d = B * (S + 1) * N * 4
    line["e2e"] = {"value": B / wall, "unit": "mixtures/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                   "path": f"mixture.generate_batch({B}, MixtureSpec(), workers={cores}): host draws (threads) "
                           "+ device RIRs + device mix + D2H of all outputs"}
    if not a.no_cpu_baseline:
        n = min(a.cpu_items, B)
        cores = len(os.sched_getaffinity(0))
        args = [({}, scenes[b], params[b], dry_h[b], noise_h[b], offsets[b], sir[b], snr[b]) for b in range(n)]
        os.environ.setdefault("OMP_NUM_THREADS", "1")
        t0 = time.perf_counter()
        with ProcessPoolExecutor(max_workers=min(cores, n)) as ex:
            list(ex.map(_cpu_item, args))
        wall = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": n / wall, "unit": "mixtures/s", "cores": min(cores, n), "kind": "port",
                                "sample": f"first {n} utterances: SyntheticPool draws + oracle/framrir_port RIRs + "
                                          f"oracle/mixture_port mixing (numpy/scipy FP64), wall {wall:.2f} s"}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
