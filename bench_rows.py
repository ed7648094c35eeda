"""Benchmarks of the widened rows without one of their own (SURVEY §8f rows 2
and 4); one JSON line each.

ism    -- the GPU image-source method on the reference's own ISM benchmark
          workload (framrir/bench.py:116-158 bench_ism: MixtureSpec rooms,
          3 sources per room uniform in [0.3, L - 0.3], the mic array at the
          room centre, max_order resolved from c0 * T60).  value: RIRs/s of
          the device launch (lattice enumerated in K1); e2e: ism.ism_batch
          (job table + H2D + render + D2H to numpy); cpu_baseline: oracle/ism_port (the
          reference's dense np.add.at + scipy chain) on a bounded sample, one
          process per core.
decay  -- batched Schroeder curves + T60 (frir_edc + frir_t60) over the
          config-2 RIRs (1024 rooms x 6 mics, full variant) resident in HBM:
          channels/s; cpu_baseline: oracle/decay_port on a bounded sample.

Inputs are seeded synthetic scenes; no dataset is needed.
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


def ism_configs(n_rooms: int, sources: int = 3, seed: int = 0):
    """bench_ism's workload shape (reference bench.py:116-140) from our host
    mirror of sample_scene."""
    from paper_2304_08052_b200 import mixture as MX
    from paper_2304_08052_b200.ism import IsmConfig

    spec = MX.MixtureSpec()
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_rooms):
        scene, params = MX.sample_scene(spec, np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, i)))))
        dims = np.asarray(scene.room_dims)
        mics = np.asarray(scene.mic_positions) + dims / 2.0
        for _ in range(sources):
            src = rng.uniform(0.3, dims - 0.3)
            out.append(IsmConfig(room_dims=tuple(dims), source_position=tuple(src), mic_positions=mics,
                                 t60=params.t60, sample_rate=params.sample_rate))
    return out


def _cpu_ism(c):
    from oracle import ism_port as IP

    IP.render(c.room_dims, c.source_position, c.mic_positions, c.t60, sample_rate=c.sample_rate,
              order=c.max_order, duration=c.duration, reflection=c.reflection)
    return 1


def _cpu_decay(rows):
    from oracle import decay_port as DP

    for r in rows:
        DP.t60(r, 16000)
    return len(rows)


def _events(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def bench_ism(a, torch, dev):
    from paper_2304_08052_b200 import engine, ism

    cfgs = ism_configs(a.ism_rooms)
    fs, jobs, mics, draws, _ = ism.ism_prepare(cfgs)
    pb = engine.prepare(fs, jobs, mics, draws=draws)
    db = engine.DeviceBatch(pb, device=dev)
    full, early, direct = db.alloc_outputs(False)
    for _ in range(a.warmup):
        db.launch(full, None, direct)
    torch.cuda.synchronize()
    e0, e1 = _events(torch)
    e0.record()
    for _ in range(a.steps):
        db.launch(full, None, direct)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    n_items = int(pb.batch.total_items)
    # end to end through the public API
    ism.ism_batch(cfgs[:4])
    t0 = time.perf_counter()
    ism.ism_batch(cfgs)
    wall = time.perf_counter() - t0
    line = {
        "metric": "ISM RIRs/sec (reference bench_ism workload), 1 B200", "value": len(cfgs) / ms * 1e3,
        "unit": "RIR/s", "n_gpus": 1, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
        "higher_is_better": True, "dtype": "f32 (FP64 geometry, delays and LP state)",
        "data": "synthetic: MixtureSpec rooms (sample_scene draws), sources uniform in [0.3, L - 0.3]",
        "config": {"workload": f"{len(cfgs)} ISM RIRs ({a.ism_rooms} rooms x 3 sources, 4 mics, 16 kHz, "
                               f"max_order from c0*T60), {n_items / len(cfgs) / 4:.0f} lattice images per RIR "
                               "enumerated on the device", "items_per_step": n_items},
        "e2e": {"value": len(cfgs) / wall, "unit": "RIR/s", "ms_per_step": wall * 1e3,
                "h2d_bytes_per_step": int(jobs.nbytes + mics.nbytes + (sum(d.nbytes for d in draws) if draws else 0)),
                "d2h_bytes_per_step": int(full.numel() * 4 + direct.numel() * 4),
                "path": "ism.ism_batch: job table H2D, lattice enumerated on the device, render, D2H to numpy"},
        "gpu_launches": int(engine_launches(db, False)) * a.steps,
    }
    if not a.no_cpu_baseline:
        n = min(a.cpu_items, len(cfgs))
        cores = len(os.sched_getaffinity(0))
        t0 = time.perf_counter()
        with ProcessPoolExecutor(max_workers=min(cores, n)) as ex:
            list(ex.map(_cpu_ism, cfgs[:n]))
        w = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": n / w, "unit": "RIR/s", "cores": min(cores, n), "kind": "port",
                                "sample": f"first {n} configurations through oracle/ism_port "
                                          f"(dense np.add.at + scipy chain, FP64), wall {w:.2f} s"}
    return line


def engine_launches(db, early):
    from paper_2304_08052_b200 import _abi

    return _abi.lib().frir_launch_count(db.plan.handle, __import__("ctypes").byref(db.batch), int(early))


def bench_decay(a, torch, dev):
    from paper_2304_08052_b200 import decay, engine, workloads

    w = workloads.build(2, a.decay_rooms, start=0)
    pb = engine.prepare(w.sample_rate, w.jobs, w.mics, padded=True)
    db = engine.DeviceBatch(pb, device=dev)
    full, _, direct = db.alloc_outputs(False)
    db.launch(full, None, direct)
    stride = int(pb.jobs[0]["out_stride"])
    C = int(pb.batch.total_channels)
    rows = full.view(C, stride)
    lens = np.repeat(pb.jobs["n2"], pb.jobs["n_mics"]).astype(np.int32)
    for _ in range(a.warmup):
        decay.measure_t60_batch(rows, 16000, lengths=lens)
    torch.cuda.synchronize()
    e0, e1 = _events(torch)
    e0.record()
    for _ in range(a.steps):
        t60 = decay.measure_t60_batch(rows, 16000, lengths=lens)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    samples = int(lens.sum())
    line = {
        "metric": "T60 measurements/sec (Schroeder EDC + crossing per channel), 1 B200",
        "value": C / ms * 1e3, "unit": "channels/s", "n_gpus": 1, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms, "higher_is_better": True, "dtype": "f64 (EDC sums in numpy's order)",
        "data": "synthetic: config-2 rooms rendered on the device",
        "config": {"workload": f"{C} channels ({a.decay_rooms} config-2 rooms x 6 mics), "
                               f"{samples / C:.0f} samples per channel on average",
                   "samples_per_step": samples},
        "nan_channels": int(torch.isnan(t60).sum()),
    }
    if not a.no_cpu_baseline:
        host = rows.cpu().numpy()
        n = min(a.cpu_channels, C)
        sample = [host[i, :lens[i]].copy() for i in range(n)]
        cores = len(os.sched_getaffinity(0))
        parts = [sample[i::cores] for i in range(cores)]
        t0 = time.perf_counter()
        with ProcessPoolExecutor(max_workers=cores) as ex:
            list(ex.map(_cpu_decay, parts))
        wl = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": n / wl, "unit": "channels/s", "cores": cores, "kind": "port",
                                "sample": f"first {n} channels through oracle/decay_port (numpy), wall {wl:.2f} s"}
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--ism-rooms", type=int, default=128)
    ap.add_argument("--decay-rooms", type=int, default=1024)
    ap.add_argument("--cpu-items", type=int, default=16)
    ap.add_argument("--cpu-channels", type=int, default=2048)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--only", choices=["ism", "decay"])
    a = ap.parse_args()

    import torch

    dev = torch.device("cuda", 0)
    if a.only in (None, "ism"):
        print(json.dumps(bench_ism(a, torch, dev)), flush=True)
    if a.only in (None, "decay"):
        print(json.dumps(bench_decay(a, torch, dev)), flush=True)


if __name__ == "__main__":
    main()
