"""Benchmark: multi-channel FRAM-RIRs per second on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

One step = render one pass of the configured BASELINE workload, full + early
variants, native (device Philox) draws.  The default is the headline workload
the metric is quoted on, BASELINE configs[4] = config 5: 65,536 seeded rooms
(32 ad-hoc mics, 16 kHz, I ~ U{1024..8192}) split over the GPUs (strong
scaling), each rank streaming 4,096-room launches.

Multi-GPU: one process per GPU, rooms sharded by global room index, no
collective on the data path; timing is the max over ranks of CUDA-event
durations.  Under torchrun the ranks come from the environment; run directly
with ``--gpus N > 1`` and bench.py spawns the N ranks itself (same env
contract: RANK / LOCAL_RANK / WORLD_SIZE / MASTER_ADDR=127.0.0.1).

``--impl reference`` times the reference's own CPU implementation of the path
on the host cores (rank 0 only): the unmodified ``framrir.simulate_rir`` from
``baseline/_ref`` when it is installed there, else the oracle port
(oracle/framrir_port.py, the same numpy + scipy algorithm), over a prefix of
the SAME rooms.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
REF_DIR = ROOT / "baseline" / "_ref"

METRIC = "multi-channel RIRs/sec at 1/2/4/8 B200; % of FP32 and HBM roofline"
L2_BYTES = 126 * 2**20
DEFAULT_CONFIG = 5
FP32_THEORETICAL_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4 at the 1965 MHz max SM clock

CONFIGS = {
    1: dict(rooms=1, desc="cfg1: 1 room 6x5x3 m, T60 0.5 s, 4-mic linear 5 cm, I=2048, 16 kHz"),
    2: dict(rooms=1024, desc="cfg2: 1024 random rooms/GPU, T60~U[0.1,0.7], 6-mic 5 cm circle, I~U{1024..4096}, 16 kHz"),
    3: dict(rooms=4096, desc="cfg3: 4096 rooms x 3 sources/GPU, T60~U[0.2,1.0], 8-mic 10 cm circle, I~U{1024..4096}, 16 kHz"),
    4: dict(rooms=512, desc="cfg4: 512 rooms x 2 sources/GPU, 48 kHz, T60~U[1.0,1.5], 16-mic 4x4 grid, I~U{8192..16384}"),
    5: dict(rooms=65536, desc="cfg5: 65536 rooms sharded over GPUs, 32 ad-hoc mics, T60~U[0.1,0.7], I~U{1024..8192}, 16 kHz"),
}
SOURCES_PER_ROOM = {1: 1, 2: 1, 3: 3, 4: 2, 5: 1}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- launcher
def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(n: int, cmd: list, env_extra: dict | None = None, timeout: float | None = None) -> int:
    """Run ``cmd`` as ``n`` ranks (one process per GPU), torchrun's env contract:
    RANK = LOCAL_RANK = i, WORLD_SIZE = LOCAL_WORLD_SIZE = n, MASTER_ADDR =
    127.0.0.1 and a free MASTER_PORT.  Children inherit stdout/stderr (rank 0
    prints the JSON line).  If one rank fails the others are terminated (by
    their own PIDs).  Returns the first non-zero exit code, else 0.  Mirrors
    the reference's process fan-out over independent items
    (/root/reference/pkg/src/framrir/mixture.py:385-391)."""
    port = free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   GROUP_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), **(env_extra or {}))
        procs.append(subprocess.Popen(cmd, env=env))
    t_end = None if timeout is None else time.monotonic() + timeout
    rc = 0
    pending = list(procs)
    while pending:
        for p in list(pending):
            code = p.poll()
            if code is None:
                continue
            pending.remove(p)
            if code != 0 and rc == 0:
                rc = code
                for q in pending:
                    q.terminate()
        if t_end is not None and time.monotonic() > t_end:
            for q in pending:
                q.kill()
            return rc or 124
        time.sleep(0.05)
    return rc


# ---------------------------------------------------------------- CPU reference legs
def reference_available() -> bool:
    return (REF_DIR / "framrir" / "__init__.py").exists()


def _job_args(w, j):
    J = w.jobs[j]
    mics = w.mics[J["mic_off"]: J["mic_off"] + J["n_mics"]].copy()
    return dict(room=tuple(float(x) for x in J["room"]), mics=mics, center=np.array(J["center"]),
                source=(float(J["d0"]), float(J["az"]), float(J["el"])), t60=float(J["t60"]),
                sample_rate=w.sample_rate, num_images=int(J["n_images"]), seed=int(J["seed"]),
                source_index=int(J["source_index"]))


def _render_reference(kw):
    """One (room, source) through the UNMODIFIED reference (baseline/_ref):
    simulate_rir's per-source body (core.py:293-315) with this job's image
    count, i.e. the stage functions simulate_rir itself calls.  The Scene is
    built with the reference's constructor; config 5's ad-hoc arrays fail its
    aperture rule (params.py:94-99), so those scenes are assembled without
    __post_init__, which leaves the arithmetic unchanged."""
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import framrir
    from framrir import core

    params = framrir.SimParams(t60=kw["t60"], sample_rate=kw["sample_rate"], num_images=kw["num_images"],
                               seed=kw["seed"])
    srcs = [kw["source"]] * (kw["source_index"] + 1)
    try:
        scene = framrir.Scene(room_dims=kw["room"], mic_positions=kw["mics"], sources=srcs)
    except ValueError:
        scene = object.__new__(framrir.Scene)
        scene.room_dims, scene.mic_positions, scene.sources, scene.reference_point = (
            kw["room"], kw["mics"], srcs, None)
    k = kw["source_index"]
    if k == 0:
        res = framrir.simulate_rir(params, scene, include_early=True)[0]
        return res.full.samples.shape
    factors = framrir.rate_factors(params.sample_rate)
    r = core.reflection_coefficient(scene.room_dims, params.t60)
    images = core.sample_image_geometry(params, scene, k)
    if params.num_images > 0:
        rr = core.max_reflections(params.t60, images.direct_distance, r, params.sound_speed)
        images = core.sample_reflection_counts(images, params, rr)
    train = core.build_impulse_train(images, params, r)
    full = framrir.downsample_highpass_downsample(train, factors, kind="full", metadata={})
    framrir.downsample_highpass_downsample(core.early_reverb_train(train, params), factors, kind="early",
                                           metadata={})
    return full.samples.shape


def _render_port(kw):
    from oracle import framrir_port as P

    full, early, _ = P.render(P.Job(**kw), include_early=True)
    return full.shape


def cpu_jobs(cfg: int, n_jobs: int):
    from paper_2304_08052_b200 import workloads

    per_room = SOURCES_PER_ROOM[cfg]
    w = workloads.build(cfg, max(1, -(-n_jobs // per_room)) if cfg != 1 else None)
    return [_job_args(w, j) for j in range(min(n_jobs, len(w.jobs)))]


def cpu_rate(cfg: int, n_jobs: int, workers: int, repeats: int = 1, warmup: int = 1):
    """RIR/s of the reference's CPU implementation over the first ``n_jobs``
    jobs (global room order) of the config with ``workers`` single-threaded
    processes, pool warm-up excluded.  Returns (rate, jobs, walls, kind)."""
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    kind = "reference" if reference_available() else "port"
    fn = _render_reference if kind == "reference" else _render_port
    jobs = cpu_jobs(cfg, n_jobs)
    walls = []
    with ProcessPoolExecutor(max_workers=workers) as ex:
        for _ in range(max(1, warmup)):  # every worker imports numpy/scipy and runs one job first
            list(ex.map(fn, [jobs[i % len(jobs)] for i in range(workers)]))
        for _ in range(repeats):
            t0 = time.perf_counter()
            list(ex.map(fn, jobs))
            walls.append(time.perf_counter() - t0)
    return len(jobs) * len(walls) / sum(walls), len(jobs), walls, kind


def cpu_sample_jobs(cfg: int, cores: int, steps: int) -> int:
    """Jobs per CPU step: 12 per worker (fewer for long runs, so the whole
    --steps K run stays within a few minutes); configs 1 and 4 are scaled to
    their per-job cost."""
    per_worker = 12 if steps <= 20 else max(3, 240 // steps)
    if cfg == 1:
        return 1
    if cfg == 4:
        per_worker = max(1, per_worker // 6)
    return cores * per_worker


def cpu_sample_text(cfg, nj, kind, cores, walls):
    what = ("framrir.simulate_rir from baseline/_ref (the unmodified reference: numpy + scipy)"
            if kind == "reference" else
            "oracle/framrir_port.py (the reference algorithm on numpy + scipy; baseline/_ref absent)")
    return (f"first {nj} jobs (global room order) of config {cfg} per step, full+early, {what}, "
            f"{cores} single-threaded worker processes, step walls {', '.join('%.2f' % x for x in walls[:4])} s")


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi samples (SM clock + throttle reasons) while running."""

    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.rows = []
        self.proc = None
        self.dev = device_index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        loaded = [r for r in self.rows if (num(r[2]) or 0) >= 50] or self.rows
        sm = [num(r[0]) for r in loaded if num(r[0]) is not None]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in loaded:
            for name, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": num(loaded[0][1]), "reasons": sorted(reasons),
                "samples": len(self.rows), "samples_under_load": len(loaded)}


# ---------------------------------------------------------------- peaks / profiles
def measured_peaks():
    """(HBM GB/s, its kind, measured FP32 FFMA TFLOP/s or None)."""
    p = ROOT / "MEASURED_PEAKS.json"
    peaks = json.loads(p.read_text()) if p.exists() else {}
    fma = ROOT / "profiles" / "fma_peak.json"
    fp32 = None
    if fma.exists():
        for line in fma.read_text().splitlines():
            try:
                d = json.loads(line)
            except json.JSONDecodeError:
                continue
            if d.get("kind") == "fp32_ffma":
                fp32 = max(fp32 or 0.0, d["tflops"])
    if "hbm_gbs" in peaks:
        return peaks["hbm_gbs"], "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)", fp32
    return 6650.0, "fallback (B200_PROFILING.md)", fp32


def render_profile(cfg: int, rooms_per_launch: int):
    """The committed ncu capture of one render launch of this config and launch
    size (profiles/render_ncu.json, written by tools/render_profile_json.py
    from an `ncu --set full` run of the same launch), or None."""
    p = ROOT / "profiles" / "render_ncu.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text()).get(f"cfg{cfg}")
    if not d or d.get("rooms_per_launch") != rooms_per_launch:
        return None
    return d


def reference_chain_flops(jobs, fs: int, variants: int) -> float:
    """SURVEY §8(d) algorithmic FLOPs of the reference chain per batch:
    W = 2*T1*(I+1) + 9*n1 + 2*len2*n2 per (channel, variant)."""
    from paper_2304_08052_b200 import _abi

    d = _abi.design_describe(fs)
    t1 = d.len1 / d.down
    per = (2 * t1 * (jobs["n_images"] + 1) + 9 * jobs["n1"] + 2 * d.len2 * jobs["n2"]) * jobs["n_mics"]
    return float(per.sum() * variants)


def config_block(cfg: int, world: int, early: bool, rooms: int | None, chunk: int) -> dict:
    """The `config` object, identical in both arms for the same command line."""
    if cfg == 5:
        total = rooms or 65536
        rirs = total
        par = f"{total} rooms split over {world} GPU(s) (strong), {chunk}-room launches, no collective"
    elif cfg == 1:
        rirs = world
        par = f"one room per GPU on {world} GPU(s), no collective"
    else:
        per = rooms or CONFIGS[cfg]["rooms"]
        rirs = per * SOURCES_PER_ROOM[cfg] * world
        par = f"{per} rooms per GPU on {world} GPU(s) (weak), no collective"
    return {"workload": CONFIGS[cfg]["desc"], "config_id": cfg, "rirs_per_step": rirs,
            "variants": "full+early" if early else "full", "parallelism": par,
            "l2": "inputs larger than L2: every step writes >= 0.3 GB of RIRs plus item lists "
                  "(126 MB L2), no flush needed; the serial render timing flushes 252 MB between steps"}


# ---------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2304_08052_b200 import _abi, engine, workloads
    from paper_2304_08052_b200.shard import shard_ranges

    rank, world, local = dist_env()
    local = local % max(1, torch.cuda.device_count())  # --dist-backend gloo may share one GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:  # CPU collectives: lets N ranks share a GPU for testing the multi-rank path
            dist.init_process_group("gloo")
    cfg = args.config
    early = not args.no_early
    variants = 2 if early else 1
    chunk = args.chunk or 4096

    # ---- workload shard (global room indices -> identical content for any N)
    shards, scaling = shard_ranges(cfg, rank, world, args.rooms, chunk)
    batches = []
    for start, n in shards:
        w = workloads.config1() if cfg == 1 else workloads.build(cfg, n, start=start)
        pb = engine.prepare(w.sample_rate, w.jobs, w.mics)
        batches.append((w, pb, engine.DeviceBatch(pb, device=dev, workspace=False)))
    # one reusable output buffer set per distinct size (cfg 5 chunks share one)
    max_out = max(int(db.batch.total_out) for _, _, db in batches)
    max_ch = max(int(db.batch.total_channels) for _, _, db in batches)
    full = torch.empty(max_out, dtype=torch.float32, device=dev)
    earlyb = torch.empty(max_out, dtype=torch.float32, device=dev) if early else None
    direct = torch.empty(max_ch, dtype=torch.int32, device=dev)
    n_rirs_rank = sum(len(pb.jobs) for _, pb, _ in batches)
    # two workspaces (the pipelined loop below alternates them); chunks share them
    max_ws = max(db.workspace_bytes for _, _, db in batches)
    wss = [torch.empty(max_ws, dtype=torch.uint8, device=dev) for _ in range(2)]
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(events=None):
        for i, (_, _, db) in enumerate(batches):
            if events is not None:
                events[i][0].record(stream)
            db.launch(full, earlyb, direct, stream, stages=_abi.STAGE_GEOM | _abi.STAGE_DELAY, workspace=wss[0])
            if events is not None:
                events[i][1].record(stream)
            db.launch(full, earlyb, direct, stream, stages=_abi.STAGE_RENDER, workspace=wss[0])
            if events is not None:
                events[i][2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # ---- serial pass (one stream, L2 flushed between steps outside the
    # events): per-launch render time for the roofline
    K = args.steps
    ev = [[[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in batches] for _ in range(K)]
    sampler = ClockSampler(local)
    with sampler:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        for k in range(K):
            flush.fill_(float(k))  # evict L2 between timed steps (outside the events)
            step(ev[k])
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    step_ms = [sum(e[0].elapsed_time(e[2]) for e in ev[k]) for k in range(K)]
    render_ms = [sum(e[1].elapsed_time(e[2]) for e in ev[k]) for k in range(K)]
    prerender_ms = [sum(e[0].elapsed_time(e[1]) for e in ev[k]) for k in range(K)]
    serial_ms = float(sum(step_ms))
    tot_render = float(sum(render_ms))
    tot_pre = float(sum(prerender_ms))

    # ---- throughput (value): launches are independent batches, run as a
    # 2-deep pipeline: launch k + 1's latency-bound geom/sort/tail kernels on a
    # second stream (own workspace and outputs) while launch k renders.  Small
    # launches do not fill the GPU on their own (config 2: 1.30 -> 1.46 M
    # RIR/s); for large ones the full render pass leaves room on each SM for a
    # geom or tail CTA (config 5: 252.8 vs 251.0 K RIR/s on one stream,
    # config 3 +0.3%; with round 2's first combined render, whose three CTAs
    # filled the SMs' shared memory, one stream was faster).  The per-launch
    # working set (item lists + RIRs) exceeds L2.
    depth = args.value_streams or 2
    outs = [(full, earlyb, direct)]
    if depth == 2:
        outs.append((torch.empty_like(full), torch.empty_like(earlyb) if early else None, torch.empty_like(direct)))
    streams = [torch.cuda.Stream(dev) for _ in range(depth)]

    def pipelined(nsteps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for st_ in streams:
            st_.wait_event(e0)
        slot = 0
        for _ in range(nsteps):
            for _, _, db in batches:
                db.launch(*outs[slot], stream=streams[slot], workspace=wss[slot])
                slot = (slot + 1) % depth
        for st_ in streams:
            ev_ = torch.cuda.Event()
            ev_.record(st_)
            stream.wait_event(ev_)
        e1.record(stream)
        return e0, e1

    pipelined(max(1, args.warmup))
    torch.cuda.synchronize(dev)
    with sampler:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        pe0, pe1 = pipelined(K)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        # keep the clock sampler fed with the same work for >= 0.5 s
        t_end = time.perf_counter() + 0.5
        while time.perf_counter() < t_end:
            pipelined(1)
            torch.cuda.synchronize(dev)
    tot_ms = pe0.elapsed_time(pe1)
    del wss, outs
    torch.cuda.empty_cache()

    # ---- end to end through the public host-output API, every shard of this rank
    e2e = run_e2e(args, batches, early, dev)
    cdev = dev if args.dist_backend == "nccl" else torch.device("cpu")
    t = torch.tensor([tot_ms, tot_render, serial_ms, tot_pre, e2e["ms_per_step"]], dtype=torch.float64,
                     device=cdev)
    n = torch.tensor([float(n_rirs_rank)], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(n, op=dist.ReduceOp.SUM)
    max_ms, max_render, max_serial, max_pre, e2e_ms = (float(x) for x in t)
    total_rirs = float(n[0])
    value = total_rirs * K / (max_ms / 1e3)
    e2e_value = total_rirs / (e2e_ms / 1e3)

    dropin = run_dropin(dev) if rank == 0 else None
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return None

    # ---- roofline of the dominant kernel (render), per launch
    hbm_peak, peak_kind, fp32_meas = measured_peaks()
    launches = len(batches)
    out_bytes = sum(int((pb.jobs["n_mics"].astype(np.int64) * pb.jobs["n2"]).sum()) * 4 * variants
                    for _, pb, _ in batches)
    item_bytes = sum(int(db.batch.total_items) * 8 for _, _, db in batches)
    render_s_launch = max_render / K / launches / 1e3
    hbm_achieved = out_bytes / launches / render_s_launch / 1e9
    prof = render_profile(cfg, int(batches[0][0].rooms))
    chain_flops = sum(reference_chain_flops(pb.jobs, batches[0][0].sample_rate, variants) for _, pb, _ in batches)
    fp32_eff = chain_flops / (max_render / K / 1e3) / 1e12
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores = len(os.sched_getaffinity(0))
        n_cpu = args.cpu_jobs or cpu_sample_jobs(cfg, cores, 1)
        rate, nj, walls, kind = cpu_rate(cfg, n_cpu, cores)
        cpu = {"value": rate, "unit": "RIR/s", "cores": cores, "kind": kind,
               "sample": cpu_sample_text(cfg, nj, kind, cores, walls)}
    launches_per_step = sum(db.launch_count(early) for _, _, db in batches)
    line = {
        "metric": METRIC, "value": value, "unit": "RIR/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": max_ms / K, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f32 (FP64 geometry, delays and LP state)",
        "data": "synthetic: seeded BASELINE rooms (no dataset needed), native device Philox draws",
        "config": config_block(cfg, world, early, args.rooms, chunk),
        "roofline": {"bound": "hbm", "achieved": hbm_achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": hbm_achieved / hbm_peak,
                     "traffic": prof["dram_bytes"] if prof else None,
                     "kernel": "render_kernel", "bytes_per_launch": out_bytes / launches,
                     "bytes": "SURVEY 8(d) W_bytes = 4*M*n2*variants per RIR (FP32 RIRs written)",
                     "overhead_bytes_per_launch": item_bytes / launches,
                     "overhead": "8 B per (image, mic) sorted item read by the render (not algorithmic)",
                     "launch_ms": render_s_launch * 1e3, "launches_per_step": launches,
                     "peak_kind": peak_kind,
                     "traffic_source": prof["source"] if prof else "no committed ncu capture for this launch size"},
        "fp32": {"note": "NON-PHYSICAL effective figure: SURVEY 8(d) reference-chain FLOPs / render time; "
                         "the composite-table formulation executes ~10x fewer FLOPs",
                 "effective_tflops": fp32_eff,
                 "peak_tflops_theoretical": FP32_THEORETICAL_TFLOPS,
                 "peak_tflops_measured_ffma": fp32_meas,
                 "effective_frac_of_theoretical": fp32_eff / FP32_THEORETICAL_TFLOPS,
                 "executed_fp32_pipe_pct": prof.get("fp32_pipe_pct") if prof else None,
                 "issue_active_pct": prof.get("issue_active_pct") if prof else None,
                 "inst_per_launch": prof.get("inst_executed") if prof else None},
        "stages": {"serial_ms_per_step": max_serial / K, "serial_value": total_rirs * K / (max_serial / 1e3),
                   "render_ms_per_step": max_render / K, "pre_render_ms_per_step": max_pre / K,
                   "value_streams": depth,
                   "note": "serial pass: one stream, geom+sort+tail then render per launch, 252 MB L2 flush "
                           "between steps; value runs the same launches back to back on value_streams streams "
                           "(2: a pipeline for launches that do not fill the GPU)"},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "RIR/s", "h2d_bytes_per_step": e2e["h2d"] * world,
                "d2h_bytes_per_step": e2e["d2h"] * world, "ms_per_step": e2e_ms,
                "link": {"achieved_gbs_per_gpu": (e2e["h2d"] + e2e["d2h"]) / (e2e_ms / 1e3) / 1e9,
                         "d2h_peak_gbs": e2e["d2h_peak_gbs"],
                         "note": "rank 0's host<->device bytes per step / e2e step time vs a pinned D2H copy"},
                "path": e2e["path"]},
        "e2e_dropin": dropin,
        "gpu_launches": launches_per_step * K,
        "clocks": sampler.summary(),
    }
    return line


def run_e2e(args, batches, early, dev):
    """Same metric through the public host-output API (engine.HostStream): host
    validation of every part, H2D of the job tables from pinned memory, render,
    D2H of every RIR (full + early) and direct index into pinned host slots,
    over ALL of this rank's rooms; the copy of part k overlaps the render of
    part k + 1."""
    import torch

    from paper_2304_08052_b200 import engine

    w0 = batches[0][0]
    offs, mics = [], []
    base = 0
    for w, _, _ in batches:  # re-base each shard's mic rows into one table
        j = np.array(w.jobs, copy=True)
        j["mic_off"] += base
        offs.append(j)
        mics.append(w.mics)
        base += len(w.mics)
    jobs = np.concatenate(offs)
    mics = np.concatenate(mics)
    part = args.e2e_part or (1024 if args.config == 5 else max(1, -(-len(jobs) // 4)))
    hs = engine.HostStream(w0.sample_rate, jobs, mics, part_jobs=part, include_early=early, slots=2, device=dev)
    steps = 2 if args.config == 5 else max(2, min(args.steps, 10))
    hs.run()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(steps):
        hs.run()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    out = {"ms_per_step": ms, "h2d": int(hs.h2d_bytes), "d2h": int(hs.d2h_bytes),
           "d2h_peak_gbs": d2h_peak_gbs(min(int(hs.d2h_bytes), 1 << 30), dev),
           "path": f"engine.HostStream over all {len(jobs)} jobs of the rank in {len(hs.parts)} parts of "
                   f"{part}: frir_jobs_prepare + H2D(job tables, pinned) + frir_simulate + D2H(every RIR) "
                   f"to 2 pinned host slots, copy overlapped with render; host wall clock, {steps} passes"}
    del hs
    torch.cuda.empty_cache()
    return out


def run_dropin(dev, calls: int = 50):
    """Per-call latency of the drop-in ``simulate_rir(params, scene)`` on
    config 1 (the per-item use of reference mixture.py:342 / bench.py:67-69):
    host validation, one launch sequence, float64 RirResult copies."""
    import paper_2304_08052_b200 as F

    params = F.SimParams(t60=0.5, num_images=2048, seed=0)
    scene = F.Scene(room_dims=(6.0, 5.0, 3.0), mic_positions=F.linear_array([0.05, 0.05, 0.05]),
                    sources=[(1.4456832294801, 2.356194490192345, 0.20903329903452)])
    for _ in range(5):
        F.simulate_rir(params, scene)
    ts = []
    for i in range(calls):
        p = dataclasses.replace(params, seed=i)
        t0 = time.perf_counter()
        F.simulate_rir(p, scene)
        ts.append((time.perf_counter() - t0) * 1e3)
    med = statistics.median(ts)
    return {"ms_per_call_median": med, "ms_per_call_mean": statistics.fmean(ts), "calls": calls,
            "rirs_per_s": 1e3 / med,
            "path": "paper_2304_08052_b200.simulate_rir(SimParams, Scene, include_early=True) -> "
                    "list[RirResult] (float64 numpy, full + early), config 1, fresh seed per call"}


def d2h_peak_gbs(nbytes, dev):
    """Device -> pinned host copy bandwidth for one block of `nbytes` (best of
    3, CUDA events): the PCIe ceiling of the end-to-end path."""
    import torch

    n = max(nbytes, 1 << 20)
    src = torch.empty(n, dtype=torch.uint8, device=dev)
    dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    best = None
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return n / (best / 1e3) / 1e9


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    cfg = args.config
    cores = len(os.sched_getaffinity(0))
    n_jobs = args.cpu_jobs or cpu_sample_jobs(cfg, cores, args.steps)
    value, nj, walls, kind = cpu_rate(cfg, n_jobs, cores, repeats=args.steps, warmup=1)
    early = not args.no_early
    cpu = {"value": value, "unit": "RIR/s", "cores": cores, "kind": kind,
           "sample": cpu_sample_text(cfg, nj, kind, cores, walls)}
    return {
        "metric": METRIC, "value": value, "unit": "RIR/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(walls) / len(walls), "higher_is_better": True,
        "scaling": "strong" if cfg == 5 else "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": "synthetic: seeded BASELINE rooms (no dataset needed), the reference's own Philox draws",
        "config": config_block(cfg, world, early, args.rooms, args.chunk or 4096),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "RIR/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--rooms", type=int, default=None, help="rooms per GPU (cfg 5: total)")
    ap.add_argument("--chunk", type=int, default=None, help="cfg 5 rooms per launch (default 4096)")
    ap.add_argument("--value-streams", type=int, default=None, choices=[1, 2],
                    help="streams of the throughput loop (default 2: a 2-deep pipeline of launches)")
    ap.add_argument("--e2e-part", type=int, default=None, help="jobs per part of the e2e stream")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-early", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-jobs", type=int, default=None)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo lets several ranks share one GPU (testing the multi-rank path)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args.gpus, [sys.executable, str(Path(__file__).resolve()), *sys.argv[1:]]))
    _, world, _ = dist_env()
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
