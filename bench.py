"""Benchmark: multi-channel FRAM-RIRs per second on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One step = render one batch of the configured BASELINE workload (default
configs[1] = config 2: 1024 seeded random rooms per GPU, 6-mic array, 16 kHz,
I ~ U{1024..4096}), full + early variants, native (device Philox) draws.
Multi-GPU: one process per GPU (torchrun), rooms sharded by global room index,
no collective on the data path ("weak" scaling for configs 2-4, "strong" for
config 5's fixed 65536 rooms); timing is the max over ranks of CUDA-event
durations.  ``--impl reference`` times the CPU oracle port of the reference
path (oracle/framrir_port.py, numpy + scipy exactly as the reference) on the
host cores instead.
"""

from __future__ import annotations

import argparse
import json
import os
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

METRIC = "multi-channel RIRs/sec at 1/2/4/8 B200; % of FP32 and HBM roofline"
L2_BYTES = 126 * 2**20

CONFIGS = {
    1: dict(rooms=1, desc="cfg1: 1 room 6x5x3 m, T60 0.5 s, 4-mic linear 5 cm, I=2048, 16 kHz"),
    2: dict(rooms=1024, desc="cfg2: 1024 random rooms/GPU, T60~U[0.1,0.7], 6-mic 5 cm circle, I~U{1024..4096}, 16 kHz"),
    3: dict(rooms=4096, desc="cfg3: 4096 rooms x 3 sources/GPU, T60~U[0.2,1.0], 8-mic 10 cm circle, I~U{1024..4096}, 16 kHz"),
    4: dict(rooms=512, desc="cfg4: 512 rooms x 2 sources/GPU, 48 kHz, T60~U[1.0,1.5], 16-mic 4x4 grid, I~U{8192..16384}"),
    5: dict(rooms=65536, desc="cfg5: 65536 rooms sharded over GPUs, 32 ad-hoc mics, T60~U[0.1,0.7], I~U{1024..8192}, 16 kHz"),
}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- CPU oracle legs
def _oracle_job_args(w, j):
    J = w.jobs[j]
    mics = w.mics[J["mic_off"]: J["mic_off"] + J["n_mics"]].copy()
    return dict(room=tuple(float(x) for x in J["room"]), mics=mics, center=np.array(J["center"]),
                source=(float(J["d0"]), float(J["az"]), float(J["el"])), t60=float(J["t60"]),
                sample_rate=w.sample_rate, num_images=int(J["n_images"]), seed=int(J["seed"]),
                source_index=int(J["source_index"]))


def _oracle_render(kw):
    from oracle import framrir_port as P

    full, early, _ = P.render(P.Job(**kw), include_early=True)
    return full.shape


def oracle_jobs(cfg: int, n_jobs: int):
    from paper_2304_08052_b200 import workloads

    per_room = {1: 1, 2: 1, 3: 3, 4: 2, 5: 1}[cfg]
    w = workloads.build(cfg, max(1, -(-n_jobs // per_room)) if cfg != 1 else None)
    return [_oracle_job_args(w, j) for j in range(min(n_jobs, len(w.jobs)))]


def cpu_oracle_rate(cfg: int, n_jobs: int, workers: int, repeats: int = 1, warmup: int = 1):
    """RIR/s of the oracle port over the first n_jobs jobs of the config with
    `workers` single-threaded processes (pool warm-up excluded).  Returns
    (rate, jobs, per-repeat walls)."""
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    jobs = oracle_jobs(cfg, n_jobs)
    walls = []
    with ProcessPoolExecutor(max_workers=workers) as ex:
        for _ in range(max(1, warmup)):
            list(ex.map(_oracle_render, jobs[:workers]))
        for _ in range(repeats):
            t0 = time.perf_counter()
            list(ex.map(_oracle_render, jobs))
            walls.append(time.perf_counter() - t0)
    return len(jobs) * len(walls) / sum(walls), len(jobs), walls


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
    return peaks.get("hbm_gbs", 6650.0), ("measured" if "hbm_gbs" in peaks else "fallback"), fp32


def profiled_traffic(cfg: int):
    p = ROOT / "profiles" / "render_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return d.get(f"cfg{cfg}")


def reference_chain_flops(jobs, fs: int, variants: int) -> float:
    """SURVEY §8(d) algorithmic FLOPs of the reference chain per batch:
    W = 2*T1*(I+1) + 9*n1 + 2*len2*n2 per (channel, variant)."""
    from paper_2304_08052_b200 import _abi

    d = _abi.design_describe(fs)
    t1 = d.len1 / d.down
    per = (2 * t1 * (jobs["n_images"] + 1) + 9 * jobs["n1"] + 2 * d.len2 * jobs["n2"]) * jobs["n_mics"]
    return float(per.sum() * variants)


# ---------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2304_08052_b200 import _abi, engine, workloads

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

    # ---- workload shard (global room indices -> identical content for any N)
    from paper_2304_08052_b200.shard import shard_ranges

    shards, scaling = shard_ranges(cfg, rank, world, args.rooms, args.chunk or 4096)
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
        # keep the clocks sampler fed with the same work for >= 0.6 s
        t_end = time.perf_counter() + 0.6
        while time.perf_counter() < t_end:
            step()
            torch.cuda.synchronize(dev)
    step_ms = [ev[k][0][0].elapsed_time(ev[k][-1][2]) for k in range(K)]
    render_ms = [sum(e[1].elapsed_time(e[2]) for e in ev[k]) for k in range(K)]
    serial_ms = float(sum(step_ms))
    tot_render = float(sum(render_ms))

    # ---- throughput: the K steps as a 2-deep pipeline.  Steps are independent
    # batches, so step k + 1's latency-bound geom/sort/tail kernels run on a
    # second stream (own workspace and outputs) while step k renders.  The
    # per-step working set (item lists + RIRs) is larger than L2, so no flush.
    outs = [(full, earlyb, direct),
            (torch.empty_like(full), torch.empty_like(earlyb) if early else None, torch.empty_like(direct))]
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]

    def pipelined(nsteps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for st_ in streams:
            st_.wait_event(e0)
        slot = 0
        for _ in range(nsteps):
            for i, (_, _, db) in enumerate(batches):
                db.launch(*outs[slot], stream=streams[slot], workspace=wss[slot])
                slot ^= 1
        for st_ in streams:
            ev_ = torch.cuda.Event()
            ev_.record(st_)
            stream.wait_event(ev_)
        e1.record(stream)
        return e0, e1

    for _ in range(2):
        pipelined(max(2, args.warmup))
    torch.cuda.synchronize(dev)
    with sampler:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        pe0, pe1 = pipelined(K)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    tot_ms = pe0.elapsed_time(pe1)
    cdev = dev if args.dist_backend == "nccl" else torch.device("cpu")
    t = torch.tensor([tot_ms, tot_render, serial_ms], dtype=torch.float64, device=cdev)
    n = torch.tensor([float(n_rirs_rank)], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(n, op=dist.ReduceOp.SUM)
    max_ms, max_render, max_serial = float(t[0]), float(t[1]), float(t[2])
    total_rirs = float(n[0])
    value = total_rirs * K / (max_ms / 1e3)

    # ---- end to end through the C-ABI with host buffers (rank-local, first shard)
    e2e = run_e2e(args, batches[0], early, dev, stream)
    if world > 1:
        te = torch.tensor([e2e["ms_per_step"]], dtype=torch.float64, device=cdev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te[0])
    else:
        e2e_ms = e2e["ms_per_step"]
    rirs_shard0 = len(batches[0][1].jobs)
    e2e_value = rirs_shard0 * world / (e2e_ms / 1e3) if cfg != 5 else rirs_shard0 * world / (e2e_ms / 1e3)

    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return None

    # ---- roofline of the dominant kernel (render), per launch
    hbm_peak, peak_kind, fp32_peak = measured_peaks()
    jobs_all = [pb.jobs for _, pb, _ in batches]
    out_bytes = sum(int(db.batch.total_out) * 4 * variants for _, _, db in batches)
    item_bytes = sum(int(db.batch.total_items) * 8 for _, _, db in batches)
    render_s_per_step = max_render / K / 1e3
    hbm_achieved = (out_bytes + item_bytes) / render_s_per_step / 1e9
    chain_flops = sum(reference_chain_flops(j, batches[0][0].sample_rate, variants) for j in jobs_all)
    fp32_eff = chain_flops / render_s_per_step / 1e12
    traffic = profiled_traffic(cfg)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores = len(os.sched_getaffinity(0))
        n_cpu = args.cpu_jobs or {1: 1, 2: 192, 3: 96, 4: 16, 5: 128}[cfg]
        rate, nj, walls = cpu_oracle_rate(cfg, n_cpu, cores)
        cpu = {"value": rate, "unit": "RIR/s", "cores": cores, "kind": "port",
               "sample": f"first {nj} jobs of config {cfg}, oracle/framrir_port.py (numpy+scipy, the reference's "
                         f"algorithm), full+early, {cores} worker processes, wall {walls[0]:.2f} s"}
    launches_per_step = sum(db.launch_count(early) for _, _, db in batches)
    line = {
        "metric": METRIC, "value": value, "unit": "RIR/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": max_ms / K, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f32 (FP64 geometry, delays and LP state)",
        "data": "synthetic: seeded BASELINE rooms (no dataset needed), native device Philox draws",
        "config": {"workload": CONFIGS[cfg]["desc"], "config_id": cfg,
                   "rirs_per_step": total_rirs, "variants": "full+early" if early else "full",
                   "l2": "value: the K steps run as a 2-deep pipeline over two streams with "
                         "double-buffered workspaces; each step's working set (%.0f MB of item lists + "
                         "%.0f MB of RIRs) exceeds the 126 MB L2, so no flush between steps.  "
                         "serial_ms_per_step / render_ms_per_step: one stream, a 252 MB L2 flush between "
                         "steps (outside the events)" % (2 * item_bytes / 1e6, out_bytes / 1e6),
                   "serial_ms_per_step": max_serial / K,
                   "serial_value": total_rirs * K / (max_serial / 1e3),
                   "parallelism": f"rooms sharded over {world} GPU(s), no collective"},
        "roofline": {"bound": "hbm", "achieved": hbm_achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": hbm_achieved / hbm_peak, "traffic": traffic,
                     "kernel": "render_kernel", "bytes_per_launch": out_bytes + item_bytes,
                     "render_ms_per_step": max_render / K, "peak_kind": peak_kind,
                     "fp32_effective": {"achieved_tflops": fp32_eff, "peak_tflops": fp32_peak,
                                        "frac": (fp32_eff / fp32_peak) if fp32_peak else None,
                                        "note": "reference-chain FLOPs (SURVEY 8d) / render time; "
                                                "the kernel executes ~10x fewer (composite tables)"}},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "RIR/s", "h2d_bytes_per_step": e2e["h2d"],
                "d2h_bytes_per_step": e2e["d2h"], "ms_per_step": e2e_ms,
                "link": {"achieved_gbs": (e2e["h2d"] + e2e["d2h"]) / (e2e_ms / 1e3) / 1e9,
                         "d2h_peak_gbs": e2e["d2h_peak_gbs"],
                         "frac": (e2e["h2d"] + e2e["d2h"]) / (e2e_ms / 1e3) / 1e9 / e2e["d2h_peak_gbs"],
                         "note": "host<->device bytes per step / e2e step time vs a pinned D2H copy of the "
                                 "same size"},
                "path": "engine.HostPipeline: frir_jobs_prepare + H2D(job tables) + frir_simulate + "
                        "D2H(all RIRs) to pinned host, 4 chunks, copy overlapped with render"},
        "gpu_launches": launches_per_step * K,
        "clocks": sampler.summary(),
    }
    issue = issue_roofline(cfg, max_render / K, line["clocks"].get("sm_mhz"), dev)
    if issue:
        line["roofline"]["issue"] = issue
    return line


def issue_roofline(cfg: int, render_ms: float, sm_mhz, dev):
    """The render kernel is instruction-issue bound: its warp
    instructions per launch (ncu, committed under profiles/) against the issue
    slots of the live render time at the sampled SM clock (one warp
    instruction per cycle per SM sub-partition)."""
    import torch

    p = ROOT / "profiles" / "r01" / "v8_cfg2_ncu_full_summary.json"
    if cfg != 2 or not p.exists() or not sm_mhz:
        return None
    d = next((r for r in json.loads(p.read_text()) if "render_kernel" in r["Kernel Name"]), None)
    if d is None:
        return None
    inst = float(d["smsp__inst_executed.sum"])
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    slots = render_ms / 1e3 * sm_mhz * 1e6 * sms * 4
    return {"bound": "issue", "achieved": inst / (render_ms / 1e3) / 1e9, "unit": "G warp-instr/s",
            "peak": sm_mhz * 1e6 * sms * 4 / 1e9, "frac": inst / slots,
            "inst_per_launch": inst, "issue_active_pct_ncu": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
            "source": str(p.relative_to(ROOT)) + " (ncu --set full, one config-2 render launch)"}


def run_e2e(args, batch, early, dev, stream):
    """Same metric through the public host-output API (engine.HostPipeline):
    host validation/layout of the job tables, H2D, render, D2H of every RIR
    into pinned memory, with the copy of chunk k overlapping the render of
    chunk k + 1."""
    from paper_2304_08052_b200 import engine

    w = batch[0]
    steps = max(2, min(args.steps, 10))
    pipe = engine.HostPipeline(w.sample_rate, w.jobs, w.mics, include_early=early, chunks=4, device=dev)
    pipe.run()
    torch_sync(dev)
    t0 = time.perf_counter()
    for _ in range(steps):
        pipe.run()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    return {"ms_per_step": ms, "h2d": int(pipe.h2d_bytes), "d2h": int(pipe.d2h_bytes),
            "d2h_peak_gbs": d2h_peak_gbs(int(pipe.d2h_bytes), dev)}


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


def torch_sync(dev):
    import torch

    torch.cuda.synchronize(dev)


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    cfg = args.config
    cores = len(os.sched_getaffinity(0))
    n_jobs = args.cpu_jobs or {1: 1, 2: 32, 3: 24, 4: 2, 5: 16}[cfg]
    value, nj, walls = cpu_oracle_rate(cfg, n_jobs, cores, repeats=args.steps, warmup=max(1, args.warmup))
    early = not args.no_early
    return {
        "metric": METRIC, "value": value, "unit": "RIR/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(walls) / len(walls), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": "synthetic: seeded BASELINE rooms",
        "config": {"workload": CONFIGS[cfg]["desc"], "config_id": cfg,
                   "variants": "full+early" if early else "full",
                   "parallelism": f"{cores} host worker processes"},
        "cpu_baseline": {"value": value, "unit": "RIR/s", "cores": cores, "kind": "port",
                         "sample": f"first {nj} jobs of config {cfg} per step; oracle/framrir_port.py "
                                   "(the reference algorithm on numpy+scipy; /root/reference is not on the box)"},
        "e2e": {"value": value, "unit": "RIR/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--rooms", type=int, default=None, help="rooms per GPU (cfg 5: total)")
    ap.add_argument("--chunk", type=int, default=None, help="cfg 5 rooms per launch")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-early", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-jobs", type=int, default=None)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo lets several ranks share one GPU (testing the multi-rank path)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
