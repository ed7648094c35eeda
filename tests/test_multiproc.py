"""N>1 path on CPU: world-size-2 gloo processes shard rooms exactly like
bench.py and reduce timings with MAX (no GPU needed)."""

import hashlib
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_08052_b200 import engine, workloads
from paper_2304_08052_b200.shard import shard_ranges


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _digest(w):
    return hashlib.sha256(w.jobs.tobytes() + w.mics.tobytes()).hexdigest()


def _worker(rank, world, port, cfg, rooms, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ranges, scaling = shard_ranges(cfg, rank, world, rooms, chunk=3)
    digests = []
    n = 0
    for start, count in ranges:
        w = workloads.build(cfg, count, start=start)
        engine.prepare(w.sample_rate, w.jobs, w.mics)  # host validation of the shard
        digests.append((start, _digest(w)))
        n += len(w.jobs)
    fake_ms = torch.tensor([10.0 + rank], dtype=torch.float64)
    dist.all_reduce(fake_ms, op=dist.ReduceOp.MAX)
    total = torch.tensor([float(n)], dtype=torch.float64)
    dist.all_reduce(total, op=dist.ReduceOp.SUM)
    gathered = [None] * world
    dist.all_gather_object(gathered, digests)
    if rank == 0:
        out_q.put((float(fake_ms[0]), float(total[0]), gathered, scaling))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,rooms", [(5, 8), (2, 3)])
def test_two_rank_sharding(cfg, rooms):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, rooms, q)) for r in range(2)]
    for p in procs:
        p.start()
    ms, total, gathered, scaling = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ms == 11.0  # max over ranks
    if cfg == 5:
        assert scaling == "strong" and total == rooms
        # the union of the shards is exactly the single-process workload, chunk by chunk
        flat = sorted(x for per_rank in gathered for x in per_rank)
        for start, dig in flat:
            count = min(3, (4 if start < 4 else 8) - start)
            assert dig == _digest(workloads.build(5, count, start=start))
        assert [s for s, _ in flat] == [0, 3, 4, 7]
    else:
        assert scaling == "weak" and total == 2 * rooms
        starts = sorted(s for per_rank in gathered for s, _ in per_rank)
        assert starts == [0, rooms]


def test_shard_ranges_cover_everything():
    for world in (1, 2, 3, 8):
        got = []
        for r in range(world):
            ranges, _ = shard_ranges(5, r, world, 65536, chunk=4096)
            for s, n in ranges:
                got.extend(range(s, s + n))
        assert got == list(range(65536))
    with pytest.raises(ValueError):
        shard_ranges(2, 2, 2)


def test_room_content_independent_of_sharding():
    whole = workloads.config2(6)
    a, b = workloads.config2(2), workloads.config2(4, start=2)
    assert np.array_equal(np.concatenate([a.jobs, b.jobs])["seed"], whole.jobs["seed"])
    assert np.array_equal(np.concatenate([a.jobs, b.jobs])["d0"], whole.jobs["d0"])


# ---------------------------------------------------------------- bench.py's own launcher
_RANK_PROBE = r'''
import json, os, sys
import torch, torch.distributed as dist
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
assert r == int(os.environ["RANK"]) == int(os.environ["LOCAL_RANK"]) and w == int(os.environ["WORLD_SIZE"])
assert os.environ["MASTER_ADDR"] == "127.0.0.1"
t = torch.tensor([10.0 + r], dtype=torch.float64)
dist.all_reduce(t, op=dist.ReduceOp.MAX)
n = torch.tensor([float(r + 1)], dtype=torch.float64)
dist.all_reduce(n, op=dist.ReduceOp.SUM)
if r == 0:
    print(json.dumps({"world": w, "max_ms": float(t[0]), "sum": float(n[0])}), flush=True)
dist.destroy_process_group()
'''


def test_launch_ranks_env_contract(tmp_path):
    """bench.launch_ranks starts N processes with torchrun's env contract
    (RANK/LOCAL_RANK/WORLD_SIZE, MASTER_ADDR=127.0.0.1, a free port); the
    ranks rendezvous and reduce with MAX/SUM; only rank 0 prints."""
    import subprocess
    import sys

    import bench

    probe = tmp_path / "probe.py"
    probe.write_text(_RANK_PROBE)
    out = tmp_path / "out.txt"
    with open(out, "w") as f:
        code = subprocess.run([sys.executable, "-c",
                               "import sys, bench; sys.exit(bench.launch_ranks(3, [sys.executable, %r]))" % str(probe)],
                              cwd=str(bench.ROOT), stdout=f, timeout=120).returncode
    assert code == 0
    lines = [json.loads(x) for x in out.read_text().splitlines() if x.startswith("{")]
    assert lines == [{"world": 3, "max_ms": 12.0, "sum": 6.0}]


def test_launch_ranks_propagates_failure(tmp_path):
    import sys

    import bench

    bad = tmp_path / "bad.py"
    bad.write_text("import os, sys, time\nif os.environ['RANK'] == '1': sys.exit(3)\ntime.sleep(60)\n")
    assert bench.launch_ranks(2, [sys.executable, str(bad)], timeout=90) == 3


def test_bench_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` without torchrun spawns the ranks itself; the
    reference arm runs on rank 0 only and reports n_gpus = 2."""
    import subprocess
    import sys

    import bench

    res = subprocess.run([sys.executable, str(bench.ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--config", "1", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [json.loads(x) for x in res.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
    assert lines[0]["config"]["rirs_per_step"] == 2 and lines[0]["value"] > 0


@pytest.mark.gpu
def test_bench_two_ranks_one_gpu_totals():
    """The GPU arm through the launcher: 2 ranks (gloo, sharing one GPU) split
    config 5's rooms; the line counts every rank's RIRs and says n_gpus 2."""
    import subprocess
    import sys

    import bench

    res = subprocess.run([sys.executable, str(bench.ROOT / "bench.py"), "--gpus", "2", "--dist-backend", "gloo",
                          "--rooms", "2048", "--chunk", "512", "--steps", "3", "--warmup", "3", "--e2e-part", "512"],
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [json.loads(x) for x in res.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["rirs_per_step"] == 2048
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["roofline"]["launches_per_step"] == 2
