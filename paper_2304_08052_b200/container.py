"""The "FRIR" filter container (persisted batches).

Byte-compatible with ``framrir.io`` (/root/reference/pkg/src/framrir/io.py:
26-107): file header ``<4sHI`` (magic b"FRIR", version 1, record count), then
per record ``<HIIBQ`` (channels, samples, sample rate, kind 0 full / 1 early,
seed) and the float32 little-endian payload, channel-major.  Besides the
mirrored ``write_rir_container`` / ``read_rir_container``,
``write_batch_container`` persists a whole rendered device batch: each job's
rows are copied device-to-host straight into the file's record layout, one
job at a time through a pinned staging buffer.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

__all__ = ["RirRecord", "write_rir_container", "read_rir_container", "write_batch_container"]

MAGIC = b"FRIR"
CONTAINER_VERSION = 1
KIND_CODES = {"full": 0, "early": 1}
KIND_NAMES = {v: k for k, v in KIND_CODES.items()}
_RECORD_HEADER = struct.Struct("<HIIBQ")  # n_channels, n_samples, f_s, kind, seed
_FILE_HEADER = struct.Struct("<4sHI")     # magic, version, count


@dataclass
class RirRecord:
    """One container entry; float32 payload, channel-major (io.py:58-66)."""

    samples: np.ndarray  # (M, N)
    sample_rate: int
    kind: str = "full"
    seed: int = 0


def write_rir_container(path, records: list) -> None:
    with open(path, "wb") as fh:
        fh.write(_FILE_HEADER.pack(MAGIC, CONTAINER_VERSION, len(records)))
        for rec in records:
            data = np.ascontiguousarray(np.atleast_2d(rec.samples), dtype="<f4")
            m, n = data.shape
            fh.write(_RECORD_HEADER.pack(m, n, int(rec.sample_rate), KIND_CODES[rec.kind], rec.seed))
            fh.write(data.tobytes())


def read_rir_container(path) -> list:
    with open(path, "rb") as fh:
        head = fh.read(_FILE_HEADER.size)
        if len(head) != _FILE_HEADER.size:
            raise ValueError("truncated container header")
        magic, version, count = _FILE_HEADER.unpack(head)
        if magic != MAGIC:
            raise ValueError(f"bad magic {magic!r}")
        if version != CONTAINER_VERSION:
            raise ValueError(f"unsupported container version {version}")
        records = []
        for _ in range(count):
            rh = fh.read(_RECORD_HEADER.size)
            if len(rh) != _RECORD_HEADER.size:
                raise ValueError("truncated record header")
            m, n, fs, kind, seed = _RECORD_HEADER.unpack(rh)
            payload = fh.read(4 * m * n)
            if len(payload) != 4 * m * n:
                raise ValueError("record payload shorter than declared")
            samples = np.frombuffer(payload, dtype="<f4").reshape(m, n)
            records.append(RirRecord(samples=samples, sample_rate=fs, kind=KIND_NAMES[kind], seed=seed))
        return records


def write_batch_container(path, result, kinds=("full",), seeds=None) -> int:
    """Persist every job of an ``engine.BatchResult`` (device tensors) as
    container records, job by job and kind by kind (job-major).  ``seeds``
    defaults to the jobs' SimParams seeds.  Returns the record count."""
    import torch

    pj = result.prepared.jobs
    fs = int(result.prepared.sample_rate)
    kinds = tuple(kinds)
    for k in kinds:
        if k not in KIND_CODES:
            raise ValueError(f"unknown kind {k!r}")
        if k == "early" and result.early is None:
            raise ValueError("the batch was rendered without the early variant")
    seeds = [int(s) for s in (pj["seed"] if seeds is None else seeds)]
    count = len(pj) * len(kinds)
    max_floats = int((pj["n_mics"].astype(np.int64) * pj["n2"]).max()) if len(pj) else 0
    stage = torch.empty(max_floats, dtype=torch.float32, pin_memory=True)
    with open(path, "wb") as fh:
        fh.write(_FILE_HEADER.pack(MAGIC, CONTAINER_VERSION, count))
        for j in range(len(pj)):
            m, n = int(pj[j]["n_mics"]), int(pj[j]["n2"])
            for k in kinds:
                view = result.job_view(j, k)  # (m, n) strided device view
                host = stage[: m * n].view(m, n)
                host.copy_(view)  # device -> pinned host, row-contiguous
                fh.write(_RECORD_HEADER.pack(m, n, fs, KIND_CODES[k], seeds[j]))
                fh.write(host.numpy().astype("<f4", copy=False).tobytes())
    return count
