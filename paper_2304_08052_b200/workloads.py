"""Seeded synthetic room batches for BASELINE.json configs 1-5.

Every room ``i`` of config ``c`` draws from its own
``Generator(Philox(SeedSequence((c, i))))`` in a fixed order, so a room's
content depends only on (config, global room index): sharding rooms across
GPUs never changes them.  Rooms are returned as a job table (one job per
(room, source)) plus mic rows in absolute room coordinates; the array
reference point is the mic centroid, as in the reference's Scene.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import engine
from .scene import linear_array

C0 = 343.0


@dataclass
class Workload:
    name: str
    sample_rate: int
    jobs: np.ndarray       # engine job table (inputs filled)
    mics: np.ndarray       # (rows, 3)
    rooms: int

    @property
    def n_rirs(self) -> int:
        return len(self.jobs)


def _rng(cfg: int, room: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(np.random.SeedSequence((cfg, room))))


def _circle(n, radius, rot):
    ang = rot + 2.0 * np.pi * np.arange(n) / n
    return np.stack([radius * np.cos(ang), radius * np.sin(ang), np.zeros(n)], -1)


def _grid(side, pitch, rot):
    g = (np.arange(side) - (side - 1) / 2.0) * pitch
    x, y = np.meshgrid(g, g, indexing="ij")
    x, y = x.ravel(), y.ravel()
    c, s = np.cos(rot), np.sin(rot)
    return np.stack([c * x - s * y, s * x + c * y, np.zeros_like(x)], -1)


def _spherical(src, center):
    v = np.asarray(src, float) - center
    d = float(np.sqrt((v**2).sum()))
    return d, math.atan2(v[1], v[0]), math.asin(v[2] / d)


def _room(rng, lo_xy, hi_xy, lo_z, hi_z):
    lx, ly = rng.uniform(lo_xy, hi_xy, 2)
    lz = rng.uniform(lo_z, hi_z)
    return np.array([lx, ly, lz])


def _inside(rng, room, margin):
    return rng.uniform(margin, room - margin)


def _emit(jobs_rows, mics_rows, room, t60, mics, center, sources, images, seed):
    off = sum(len(m) for m in mics_rows)
    mics_rows.append(mics)
    for k, (src, n) in enumerate(zip(sources, images)):
        d, az, el = _spherical(src, center)
        jobs_rows.append((room, center, d, az, el, t60, int(seed), k, int(n), off, len(mics)))


def _finish(name, fs, jobs_rows, mics_rows, rooms) -> Workload:
    jobs = engine.new_jobs(len(jobs_rows))
    for j, (room, center, d, az, el, t60, seed, k, n, off, m) in enumerate(jobs_rows):
        jobs[j]["room"] = room
        jobs[j]["center"] = center
        jobs[j]["d0"], jobs[j]["az"], jobs[j]["el"] = d, az, el
        jobs[j]["t60"] = t60
        jobs[j]["seed"] = seed
        jobs[j]["source_index"] = k
        jobs[j]["n_images"] = n
        jobs[j]["mic_off"] = off
        jobs[j]["n_mics"] = m
    return Workload(name, fs, jobs, np.concatenate(mics_rows, 0), rooms)


def config1() -> Workload:
    """Single CPU-runnable room (BASELINE configs[0]): the array is the
    reference's linear_array([0.05]*3) in its own frame, the source given
    relative to the array centre (3.0, 2.5, 1.2) of the room."""
    room = np.array([6.0, 5.0, 3.0])
    mics = linear_array([0.05, 0.05, 0.05])
    center = mics.mean(axis=0)
    d, az, el = _spherical(np.array([2.0, 3.5, 1.5]), np.array([3.0, 2.5, 1.2]))
    jr, mr = [], [mics]
    jr.append((room, center, d, az, el, 0.5, 0, 0, 2048, 0, len(mics)))
    return _finish("cfg1", 16000, jr, mr, 1)


def config2(n_rooms: int = 1024, start: int = 0) -> Workload:
    """Random rooms, 6-mic 5 cm circle, I ~ U{1024..4096} (configs[1])."""
    jr, mr = [], []
    for i in range(start, start + n_rooms):
        g = _rng(2, i)
        room = _room(g, 3.0, 10.0, 2.5, 4.0)
        t60 = g.uniform(0.1, 0.7)
        while True:
            src = _inside(g, room, 0.5)
            ctr = _inside(g, room, 0.5)
            if np.sqrt(((src - ctr) ** 2).sum()) >= 0.3:
                break
        rot = g.uniform(0.0, 2.0 * np.pi)
        n = g.integers(1024, 4097)
        seed = g.integers(2**63)
        mics = ctr + _circle(6, 0.05, rot)
        _emit(jr, mr, room, t60, mics, mics.mean(axis=0), [src], [n], seed)
    return _finish("cfg2", 16000, jr, mr, n_rooms)


def config3(n_rooms: int = 4096, start: int = 0) -> Workload:
    """3 sources >= 1 m from an 8-mic 10 cm circle (configs[2])."""
    jr, mr = [], []
    for i in range(start, start + n_rooms):
        g = _rng(3, i)
        room = _room(g, 3.0, 12.0, 2.5, 4.5)
        t60 = g.uniform(0.2, 1.0)
        ctr = _inside(g, room, 0.5)
        rot = g.uniform(0.0, 2.0 * np.pi)
        srcs, ns = [], []
        for _ in range(3):
            while True:
                s = _inside(g, room, 0.5)
                if np.sqrt(((s - ctr) ** 2).sum()) >= 1.0:
                    break
            srcs.append(s)
            ns.append(g.integers(1024, 4097))
        seed = g.integers(2**63)
        mics = ctr + _circle(8, 0.10, rot)
        _emit(jr, mr, room, t60, mics, mics.mean(axis=0), srcs, ns, seed)
    return _finish("cfg3", 16000, jr, mr, n_rooms)


def config4(n_rooms: int = 512, start: int = 0) -> Workload:
    """48 kHz long-reverb rooms, 16-mic 4x4 grid, I ~ U{8192..16384} (configs[3])."""
    jr, mr = [], []
    for i in range(start, start + n_rooms):
        g = _rng(4, i)
        room = _room(g, 8.0, 20.0, 3.0, 6.0)
        t60 = g.uniform(1.0, 1.5)
        ctr = _inside(g, room, 0.5)
        rot = g.uniform(0.0, 2.0 * np.pi)
        srcs, ns = [], []
        for _ in range(2):
            while True:
                s = _inside(g, room, 0.5)
                if np.sqrt(((s - ctr) ** 2).sum()) >= 0.6:
                    break
            srcs.append(s)
            ns.append(g.integers(8192, 16385))
        seed = g.integers(2**63)
        mics = ctr + _grid(4, 0.04, rot)
        _emit(jr, mr, room, t60, mics, mics.mean(axis=0), srcs, ns, seed)
    return _finish("cfg4", 48000, jr, mr, n_rooms)


def config5(n_rooms: int = 65536, start: int = 0) -> Workload:
    """32 ad-hoc mics anywhere in the room, I ~ U{1024..8192} (configs[4])."""
    jr, mr = [], []
    for i in range(start, start + n_rooms):
        g = _rng(5, i)
        room = _room(g, 3.0, 10.0, 2.5, 4.0)
        t60 = g.uniform(0.1, 0.7)
        mics = g.uniform(0.3, room - 0.3, size=(32, 3))
        center = mics.mean(axis=0)
        while True:
            src = _inside(g, room, 0.5)
            if np.sqrt(((src - center) ** 2).sum()) >= 0.3:
                break
        n = g.integers(1024, 8193)
        seed = g.integers(2**63)
        _emit(jr, mr, room, t60, mics, center, [src], [n], seed)
    return _finish("cfg5", 16000, jr, mr, n_rooms)


BUILDERS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def build(cfg: int, n_rooms: int | None = None, start: int = 0) -> Workload:
    if cfg == 1:
        return config1()
    fn = BUILDERS[cfg]
    return fn(start=start) if n_rooms is None else fn(n_rooms=n_rooms, start=start)
