"""CPU oracle for the FRAM-RIR hot path -- TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference's ``simulate_rir`` path
(/root/reference/pkg/src/framrir/core.py:86-316 and resample.py:59-136),
written job-by-job: one job = one (room, source).  It reproduces the
reference's arithmetic and cost profile (dense high-rate train, scipy
``resample_poly`` / ``sosfilt``), so it serves both as the parity checker and
as the CPU baseline ``bench.py`` reports (``cpu_baseline.kind = "port"``).

Third-party arithmetic it relies on, exactly as the reference does: numpy
(Philox4x64-10 + SeedSequence, ``np.add.at``; reference pins numpy>=1.24,
pkg/pyproject.toml:10-14, run here with 2.3.5) and scipy (``firwin``,
``butter``, ``resample_poly``/``upfirdn``, ``sosfilt``; pinned scipy>=1.10, run
here with 1.18.1).  Pinned against the reference itself by
tests/test_oracle_golden.py with the fixtures tools/make_golden.py writes.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module.  The product (paper_2304_08052_b200) never does.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy import signal

C0_DEFAULT = 343.0


@dataclass
class Job:
    """One (room, source) with the reference's SimParams knobs."""

    room: tuple                 # room_dims
    mics: np.ndarray            # (M, 3) array-local frame
    center: np.ndarray          # reference point (params.py:149-153)
    source: tuple               # (d0, az, el) relative to center
    t60: float
    sample_rate: int = 16000
    num_images: int = 2048
    seed: int = 0
    source_index: int = 0
    alpha: float = 0.1
    beta: float = 1.0
    perturb_lo: float = -2.0
    perturb_hi: float = 2.0
    tau: float = 0.25
    sound_speed: float = C0_DEFAULT


@dataclass
class Draws:
    """The reference ImageSet fields for one job (core.py:43-62)."""

    distances: np.ndarray
    azimuths: np.ndarray
    elevations: np.ndarray
    reflections: np.ndarray
    mic_distances: np.ndarray = field(default=None)


def factors(fs: int):
    """(r_h, r_l) as resample.py:59-71."""
    r_h = 10**6 // int(fs)
    r_l = math.isqrt(r_h)
    if not 1 < r_l < r_h:
        raise ValueError(f"sample_rate {fs} leaves no room for the two-stage chain")
    return r_h, r_l


def wall_reflection(room, t60: float) -> float:
    """Eyring-style coefficient, core.py:113-128."""
    lx, ly, lz = np.asarray(room, dtype=float)
    vs = (lx * ly * lz) / (2.0 * (lx * ly + lx * lz + ly * lz))
    return float(np.sqrt(1.0 - (1.0 - np.exp(-0.16 * vs / t60)) ** 2))


def rr_limit(t60, d0, r, c0) -> float:
    """core.py:186-192."""
    return (math.log10(c0 * t60) - math.log10(d0) - 3.0) / math.log10(r)


def _gen(seed, k, stage):
    return np.random.Generator(np.random.Philox(np.random.SeedSequence((int(seed), int(k), int(stage)))))


def draw(job: Job) -> Draws:
    """Native draws of core.py:131-221 (stage-0 geometry, stage-1 perturbation)."""
    d0, az0, el0 = job.source
    c_max = job.sound_speed * job.t60
    n = job.num_images
    g0 = _gen(job.seed, job.source_index, 0)
    th = g0.uniform(0.0, 2.0 * np.pi, n)
    ph = g0.uniform(-np.pi / 2.0, np.pi / 2.0, n)
    u = g0.random(n)
    a, b = job.alpha, job.beta
    drh = np.cbrt(a**3 + (1.0 - u) * (b**3 - a**3))
    dr = 1.0 + (a / (b - a)) * (drh / a - 1.0) * (c_max / d0 - 1.0)
    dist = d0 * dr
    refl = np.zeros(n + 1)
    if n > 0:
        r = wall_reflection(job.room, job.t60)
        rr = rr_limit(job.t60, d0, r, job.sound_speed)
        if rr < 1.0:
            raise ValueError(f"rr_max must be >= 1, got {rr}")
        p = _gen(job.seed, job.source_index, 1).uniform(job.perturb_lo, job.perturb_hi, n)
        g = 1.0 + (dist / c_max) ** 2 * (rr - 1.0) + p * dr**job.tau
        refl[1:] = np.clip(g, 1.0, rr)
    return Draws(
        distances=np.concatenate([[d0], dist]),
        azimuths=np.concatenate([[az0], th]),
        elevations=np.concatenate([[el0], ph]),
        reflections=refl,
    )


def positions(job: Job, dr: Draws) -> np.ndarray:
    """center + sph_to_cart rows (params.py:138-159)."""
    d, az, el = dr.distances, dr.azimuths, dr.elevations
    off = np.stack([d * np.cos(el) * np.cos(az), d * np.cos(el) * np.sin(az), d * np.sin(el)], -1)
    return np.asarray(job.center, dtype=float) + off


def delays_gains(job: Job, dr: Draws):
    """Integer high-rate delays and gains per (image, mic), core.py:238-246."""
    r_h, _ = factors(job.sample_rate)
    rate = r_h * job.sample_rate
    L = math.ceil(job.t60 * rate)
    pos = positions(job, dr)
    mics = np.atleast_2d(np.asarray(job.mics, dtype=float))
    md = np.sqrt(((pos[:, None, :] - mics[None, :, :]) ** 2).sum(-1))
    dr.mic_distances = md
    q = np.minimum(np.ceil(md / job.sound_speed * rate).astype(np.int64), L - 1)
    r = wall_reflection(job.room, job.t60)
    amp = r ** dr.reflections[:, None] / md
    return q, amp, L, rate


def dense_train(q, amp, L):
    """np.add.at scatter into the (M, L) FP64 train, core.py:248-250."""
    x = np.zeros((q.shape[1], L))
    for m in range(q.shape[1]):
        np.add.at(x[m], q[:, m], amp[:, m])
    return x


def early_only(x, q0, rate, window_ms=None):
    """[-6, +50] ms window around each channel's direct arrival, core.py:254-265
    (``window_ms`` restates the product's early-window extension for tests)."""
    if window_ms is None:
        lo, hi = -(-6 * rate // 1000), -(-50 * rate // 1000)
    else:
        lo, hi = math.ceil(window_ms[0] * rate / 1000.0), math.ceil(window_ms[1] * rate / 1000.0)
    idx = np.arange(x.shape[1])
    keep = (idx[None, :] >= (q0[:, None] - lo)) & (idx[None, :] <= (q0[:, None] + hi))
    return np.where(keep, x, 0.0)


def chain(x, fs):
    """Stage-1 Kaiser decimation, 80 Hz HP, stage-2 decimation (resample.py:106-113)."""
    r_h, r_l = factors(fs)
    k1 = signal.firwin(20 * max(r_l, r_h) + 1, 1.0 / max(r_l, r_h), window=("kaiser", 7.0))
    y = signal.resample_poly(x, r_l, r_h, axis=1, window=k1)
    sos = signal.butter(2, 80.0, btype="highpass", fs=r_l * fs, output="sos")
    y = signal.sosfilt(sos, y, axis=1)
    k2 = signal.firwin(20 * r_l + 1, 1.0 / r_l, window=("kaiser", 7.0))
    return signal.resample_poly(y, 1, r_l, axis=1, window=k2)


def render(job: Job, draws: Draws | None = None, include_early: bool = True, early_window_ms=None):
    """Full (and early) RIR of one job: ``(full (M, n2), early or None, direct (M,))``."""
    if job.alpha == 0.0:
        raise ValueError("alpha must be > 0 to sample image distances")
    if job.sound_speed * job.t60 <= job.source[0]:
        raise ValueError("c0*t60 must exceed the direct distance")
    dr = draws if draws is not None else draw(job)
    q, amp, L, rate = delays_gains(job, dr)
    x = dense_train(q, amp, L)
    full = chain(x, job.sample_rate)
    r_h, _ = factors(job.sample_rate)
    direct = np.clip(np.round(q[0] / r_h).astype(np.int64), 0, full.shape[1] - 1)
    early = chain(early_only(x, q[0], rate, early_window_ms), job.sample_rate) if include_early else None
    return full, early, direct


def jobs_from_scene(params, scene):
    """One Job per source of a reference-shaped (SimParams, Scene) pair."""
    mics = np.atleast_2d(np.asarray(scene.mic_positions, dtype=float))
    if getattr(scene, "reference_point", None) is not None:
        center = np.asarray(scene.reference_point, dtype=float)
    else:
        center = mics.mean(axis=0)
    out = []
    for k, src in enumerate(np.atleast_2d(np.asarray(scene.sources, dtype=float))):
        out.append(Job(room=tuple(scene.room_dims), mics=mics, center=center, source=tuple(src),
                       t60=params.t60, sample_rate=params.sample_rate,
                       num_images=params.num_images, seed=params.seed, source_index=k,
                       alpha=params.alpha, beta=params.beta, perturb_lo=params.perturb_lo,
                       perturb_hi=params.perturb_hi, tau=params.tau,
                       sound_speed=params.sound_speed))
    return out
