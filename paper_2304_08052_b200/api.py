"""Drop-in ``simulate_rir`` (reference core.py:268-316) on the B200 engine.

Validation runs first, in the reference's order and with its texts, so the
same inputs raise the same ``ValueError``; then every source of the scene is
rendered in ONE batched launch sequence (libfrir) and copied back as the
reference's ``RirResult`` objects.  The batched device API for dataloaders is
``simulate_batch`` (device tensors, no host round trip).
"""

from __future__ import annotations

import hashlib
import math

import numpy as np

from . import engine
from .rir import RirFilter, RirResult, rate_factors
from .scene import Scene, SimParams, array_center

HIGHPASS_HZ = 80.0


def reflection_coefficient(room_dims, t60: float) -> float:
    """Wall reflection coefficient from V/S and T60 (core.py:113-128)."""
    dims = np.asarray(room_dims, dtype=float)
    if dims.shape != (3,) or np.any(dims <= 0):
        raise ValueError(f"room_dims must be 3 positive lengths, got {room_dims}")
    if t60 <= 0:
        raise ValueError(f"t60 must be > 0, got {t60}")
    lx, ly, lz = dims
    ratio = (lx * ly * lz) / (2.0 * (lx * ly + lx * lz + ly * lz))
    return float(np.sqrt(1.0 - (1.0 - np.exp(-0.16 * ratio / t60)) ** 2))


def max_reflections(t60: float, d0: float, r: float, c0: float = 343.0) -> float:
    """Reflection count of the -60 dB arrival (core.py:186-192)."""
    if not 0.0 < r < 1.0:
        raise ValueError(f"reflection coefficient must be in (0, 1), got {r}")
    if c0 * t60 <= d0:
        raise ValueError("c0*t60 must exceed the direct distance")
    return (math.log10(c0 * t60) - math.log10(d0) - 3.0) / math.log10(r)


def scene_fingerprint(scene: Scene) -> str:
    """16-hex-digit sha256 of the geometry (params.py:174-186), metadata only."""
    parts = (
        np.asarray(scene.room_dims, dtype=float),
        np.atleast_2d(np.asarray(scene.mic_positions, dtype=float)),
        np.atleast_2d(np.asarray(scene.sources, dtype=float)),
        array_center(scene),
    )
    return hashlib.sha256(b"".join(p.tobytes() for p in parts)).hexdigest()[:16]


def _extensions(params):
    """(image range, early window or None, normalize) of a SimParams; works for
    the reference's own SimParams too (no extension fields -> reference behaviour)."""
    n = params.num_images
    rng = (int(n[0]), int(n[1])) if isinstance(n, (tuple, list)) else (int(n), int(n))
    window = tuple(getattr(params, "early_window_ms", (6.0, 50.0)))
    return rng, (None if window == (6.0, 50.0) else window), getattr(params, "normalize", None)


def _validate_sources(params: SimParams, scene: Scene, r: float) -> None:
    """Per-source checks in simulate_rir's order (core.py:140-148, 186-192, 209-210)."""
    srcs = np.atleast_2d(np.asarray(scene.sources, dtype=float))
    c_max = params.sound_speed * params.t60
    for d0 in srcs[:, 0]:
        if params.alpha == 0.0:
            raise ValueError("alpha must be > 0 to sample image distances")
        if c_max <= d0:
            raise ValueError(f"c0*t60 = {c_max:.3f} m must exceed the direct distance {d0:.3f} m")
        if _extensions(params)[0][1] > 0:
            rr = max_reflections(params.t60, float(d0), r, params.sound_speed)
            if rr < 1.0:
                raise ValueError(f"rr_max must be >= 1, got {rr}")


def scene_jobs(params: SimParams, scene: Scene, seed=None):
    """Job table (one job per source) and mic rows for one scene."""
    srcs = np.atleast_2d(np.asarray(scene.sources, dtype=float))
    mics = np.atleast_2d(np.asarray(scene.mic_positions, dtype=float))
    center = array_center(scene)
    jobs = engine.new_jobs(len(srcs))
    jobs["room"] = np.asarray(scene.room_dims, dtype=float)
    jobs["center"] = center
    jobs["d0"], jobs["az"], jobs["el"] = srcs[:, 0], srcs[:, 1], srcs[:, 2]
    jobs["t60"] = params.t60
    jobs["c0"] = params.sound_speed
    jobs["alpha"], jobs["beta"] = params.alpha, params.beta
    jobs["perturb_lo"], jobs["perturb_hi"] = params.perturb_lo, params.perturb_hi
    jobs["tau"] = params.tau
    jobs["seed"] = int(params.seed if seed is None else seed)
    jobs["source_index"] = np.arange(len(srcs))
    (lo, hi), window, normalize = _extensions(params)
    jobs["n_images"] = lo
    jobs["n_images_hi"] = hi if hi > lo else 0
    if window is not None:
        jobs["early_lo_ms"], jobs["early_hi_ms"] = window
    jobs["normalize"] = 1 if normalize == "direct" else 0
    jobs["mic_off"] = 0
    jobs["n_mics"] = len(mics)
    return jobs, mics


def simulate_rir(params: SimParams, scene: Scene, include_early: bool = True, *, device=None) -> list:
    """One RirResult per source, bit-reproducible for a fixed seed.

    Same contract as the reference (core.py:268-316): full filter and, when
    requested, the early [-6, +50] ms variant, both at ``params.sample_rate``.
    """
    factors = rate_factors(params.sample_rate)
    r = reflection_coefficient(scene.room_dims, params.t60)
    _validate_sources(params, scene, r)
    if not (0 <= int(params.seed) < 2**64):
        raise ValueError("seed must be in [0, 2**64)")
    jobs, mics = scene_jobs(params, scene)
    # one launch sequence for all sources; one copy each way (engine.CallRunner)
    pb, full_h, early_h, direct_h = engine.CallRunner.get(params.sample_rate, device).run(
        jobs, mics, include_early=include_early)
    direct_h = direct_h.astype(np.int64)

    meta_base = {
        "t60": params.t60, "seed": params.seed, "num_images": params.num_images,
        "alpha": params.alpha, "beta": params.beta, "perturb_lo": params.perturb_lo,
        "perturb_hi": params.perturb_hi, "tau": params.tau, "sound_speed": params.sound_speed,
        "sample_rate": params.sample_rate, "reflection_coefficient": r,
        "scene": scene_fingerprint(scene),
    }
    chain_meta = {"r_h": factors.r_h, "r_l": factors.r_l, "highpass_hz": HIGHPASS_HZ,
                  "direct_index_map": "round(high_rate_index / r_h)"}
    srcs = np.atleast_2d(np.asarray(scene.sources, dtype=float))
    pj = pb.jobs
    out = []
    for k in range(len(srcs)):
        meta = dict(meta_base, source_index=k, distance=float(srcs[k, 0]),
                    azimuth=float(srcs[k, 1]), elevation=float(srcs[k, 2]))
        (lo, hi), window, normalize = _extensions(params)
        if hi > lo:
            meta["num_images_drawn"] = int(pj[k]["n_images"])
        if window is not None:
            meta["early_window_ms"] = window
        if normalize is not None:
            meta["normalize"] = normalize
        meta.update(chain_meta)
        m, stride, n2, off = (int(pj[k][f]) for f in ("n_mics", "out_stride", "n2", "out_off"))
        ch = int(pj[k]["chan_off"])
        direct = direct_h[ch: ch + m].copy()

        def filt(buf, kind):
            samples = buf[off: off + m * stride].reshape(m, stride)[:, :n2].astype(np.float64)
            return RirFilter(samples=samples, direct_path_sample=direct.copy(),
                             sample_rate=factors.sample_rate, kind=kind, metadata=dict(meta))

        out.append(RirResult(full=filt(full_h, "full"),
                             early=filt(early_h, "early") if include_early else None))
    return out
