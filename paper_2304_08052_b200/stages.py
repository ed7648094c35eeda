"""The reference's public stage functions on the device.

``framrir`` exports the stages ``simulate_rir`` is made of
(/root/reference/pkg/src/framrir/__init__.py:15-28, core.py:43-265,
resample.py:81-136): ``ImageSet``, ``HighRateTrain``,
``quadratic_ratio_sample``, ``rescale_distance_ratio``,
``sample_image_geometry``, ``sample_reflection_counts``,
``build_impulse_train``, ``early_reverb_train`` and
``downsample_highpass_downsample``.  Same names, arguments, return types and
``ValueError`` texts; the arithmetic runs in libfrir's stage kernels
(csrc/frir_stages.cu, frir_image_set in csrc/frir_kernels.cu) in FP64 with
numpy's operation order, and results come back as numpy arrays like the
reference's.  Random draws from a caller-supplied ``numpy.random.Generator``
are taken on the host in the reference's order (they are inputs); every
other draw comes from the device Philox streams, bit-identical to numpy's.

``downsample_highpass_downsample`` renders any (M, L) high-rate train through
the same sort / tail / render kernels as ``simulate_rir`` (its nonzero
samples become the items), so a caller that builds or edits trains by hand
gets the reference's filters to FP32 accuracy.  The batched hot path never
materialises these intermediates: use ``simulate_rir`` / ``engine`` for
throughput.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _abi
from .rir import RateFactors, RirFilter, rate_factors
from .scene import Scene, SimParams

__all__ = ["ImageSet", "HighRateTrain", "quadratic_ratio_sample", "rescale_distance_ratio",
           "sample_image_geometry", "sample_reflection_counts", "build_impulse_train", "early_reverb_train",
           "downsample_highpass_downsample"]


@dataclass
class ImageSet:
    """Virtual-source population for one source; row 0 is the direct path (core.py:43-62)."""

    distances: np.ndarray        # (I+1,) distance to the array reference point
    azimuths: np.ndarray         # (I+1,) rad
    elevations: np.ndarray       # (I+1,) rad
    distance_ratios: np.ndarray  # (I+1,) D_i / direct distance, 1.0 for row 0
    mic_distances: np.ndarray    # (I+1, M) per-mic propagation distances
    reflections: np.ndarray      # (I+1,) fractional reflection counts, 0 for row 0
    direct_distance: float
    source_index: int = 0

    @property
    def n_images(self) -> int:
        return len(self.distances) - 1

    @property
    def direct_mic_distances(self) -> np.ndarray:
        return self.mic_distances[0]


@dataclass
class HighRateTrain:
    """Multi-channel impulse train at the oversampled rate (core.py:65-75)."""

    channels: np.ndarray      # (M, L)
    direct_index: np.ndarray  # (M,) sample of the direct impulse per channel
    rate: int                 # Hz, r_h * sample_rate

    @property
    def length(self) -> int:
        return self.channels.shape[1]


# ---------------------------------------------------------------- plumbing
def _torch():
    import torch

    return torch


def _dev():
    from . import engine

    engine.require_cuda()
    torch = _torch()
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(a, dtype=np.float64):
    torch = _torch()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=dtype)).to(_dev())


def _stream():
    return _torch().cuda.current_stream().cuda_stream


def _eval(op, params, *xs):
    torch = _torch()
    x = [_to_dev(v) for v in xs]
    n = x[0].numel()
    out = torch.empty(n, dtype=torch.float64, device=x[0].device)
    ptrs = [t.data_ptr() for t in x] + [None] * (3 - len(x))
    prm = (ctypes.c_double * 4)(*(list(params) + [0.0] * (4 - len(params))))
    _abi.check(_abi.lib().frir_stage_eval(op, ptrs[0], ptrs[1], ptrs[2], n, prm, out.data_ptr(), _stream()),
               "frir_stage_eval")
    return out.cpu().numpy()


# ---------------------------------------------------------------- core.py stages
def quadratic_ratio_sample(rng: np.random.Generator, n: int, alpha: float, beta: float) -> np.ndarray:
    """Draws of the density 3x^2/(beta^3 - alpha^3) on (alpha, beta] by the
    inverse CDF (core.py:94-100); ``rng.random(n)`` is consumed exactly as the
    reference does."""
    u = rng.random(n)
    return _eval(_abi.STAGE_RATIO_SAMPLE, (alpha ** 3, beta ** 3), u).reshape(np.shape(u))


def rescale_distance_ratio(dr_hat, alpha: float, beta: float, max_ratio: float):
    """Map raw draws on (alpha, beta] linearly onto [1, max_ratio] (core.py:103-110)."""
    dr_hat = np.asarray(dr_hat, dtype=float)
    return _eval(_abi.STAGE_RESCALE, (alpha, beta, max_ratio), dr_hat.reshape(-1)).reshape(dr_hat.shape)


def _source_job(params: SimParams, scene: Scene, source_index: int):
    from . import engine
    from .api import scene_jobs

    jobs, mics = scene_jobs(params, scene)
    if not 0 <= source_index < len(jobs):
        raise IndexError(f"source_index {source_index} out of range")
    job = jobs[source_index: source_index + 1].copy()
    job["mic_off"] = 0
    return engine.prepare(params.sample_rate, job, mics)


def sample_image_geometry(params: SimParams, scene: Scene, source_index: int = 0) -> ImageSet:
    """Virtual-source positions of one source (core.py:131-183) from the
    device stage-0 Philox stream; reflection counts stay NaN (row 0: 0) until
    ``sample_reflection_counts``."""
    if params.alpha == 0.0:
        raise ValueError("alpha must be > 0 to sample image distances")
    srcs = np.atleast_2d(np.asarray(scene.sources, dtype=float))
    d0 = float(srcs[source_index][0])
    c_max = params.sound_speed * params.t60
    if c_max <= d0:
        raise ValueError(f"c0*t60 = {c_max:.3f} m must exceed the direct distance {d0:.3f} m")
    return _image_set(params, scene, source_index, with_reflections=False)


def _image_set(params, scene, source_index, with_reflections):
    from . import engine

    torch = _torch()
    pb = _source_job(params, scene, source_index)
    db = engine.DeviceBatch(pb, device=_dev(), workspace=False)
    rows = int(pb.jobs[0]["n_images"]) + 1
    M = int(pb.jobs[0]["n_mics"])
    f = [torch.empty(rows, dtype=torch.float64, device=db.device) for _ in range(5)]
    md = torch.empty(rows * M, dtype=torch.float64, device=db.device)
    _abi.check(_abi.lib().frir_image_set(db.plan.handle, ctypes.byref(db.batch), *(t.data_ptr() for t in f),
                                         md.data_ptr(), int(with_reflections), _stream()), "frir_image_set")
    d, az, el, ratio, refl = (t.cpu().numpy() for t in f)
    return ImageSet(distances=d, azimuths=az, elevations=el, distance_ratios=ratio,
                    mic_distances=md.cpu().numpy().reshape(rows, M), reflections=refl,
                    direct_distance=float(d[0]), source_index=int(source_index))


def sample_reflection_counts(images: ImageSet, params: SimParams, rr_max: float,
                             rng: np.random.Generator | None = None) -> ImageSet:
    """Fill the fractional reflection counts of every non-direct image
    (core.py:195-221): perturbation p from ``rng`` if given, else from the
    device stream (seed, source_index, 1); clamped to [1, rr_max]."""
    if rr_max < 1.0:
        raise ValueError(f"rr_max must be >= 1, got {rr_max}")
    n = images.n_images
    if rng is not None:
        p = _to_dev(rng.uniform(params.perturb_lo, params.perturb_hi, n))
    else:
        torch = _torch()
        p = torch.empty(n, dtype=torch.float64, device=_dev())
        if n:
            _abi.check(_abi.lib().frir_philox_uniform(int(params.seed), int(images.source_index), 1, 0, n,
                                                      float(params.perturb_lo), float(params.perturb_hi),
                                                      p.data_ptr(), _stream()), "frir_philox_uniform")
    if n:
        g = _eval(_abi.STAGE_REFLECTIONS, (params.sound_speed * params.t60, float(rr_max), params.tau),
                  images.distances[1:], images.distance_ratios[1:], p.cpu().numpy())
        images.reflections[1:] = g
    images.reflections[0] = 0.0
    return images


def build_impulse_train(images: ImageSet, params: SimParams, r: float) -> HighRateTrain:
    """All arrivals in a high-rate (M, L) train (core.py:228-251): index
    ceil(D/c0 * rate) clamped to L - 1, amplitude r**g / D, collisions summed
    in row order like ``np.add.at``."""
    if np.any(np.isnan(images.reflections)):
        raise ValueError("reflection counts not sampled; call sample_reflection_counts first")
    torch = _torch()
    factors = rate_factors(params.sample_rate)
    rate = factors.r_h * params.sample_rate
    length = math.ceil(params.t60 * rate)
    md = _to_dev(images.mic_distances)
    rows, M = images.mic_distances.shape
    refl = _to_dev(images.reflections)
    lib = _abi.lib()
    nscr = int(lib.frir_impulse_train_scratch(rows, M, length))
    scratch = torch.empty(nscr, dtype=torch.uint8, device=md.device)
    train = torch.empty(M * length, dtype=torch.float64, device=md.device)
    q = torch.empty(rows * M, dtype=torch.int32, device=md.device)
    _abi.check(lib.frir_impulse_train(md.data_ptr(), refl.data_ptr(), rows, M, float(r), float(params.sound_speed),
                                      int(rate), int(length), train.data_ptr(), q.data_ptr(), scratch.data_ptr(),
                                      nscr, _stream()), "frir_impulse_train")
    q0 = q.view(rows, M)[0].cpu().numpy().astype(np.int64)
    return HighRateTrain(channels=train.view(M, length).cpu().numpy(), direct_index=q0, rate=int(rate))


def early_reverb_train(train: HighRateTrain, params: SimParams) -> HighRateTrain:
    """Only the [-6, +50] ms context around each channel's direct path (core.py:254-265)."""
    torch = _torch()
    rate = train.rate
    lo, hi = -(-6 * rate // 1000), -(-50 * rate // 1000)
    x = _to_dev(train.channels)
    M, L = train.channels.shape
    q0 = _to_dev(train.direct_index, np.int32)
    out = torch.empty_like(x)
    _abi.check(_abi.lib().frir_early_window(x.data_ptr(), M, L, q0.data_ptr(), int(lo), int(hi), out.data_ptr(),
                                            _stream()), "frir_early_window")
    return HighRateTrain(channels=out.cpu().numpy(), direct_index=train.direct_index.copy(), rate=rate)


# ---------------------------------------------------------------- resample.py
def _render_train(x, sample_rate):
    """Full-variant filters of the rows of a device (M, L) FP64 train."""
    from . import engine

    torch = _torch()
    M, L = x.shape
    lib = _abi.lib()
    out = None
    for sign in (1, -1):
        cnt = torch.empty(M, dtype=torch.int32, device=x.device)
        _abi.check(lib.frir_train_nonzeros(x.data_ptr(), L, M, L, sign, cnt.data_ptr(), _stream()),
                   "frir_train_nonzeros")
        rows = int(cnt.max()) if M else 0
        if sign == -1 and rows == 0:
            break
        job = engine.new_jobs(1)
        job["kind"] = _abi.KIND_TRAIN
        job["duration"] = float(L)
        job["n_images"] = max(rows, 1) - 1
        job["n_mics"] = M
        job["d0"] = 1.0
        pb = engine.prepare(sample_rate, job, np.zeros((M, 3)))
        db = engine.DeviceBatch(pb, device=x.device, workspace=True)
        y = torch.empty(int(pb.batch.total_out), dtype=torch.float32, device=x.device)
        direct = torch.empty(M, dtype=torch.int32, device=x.device)
        _abi.check(lib.frir_simulate_train(db.plan.handle, ctypes.byref(db.batch), db.workspace.data_ptr(),
                                           db.workspace.numel(), x.data_ptr(), L, sign, y.data_ptr(),
                                           direct.data_ptr(), _stream()), "frir_simulate_train")
        n2, stride = int(pb.jobs[0]["n2"]), int(pb.jobs[0]["out_stride"])
        y = y.view(M, stride)[:, :n2]
        out = y.double() if out is None else out - y.double()
    return out


def downsample_highpass_downsample(train, factors: RateFactors, highpass_hz: float = 80.0,
                                   kaiser_beta: float = 7.0, taps_per_phase: int = 10, kind: str = "full",
                                   metadata: dict | None = None) -> RirFilter:
    """The two-stage decimation chain with the 80 Hz high-pass between
    (resample.py:81-136), for a HighRateTrain or an (M, L) array at
    ``factors.high_rate``; direct index round(index / r_h) (zeros for arrays)."""
    if (highpass_hz, kaiser_beta, taps_per_phase) != (80.0, 7.0, 10):
        raise NotImplementedError("the device filter tables implement the reference's chain "
                                  "(highpass_hz=80, kaiser_beta=7, taps_per_phase=10)")
    if hasattr(train, "channels"):
        x = np.atleast_2d(train.channels)
        direct_hi = np.asarray(train.direct_index)
    else:
        x = np.atleast_2d(np.asarray(train, dtype=float))
        direct_hi = None
    if x.size == 0:
        raise ValueError("empty train")
    y = _render_train(_to_dev(x), factors.sample_rate).cpu().numpy()
    n_out = y.shape[1]
    if direct_hi is not None:
        direct = np.clip(np.round(direct_hi / factors.r_h).astype(np.int64), 0, n_out - 1)
    else:
        direct = np.zeros(x.shape[0], dtype=np.int64)
    meta = dict(metadata or {})
    meta.update({"r_h": factors.r_h, "r_l": factors.r_l, "highpass_hz": highpass_hz,
                 "direct_index_map": "round(high_rate_index / r_h)"})
    return RirFilter(samples=y, direct_path_sample=direct, sample_rate=factors.sample_rate, kind=kind,
                     metadata=meta)
