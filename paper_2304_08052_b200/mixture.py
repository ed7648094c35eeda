"""Spatialise-and-mix on the GPU.

Mirrors the reference's consumer of the RIR path,
``framrir.mixture.spatialize_and_mix`` (/root/reference/pkg/src/framrir/
mixture.py:225-332) and its ``MixtureSpec`` / ``MixtureResult`` types
(:38-80, :107-113): same arguments, defaults, random draws (in the same order
from the caller's ``numpy`` Generator), ``ValueError`` texts and metadata.

The convolutions run batched on the device in libfrir's own partitioned
overlap-save FFT convolution (``include/frir.h``: frir_mix_convolve, 8192-point
shared-memory FFTs), then its kernels for the FP64 reference-channel powers,
the SIR/SNR gains and the scaled references plus the mixture
(frir_mix_powers / frir_mix_gains / frir_mix_combine).  ``mix_device`` is the
batched tensor API (many utterances per launch); ``spatialize_and_mix`` is the
drop-in for one utterance with numpy in and out.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, replace

import numpy as np

from . import _abi

__all__ = ["MixtureSpec", "CurriculumState", "MixtureResult", "SyntheticPool", "curriculum_step",
           "sample_scene", "scene_batch_jobs", "spatialize_and_mix", "mix_device", "generate_batch"]


def _check_range(name, rng):
    lo, hi = rng
    if lo > hi:
        raise ValueError(f"{name} range is empty: {rng}")


@dataclass
class MixtureSpec:
    """Sampling ranges for one training utterance (mixture.py:38-80)."""

    n_speakers: int = 2
    sir_db: tuple = (-6.0, 6.0)
    snr_db: tuple = (10.0, 20.0)
    min_overlap_ratio: float = 0.5
    speaker_distance: tuple = (0.3, 6.0)
    t60_range: tuple = (0.1, 0.7)
    room_length: tuple = (3.0, 10.0)
    room_width: tuple = (3.0, 10.0)
    room_height: tuple = (2.5, 4.0)
    elevation_range: tuple = (-np.pi / 4, np.pi / 4)
    mic_spacings: tuple = (0.04, 0.08, 0.04)
    sample_rate: int = 16000
    num_images: int = 2048
    utterance_seconds: float = 4.0
    sir_scope: str = "full"  # "full" or "overlap" (interferer power over the overlap only)

    def __post_init__(self):
        if self.n_speakers < 1:
            raise ValueError("need at least one speaker")
        for name in ("sir_db", "snr_db", "speaker_distance", "t60_range", "room_length",
                     "room_width", "room_height", "elevation_range"):
            _check_range(name, getattr(self, name))
        if not 0.0 <= self.min_overlap_ratio <= 1.0:
            raise ValueError("min_overlap_ratio must be in [0, 1]")
        if self.sir_scope not in ("full", "overlap"):
            raise ValueError("sir_scope must be 'full' or 'overlap'")


@dataclass(frozen=True)
class CurriculumState:
    """Epoch-indexed cap on the sampled decay range, in milliseconds (mixture.py:83-96)."""

    epoch: int = 0
    lower_ms: float = 50.0
    upper_ms: float = 100.0
    step_ms: float = 50.0
    max_ms: float = 700.0

    @property
    def t60_bounds(self) -> tuple:
        return self.lower_ms / 1000.0, self.upper_ms / 1000.0


def curriculum_step(state: CurriculumState) -> CurriculumState:
    """Advance one epoch: raise the upper bound by the step, capped (mixture.py:99-105)."""
    return replace(state, epoch=state.epoch + 1, upper_ms=min(state.upper_ms + state.step_ms, state.max_ms))


@dataclass(frozen=True)
class SyntheticPool:
    """Self-contained source material: amplitude-modulated filtered noise
    (mixture.py:116-139), drawn on the host from the caller's rng exactly as
    the reference draws it (normals, leaky integrator, envelope phase)."""

    lowpass_hz: float = 3800.0
    modulation_hz: float = 3.0

    def draw(self, rng, n_samples: int, sample_rate: int) -> np.ndarray:
        from scipy.signal import lfilter

        x = rng.standard_normal(n_samples)
        a = math.exp(-2.0 * math.pi * self.lowpass_hz / sample_rate)
        x = lfilter([1.0 - a], [1.0, -a], x)
        x -= x.mean()
        t = np.arange(n_samples) / sample_rate
        phase = rng.uniform(0.0, 2.0 * np.pi)
        envelope = 0.55 + 0.45 * np.sin(2.0 * np.pi * self.modulation_hz * t + phase)
        x = x * envelope
        peak = np.abs(x).max()
        return x / peak if peak > 0 else x


@dataclass
class WavDirectoryPool:
    """Clean mono WAV files from a user-supplied directory (mixture.py:143-168):
    a file and a start drawn from the caller's rng in the reference's order;
    integer PCM normalised by its type range (io.py:39-55).  Source material
    I/O on the host, like the reference's."""

    directory: str

    def _files(self):
        import pathlib

        files = sorted(pathlib.Path(self.directory).glob("*.wav"))
        if not files:
            raise ValueError(f"no .wav files under {self.directory}")
        return files

    @staticmethod
    def _read(path):
        from scipy.io import wavfile

        fs, data = wavfile.read(path)
        scale = {np.dtype(np.int16): 32768.0, np.dtype(np.int32): 2147483648.0}.get(data.dtype)
        if scale is not None:
            data = data / scale
        elif data.dtype == np.uint8:
            data = (data.astype(float) - 128.0) / 128.0
        else:
            data = data.astype(np.float64)
        return (data[None, :] if data.ndim == 1 else data.T), int(fs)

    def draw(self, rng, n_samples: int, sample_rate: int) -> np.ndarray:
        files = self._files()
        x, fs = self._read(files[int(rng.integers(len(files)))])
        if fs != sample_rate:
            raise ValueError(f"expected {sample_rate} Hz material, got {fs} Hz")
        x = x[0] if x.ndim == 2 else x
        if len(x) >= n_samples:
            start = int(rng.integers(len(x) - n_samples + 1))
            return x[start: start + n_samples]
        reps = int(np.ceil(n_samples / len(x)))
        return np.tile(x, reps)[:n_samples]


def sample_scene(spec: MixtureSpec, rng, curriculum: CurriculumState | None = None) -> tuple:
    """One utterance's (Scene, SimParams), drawing from ``rng`` in the
    reference's order (mixture.py:171-213): room (3 uniforms), T60, then per
    speaker and the point noise (last) distance / azimuth / elevation, then
    the simulation seed."""
    from .scene import Scene, SimParams, linear_array

    room = (rng.uniform(*spec.room_length), rng.uniform(*spec.room_width), rng.uniform(*spec.room_height))
    lo, hi = curriculum.t60_bounds if curriculum is not None else spec.t60_range
    t60 = rng.uniform(lo, hi)
    placements = []
    for _ in range(spec.n_speakers + 1):  # + point noise
        placements.append((rng.uniform(*spec.speaker_distance), rng.uniform(0.0, 2.0 * np.pi),
                           rng.uniform(*spec.elevation_range)))
    scene = Scene(room_dims=room, mic_positions=linear_array(spec.mic_spacings), sources=placements)
    params = SimParams(t60=t60, sample_rate=spec.sample_rate, num_images=spec.num_images,
                       seed=int(rng.integers(2**63)))
    return scene, params


def scene_batch_jobs(scenes, params):
    """One job table (one job per (scene, source), scenes in order) and the
    concatenated mic rows, for rendering many utterances' RIRs in one launch."""
    from .api import scene_jobs

    jobs, mics, off = [], [], 0
    for sc, pr in zip(scenes, params):
        j, m = scene_jobs(pr, sc)
        j["mic_off"] = off
        off += len(m)
        jobs.append(j)
        mics.append(m)
    return np.concatenate(jobs), np.concatenate(mics, axis=0)


@dataclass
class MixtureResult:
    mixture: np.ndarray          # (M, N)
    sources: list                # per speaker, (M, N) reverberant reference
    early_sources: list          # per speaker, (M, N) early-reverb reference
    noise: np.ndarray            # (M, N)
    metadata: dict


def _torch():
    import torch

    return torch


def _upload(dev, parts):
    """Device copies of small host arrays through one pinned staging block and
    one non-blocking copy on the current stream; returns views of one device
    buffer in the order given (int32 / int64 / float64)."""
    torch = _torch()
    dt = {np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64, np.dtype(np.float64): torch.float64}
    offs, n = [], 0
    for a in parts:
        n = (n + 7) & ~7
        offs.append(n)
        n += a.nbytes
    host = torch.empty(max(n, 8), dtype=torch.uint8, pin_memory=True)
    hv = host.numpy()
    for a, o in zip(parts, offs):
        hv[o:o + a.nbytes] = np.ascontiguousarray(a).view(np.uint8).ravel()
    buf = host.to(dev, non_blocking=True)  # the caching host allocator keeps `host` until the copy is done
    return [buf[o:o + a.nbytes].view(dt[a.dtype]) for a, o in zip(parts, offs)]


def mix_device(dry, dry_len, offsets, noise, noise_len, rir_full, rir_early, rir_len, sir_db, snr_db,
               sir_scope: str = "full"):
    """Batched spatialise-and-mix of B utterances on one device.

    dry (B, S, N) float32 with valid lengths dry_len (B, S); offsets (B, S)
    (offsets[:, 0] == 0); noise (B, Nn) with lengths noise_len (B,);
    rir_full (B, S + 1, M, R) float32 (the noise filter last) with valid
    lengths rir_len (B,); rir_early (B, >= S, M, R) or None (then the full
    filter, as the reference copies the full image) -- both may be strided
    views over the render's padded output (per-item blocks contiguous); sir_db (B, max(S - 1, 1)) and
    snr_db (B,) in dB.  Integer/size arguments are host arrays.  Returns a dict
    of device tensors: mixture (B, M, T), sources and early (B, S, M, T), noise
    (B, M, T), gains (B, S + 1) [speaker gains then the noise gain], total (B,)
    valid lengths (T = max total).  Samples past an item's total are zero.
    """
    torch = _torch()
    dev = rir_full.device
    B, S1, M, R = rir_full.shape
    S = S1 - 1
    if S < 1 or dry.shape[:2] != (B, S):
        raise ValueError("need one RIR per speaker plus one for the noise")
    dry_len = np.asarray(dry_len, dtype=np.int64).reshape(B, S)
    offsets = np.asarray(offsets, dtype=np.int64).reshape(B, S)
    noise_len = np.asarray(noise_len, dtype=np.int64).reshape(B)
    rir_len = np.asarray(rir_len, dtype=np.int64).reshape(B)
    total = (offsets + dry_len).max(axis=1) + rir_len - 1          # mixture.py:272
    T = int(total.max()) if B else 0
    lib = _abi.lib()
    stream = torch.cuda.current_stream(dev).cuda_stream
    dry = dry.contiguous()
    noise = noise.contiguous()
    # filters: each item's [S(+1)][M][R] block must be contiguous; items may be strided
    if rir_full.stride()[1:] != (M * R, R, 1):
        rir_full = rir_full.contiguous()
    if rir_early is not None and (rir_early.shape[0] != B or rir_early.shape[1] < S
                                  or rir_early.shape[2:] != (M, R)):
        raise ValueError("rir_early must be (B, >= S, M, R) like rir_full")
    if rir_early is not None and rir_early.stride()[1:] != (M * R, R, 1):
        rir_early = rir_early.contiguous()
    J = (2 * S + 1) * M
    dlen = total - rir_len + 1
    # reference-channel power requests (mixture.py:284-303, 311), per item:
    # p_ref, (p_int_k, p_tgt_k) for k = 1..S-1, p_noise
    base = np.arange(B, dtype=np.int64) * J
    rows = np.empty((B, 2 * S), dtype=np.int64)
    lo = np.zeros((B, 2 * S), dtype=np.int64)
    hi = np.repeat(total[:, None], 2 * S, axis=1).astype(np.int64)
    rows[:, 0] = base
    rows[:, 2 * S - 1] = base + 2 * S * M
    for k in range(1, S):
        rows[:, 2 * k - 1] = base + k * M
        rows[:, 2 * k] = base
        if sir_scope == "overlap":
            a = offsets[:, k]
            e = np.minimum(total, offsets[:, k] + dry_len[:, k] + rir_len - 1)
            lo[:, 2 * k - 1] = lo[:, 2 * k] = a
            hi[:, 2 * k - 1] = hi[:, 2 * k] = e
    rows, lo, hi = rows.ravel(), lo.ravel(), hi.ravel()
    i32 = lambda a: np.asarray(a, dtype=np.int32).ravel()  # noqa: E731
    # every small per-item table in one pinned block and one async copy (no
    # pageable copies that would stall the host behind the queued kernels)
    (off_d, len_d, nlen_d, dlen_d, rl, req_row, req_lo, req_hi, tot_d, sir, snr) = _upload(dev, [
        i32(offsets), i32(dry_len), i32(noise_len), i32(dlen), i32(rir_len), rows, i32(lo), i32(hi), i32(total),
        np.asarray(sir_db, dtype=np.float64).reshape(B * max(S - 1, 1)),
        np.asarray(snr_db, dtype=np.float64).reshape(B)])
    # convolution of every filter row with its source: libfrir's hand-written
    # partitioned overlap-save FFT convolution (placed speakers, tiled noise)
    ys = ctypes.c_int64(0)
    nscr = lib.frir_mix_convolve_scratch(B, S, M, R, T, ctypes.byref(ys))
    F = int(ys.value)  # row stride of y
    scratch = torch.empty(max(int(nscr), 1), dtype=torch.uint8, device=dev)
    y = torch.empty((B, J, F), dtype=torch.float32, device=dev)
    _abi.check(lib.frir_mix_convolve(
        dry.data_ptr(), dry.stride(0), dry.stride(1), noise.data_ptr(), noise.stride(0), off_d.data_ptr(),
        len_d.data_ptr(), nlen_d.data_ptr(), dlen_d.data_ptr(), rir_full.data_ptr(), rir_full.stride(0),
        rir_early.data_ptr() if rir_early is not None else None, rir_early.stride(0) if rir_early is not None else 0,
        rl.data_ptr(), B, S, M, R, T, scratch.data_ptr(), scratch.numel(), y.data_ptr(), F, stream),
        "frir_mix_convolve")
    del scratch
    pw = torch.empty(len(rows), dtype=torch.float64, device=dev)
    scratch = torch.empty(len(rows) * _abi.MIX_POWER_CHUNKS, dtype=torch.float64, device=dev)
    _abi.check(lib.frir_mix_powers(y.data_ptr(), F, req_row.data_ptr(), req_lo.data_ptr(),
                                   req_hi.data_ptr(), len(rows), scratch.data_ptr(), pw.data_ptr(), stream),
               "frir_mix_powers")
    gains = torch.empty((B, S + 1), dtype=torch.float64, device=dev)
    _abi.check(lib.frir_mix_gains(pw.data_ptr(), sir.data_ptr(), snr.data_ptr(), B, S, gains.data_ptr(),
                                  stream), "frir_mix_gains")
    out = {
        "mixture": torch.empty((B, M, T), dtype=torch.float32, device=dev),
        "sources": torch.empty((B, S, M, T), dtype=torch.float32, device=dev),
        "early": torch.empty((B, S, M, T), dtype=torch.float32, device=dev),
        "noise": torch.empty((B, M, T), dtype=torch.float32, device=dev),
    }
    _abi.check(lib.frir_mix_combine(y.data_ptr(), gains.data_ptr(), tot_d.data_ptr(), B, S, M, F, T,
                                    out["mixture"].data_ptr(), out["sources"].data_ptr(),
                                    out["early"].data_ptr(), out["noise"].data_ptr(), stream),
               "frir_mix_combine")
    out["gains"] = gains
    out["total"] = total
    out["powers"] = pw
    return out


def _draw_offsets(sources, spec: MixtureSpec, rng):
    """mixture.py:245-257: overlap-constrained offsets from the caller's rng."""
    n0 = len(sources[0])
    offsets = [0]
    for k in range(1, len(sources)):
        need = math.ceil(spec.min_overlap_ratio * min(n0, len(sources[k])))
        hi = n0 - need
        if hi < 0:
            raise ValueError(f"speaker {k} is shorter than the required overlap window")
        offsets.append(int(rng.integers(0, hi + 1)))
    return offsets


def _overlap_ratio(n0, off, nk):
    return max(0, min(n0, off + nk) - off) / min(n0, nk)


def spatialize_and_mix(sources: list, noise: np.ndarray, rirs: list, spec: MixtureSpec, rng,
                       sir_db: list | None = None, snr_db: float | None = None,
                       offsets: list | None = None, *, device=None) -> MixtureResult:
    """Convolve, overlap and scale one utterance (drop-in for mixture.py:225-332).

    ``rirs`` holds one RirResult per speaker plus one for the noise (last).
    Offsets, SIR and SNR are drawn from ``rng`` exactly as the reference does
    when not given; the arrays are computed on the GPU (FP32 samples, FP64
    powers and gains) and returned as float64 numpy arrays like the reference.
    """
    torch = _torch()
    if len(rirs) != len(sources) + 1:
        raise ValueError("need one RIR per speaker plus one for the noise")
    n0 = len(sources[0])
    if offsets is None:
        offsets = _draw_offsets(sources, spec, rng)
    for k in range(1, len(sources)):
        achieved = _overlap_ratio(n0, offsets[k], len(sources[k]))
        if achieved < spec.min_overlap_ratio:
            raise ValueError(
                f"speaker {k} overlap ratio {achieved:.2f} is below the "
                f"required {spec.min_overlap_ratio}"
            )
    S = len(sources)
    if sir_db is None:
        sir_db = [float(rng.uniform(*spec.sir_db)) for _ in range(S - 1)]
    if snr_db is None:
        snr_db = float(rng.uniform(*spec.snr_db))
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())

    R = rirs[0].full.n_samples
    M = rirs[0].full.samples.shape[0]
    lens = [len(s) for s in sources]
    N = max(lens)
    dry = np.zeros((1, S, N), dtype=np.float32)
    for k, s in enumerate(sources):
        dry[0, k, :len(s)] = s
    rf = np.zeros((1, S + 1, M, R), dtype=np.float32)
    re = np.zeros((1, S, M, R), dtype=np.float32)
    for k, r in enumerate(rirs):
        rf[0, k] = r.full.samples[:, :R]
        if k < S:
            re[0, k] = (r.early if r.early is not None else r.full).samples[:, :R]
    nz = np.asarray(noise, dtype=np.float32)[None, :]
    out = mix_device(
        torch.from_numpy(dry).to(dev), [lens], [offsets], torch.from_numpy(nz).to(dev), [len(noise)],
        torch.from_numpy(rf).to(dev), torch.from_numpy(re).to(dev), [R],
        [list(sir_db) if S > 1 else [0.0]], [snr_db],
        sir_scope=spec.sir_scope,
    )
    T = int(out["total"][0])
    mixture = out["mixture"][0, :, :T].double().cpu().numpy()
    srcs = out["sources"][0, :, :, :T].double().cpu().numpy()
    early = out["early"][0, :, :, :T].double().cpu().numpy()
    noise_img = out["noise"][0, :, :T].double().cpu().numpy()
    gains = out["gains"][0].cpu().numpy()
    overlap_ratios = [_overlap_ratio(n0, offsets[k], len(sources[k])) for k in range(1, S)]
    return MixtureResult(
        mixture=mixture,
        sources=[srcs[k] for k in range(S)],
        early_sources=[early[k] for k in range(S)],
        noise=noise_img,
        metadata={
            "offsets": list(offsets),
            "gains": [float(g) for g in gains[:S]],
            "noise_gain": float(gains[S]),
            "sir_db": list(sir_db),
            "snr_db": snr_db,
            "overlap_ratios": overlap_ratios,
        },
    )


def _item_draws(args):
    """Host draws of one utterance in the reference's order (mixture.py:335-342,
    then spatialize_and_mix's offsets / SIR / SNR, :245-263)."""
    spec, curriculum, seed, i, pool = args
    S = spec.n_speakers
    fs = spec.sample_rate
    n_dry = int(spec.utterance_seconds * spec.sample_rate)
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence((int(seed), int(i)))))
    sc, pr = sample_scene(spec, rng, curriculum)
    srcs = [pool.draw(rng, n_dry, fs) for _ in range(S)]
    nz = pool.draw(rng, n_dry, fs)
    offs = _draw_offsets(srcs, spec, rng)
    for k in range(1, S):
        achieved = _overlap_ratio(len(srcs[0]), offs[k], len(srcs[k]))
        if achieved < spec.min_overlap_ratio:
            raise ValueError(f"speaker {k} overlap ratio {achieved:.2f} is below the "
                             f"required {spec.min_overlap_ratio}")
    sir = [float(rng.uniform(*spec.sir_db)) for _ in range(S - 1)]
    snr = float(rng.uniform(*spec.snr_db))
    return (sc, pr, np.stack([np.asarray(x, dtype=np.float32) for x in srcs]), np.asarray(nz, dtype=np.float32),
            offs, sir, snr)


def generate_batch(batch_size: int, spec: MixtureSpec, curriculum: CurriculumState | None = None, seed: int = 0,
                   workers: int = 1, pool=None, executor=None, *, device=None) -> list:
    """``batch_size`` independent utterances (drop-in for mixture.py:365-395).

    Every random draw happens on the host in the reference's order from the
    per-item stream Philox(SeedSequence((seed, index))) -- scene, dry sources
    and noise, offsets, SIR, SNR -- so the content matches the reference item
    for item.  All RIRs of the batch then render in ONE device launch (full +
    early, (n_speakers + 1) sources per item) and are mixed on the device in
    one ``mix_device`` call.  ``workers`` (threads) or ``executor`` (any
    ``map``-capable executor) parallelise the host draws.
    """
    if batch_size < 0:
        raise ValueError("batch_size must be >= 0")
    if batch_size == 0:
        return []
    torch = _torch()
    from . import engine

    pool = SyntheticPool() if pool is None else pool
    S = spec.n_speakers
    fs = spec.sample_rate
    n_dry = int(spec.utterance_seconds * spec.sample_rate)
    # per-item streams are independent: the host draws run on `executor`
    # (e.g. a warm ProcessPoolExecutor, as the reference takes one) or on
    # `workers` threads (numpy/scipy release the GIL in the bulk work)
    args = [(spec, curriculum, seed, i, pool) for i in range(batch_size)]
    if executor is not None:
        items = list(executor.map(_item_draws, args))
    elif workers > 1 and batch_size > 1:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=workers) as ex:
            items = list(ex.map(_item_draws, args))
    else:
        items = [_item_draws(a) for a in args]
    scenes, params, dry, noises, offsets, sirs, snrs = (list(x) for x in zip(*items))
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    jobs, mics = scene_batch_jobs(scenes, params)
    pb = engine.prepare(fs, jobs, mics, padded=True)
    res = engine.DeviceBatch(pb, device=dev).run(include_early=True)
    B = batch_size
    M = len(scenes[0].mic_positions)
    stride = int(pb.jobs[0]["out_stride"])
    rir_len = pb.jobs["n2"].reshape(B, S + 1)[:, 0]
    dry_p = torch.from_numpy(np.stack(dry)).pin_memory()
    noise_p = torch.from_numpy(np.stack(noises)).pin_memory()
    out = mix_device(dry_p.to(dev, non_blocking=True), [[n_dry] * S] * B, offsets,
                     noise_p.to(dev, non_blocking=True), [n_dry] * B,
                     res.full.view(B, S + 1, M, stride), res.early.view(B, S + 1, M, stride), rir_len,
                     [x if S > 1 else [0.0] for x in sirs], snrs, sir_scope=spec.sir_scope)
    # device -> pinned host (the per-item arrays below are views into these;
    # each view keeps its pinned block alive)
    host = {k: torch.empty(out[k].shape, dtype=out[k].dtype, pin_memory=True)
            for k in ("mixture", "sources", "early", "noise")}
    for k, t in host.items():
        t.copy_(out[k], non_blocking=True)
    gains = out["gains"].cpu().numpy()  # synchronises the stream
    mix_h, src_h, early_h, noise_h = (host[k].numpy() for k in ("mixture", "sources", "early", "noise"))
    results = []
    for b in range(B):
        T = int(out["total"][b])
        md = {
            "offsets": list(offsets[b]),
            "gains": [float(g) for g in gains[b, :S]],
            "noise_gain": float(gains[b, S]),
            "sir_db": sirs[b],
            "snr_db": snrs[b],
            "overlap_ratios": [_overlap_ratio(n_dry, offsets[b][k], n_dry) for k in range(1, S)],
            "index": b,
            "seed": seed,
            "sim_seed": params[b].seed,
            "t60": params[b].t60,
            "room_dims": list(scenes[b].room_dims),
            "doas_deg": [float(np.degrees(x[1])) for x in np.atleast_2d(scenes[b].sources)],
            "distances": [float(x[0]) for x in np.atleast_2d(scenes[b].sources)],
        }
        results.append(MixtureResult(
            mixture=mix_h[b, :, :T],
            sources=[src_h[b, k, :, :T] for k in range(S)],
            early_sources=[early_h[b, k, :, :T] for k in range(S)],
            noise=noise_h[b, :, :T],
            metadata=md,
        ))
    return results
