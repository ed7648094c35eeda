"""On-device scene sampler.

``DeviceSceneSampler`` draws the reference's ``sample_scene`` (mixture.py:
171-213) for a range of item indices directly on the GPU -- room, T60,
placements and simulation seed from the per-item stream
Philox(SeedSequence((seed, index))), bit-identical to numpy -- and writes
them as render jobs (libfrir ``frir_sample_scene_jobs``), so a batch of
rooms goes from two integers to device-resident RIRs with no host work per
room.  The curriculum (``CurriculumState.t60_bounds``) caps the T60 range as
in the reference.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _abi
from .rir import rate_factors

__all__ = ["DeviceSceneSampler"]

_STATUS = {
    1: "array aperture must be smaller than the smallest room dimension",
    2: "c0*t60 must exceed the direct distance",
    3: "rr_max must be >= 1 (reflection coefficient / source distance rule)",
    4: "T60 beyond the sampler's row stride",
}


class DeviceSceneSampler:
    """Samples ``MixtureSpec`` scenes on the device and renders their RIRs."""

    def __init__(self, spec, curriculum=None, device=None):
        import torch

        from . import engine
        from .scene import linear_array, max_pairwise_distance

        self.spec = spec
        self.S1 = spec.n_speakers + 1
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index)
        mics = linear_array(spec.mic_spacings)
        self.M = len(mics)
        self.center = mics.mean(axis=0)
        lo, hi = curriculum.t60_bounds if curriculum is not None else spec.t60_range
        f = rate_factors(spec.sample_rate)
        rate = f.r_h * spec.sample_rate
        d = _abi.design_describe(spec.sample_rate)
        n2_max = math.ceil(math.ceil(math.ceil(hi * rate) * d.up / d.down) / f.r_l)
        self.out_stride = (n2_max + 3) & ~3
        self.max_windows = (n2_max + 32 + 31) // 32
        s = _abi.FrirSceneSpec()
        s.room_length[:] = spec.room_length
        s.room_width[:] = spec.room_width
        s.room_height[:] = spec.room_height
        s.t60[:] = (lo, hi)
        s.distance[:] = spec.speaker_distance
        s.elevation[:] = spec.elevation_range
        s.center[:] = self.center
        s.aperture = max_pairwise_distance(mics)
        s.c0 = 343.0
        s.alpha3 = 0.1 ** 3
        s.b3a3 = 1.0 ** 3 - 0.1 ** 3
        s.n_sources = self.S1
        s.n_mics = self.M
        s.num_images = int(spec.num_images)
        s.out_stride = self.out_stride
        self.cspec = s
        self.plan = engine.get_plan(spec.sample_rate, self.device)
        self._ws, self._ws_done = None, None
        self.mics = torch.as_tensor(mics.reshape(-1), dtype=torch.float64, device=self.device)

    def jobs(self, seed: int, first: int, count: int, stream=None):
        """(jobs uint8 device tensor of count * (n_speakers + 1) frir_job rows,
        chan_job int32 device tensor).  Raises ValueError like the reference
        when a sampled scene breaks one of its rules."""
        import torch

        n = count * self.S1
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        # allocations and the status read run on `st`, ordered with the kernel
        with torch.cuda.stream(st):
            jobs = torch.empty(n * _abi.JOB_DTYPE.itemsize, dtype=torch.uint8, device=self.device)
            chan_job = torch.empty(n * self.M, dtype=torch.int32, device=self.device)
            status = torch.empty(count, dtype=torch.int32, device=self.device)
            _abi.check(_abi.lib().frir_sample_scene_jobs(self.plan.handle, ctypes.byref(self.cspec), int(seed),
                                                        int(first), int(count), jobs.data_ptr(),
                                                        chan_job.data_ptr(), status.data_ptr(), st.cuda_stream),
                       "frir_sample_scene_jobs")
            bad = torch.nonzero(status).flatten()
            if bad.numel():
                i = int(bad[0])
                raise ValueError(f"item {first + i}: {_STATUS.get(int(status[i]), 'invalid scene')}")
        return jobs, chan_job

    def render(self, seed: int, first: int, count: int, include_early: bool = True, stream=None):
        """Sample items first .. first + count - 1 and render all their RIRs in
        one launch.  Returns (full, early or None, direct_index) device
        tensors: full/early viewed as (count, n_speakers + 1, M, out_stride)
        float32 (rows past each job's n2 hold zeros), direct (count, S + 1, M)."""
        import torch

        jobs, chan_job = self.jobs(seed, first, count, stream)
        n = count * self.S1
        rows = int(self.spec.num_images) + 1
        b = _abi.FrirBatch()
        b.jobs = jobs.data_ptr()
        b.n_jobs = n
        b.total_channels = n * self.M
        b.chan_job = chan_job.data_ptr()
        b.chan_order = None
        b.mics = self.mics.data_ptr()
        b.total_images = n * rows
        b.total_items = n * rows * self.M
        b.total_out = n * self.M * self.out_stride
        b.max_rows = rows
        b.max_windows = self.max_windows
        lib = _abi.lib()
        need = int(lib.frir_workspace_size(self.plan.handle, ctypes.byref(b)))
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        with torch.cuda.stream(st):  # zero fills and outputs ordered with the render on `st`
            ws = getattr(self, "_ws", None)
            if ws is None or ws.numel() < need:
                ws = self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
            elif self._ws_done is not None:  # the reused workspace: wait for the last call's render
                st.wait_event(self._ws_done)
            full = torch.zeros(int(b.total_out), dtype=torch.float32, device=self.device)
            early = torch.zeros_like(full) if include_early else None
            direct = torch.empty(int(b.total_channels), dtype=torch.int32, device=self.device)
            _abi.check(lib.frir_simulate(self.plan.handle, ctypes.byref(b), ws.data_ptr(), ws.numel(),
                                         full.data_ptr(), early.data_ptr() if early is not None else None,
                                         direct.data_ptr(), st.cuda_stream), "frir_simulate")
            self._ws_done = torch.cuda.Event()
            self._ws_done.record(st)
            ws.record_stream(st)
        shape = (count, self.S1, self.M, self.out_stride)
        self._keep = (jobs, chan_job, ws)  # device tables stay alive until the launch is done
        return (full.view(shape), early.view(shape) if early is not None else None,
                direct.view(count, self.S1, self.M))

    def host_jobs(self, jobs_dev) -> np.ndarray:
        """The device job table as a numpy structured array (inspection, tests)."""
        return np.frombuffer(jobs_dev.cpu().numpy().tobytes(), dtype=_abi.JOB_DTYPE).copy()
