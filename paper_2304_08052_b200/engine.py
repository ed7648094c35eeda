"""Device engine: job tables -> libfrir -> device tensors.

torch provides device memory and the current stream (plumbing only); all
arithmetic runs in libfrir.so (csrc/).  One call renders a whole batch of
(room, source) jobs; see DESIGN.md for the data layout.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi

_plan_lock = threading.Lock()
_plans: dict = {}


class Plan:
    """Per (sample_rate, device) filter tables resident on the GPU."""

    def __init__(self, sample_rate: int, device: int):
        self.sample_rate = int(sample_rate)
        self.device = device
        handle = ctypes.c_void_p()
        with torch.cuda.device(device):
            _abi.check(_abi.lib().frir_plan_create(self.sample_rate, ctypes.byref(handle)),
                       "frir_plan_create")
        self.handle = handle
        self.desc = _abi.FrirPlanDesc()
        _abi.check(_abi.lib().frir_plan_describe(handle, ctypes.byref(self.desc)), "frir_plan_describe")

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            if self.handle:
                _abi.lib().frir_plan_destroy(self.handle)
        except Exception:
            pass


def require_cuda() -> None:
    """The engine has no CPU path: fail loudly without a GPU or the library."""
    _abi.lib()
    if not torch.cuda.is_available():
        raise _abi.FrirLibraryError("no CUDA device: the FRAM-RIR engine runs only on the GPU")


def get_plan(sample_rate: int, device=None) -> Plan:
    require_cuda()
    dev = torch.cuda.current_device() if device is None else torch.device(device).index
    if dev is None:
        dev = torch.cuda.current_device()
    key = (int(sample_rate), dev)
    with _plan_lock:
        plan = _plans.get(key)
        if plan is None:
            plan = Plan(sample_rate, dev)
            _plans[key] = plan
    return plan


def new_jobs(n: int) -> np.ndarray:
    """Zeroed job table with the reference SimParams defaults."""
    jobs = np.zeros(n, dtype=_abi.JOB_DTYPE)
    jobs["c0"] = 343.0
    jobs["alpha"] = 0.1
    jobs["beta"] = 1.0
    jobs["perturb_lo"] = -2.0
    jobs["perturb_hi"] = 2.0
    jobs["tau"] = 0.25
    return jobs


@dataclass
class PreparedBatch:
    """Host-side job table after frir_jobs_prepare (validated, laid out)."""

    sample_rate: int
    jobs: np.ndarray
    mics: np.ndarray
    chan_job: np.ndarray
    chan_order: np.ndarray
    batch: _abi.FrirBatch
    padded: bool
    draws: tuple | None = None

    @property
    def n_jobs(self) -> int:
        return len(self.jobs)


def prepare(sample_rate: int, jobs: np.ndarray, mics: np.ndarray, padded: bool = False,
            draws=None) -> PreparedBatch:
    """Validate and lay out a job table on the host (no GPU needed)."""
    jobs = np.ascontiguousarray(jobs, dtype=_abi.JOB_DTYPE).copy()
    mics = np.ascontiguousarray(mics, dtype=np.float64).reshape(-1, 3)
    n_ch = int(jobs["n_mics"].sum()) if len(jobs) else 0
    chan_job = np.zeros(n_ch, dtype=np.int32)
    chan_order = np.zeros(n_ch, dtype=np.int32)
    batch = _abi.FrirBatch()
    _abi.check(
        _abi.lib().frir_jobs_prepare(int(sample_rate), jobs.ctypes.data, len(jobs), int(bool(padded)),
                                     ctypes.byref(batch), chan_job.ctypes.data,
                                     chan_order.ctypes.data),
        "frir_jobs_prepare",
    )
    if draws is not None:
        draws = tuple(np.ascontiguousarray(d, dtype=np.float64) for d in draws)
        if len(draws) != 4 or any(d.shape != (batch.total_images,) for d in draws):
            raise ValueError("oracle draws must be 4 arrays of total_images rows")
    return PreparedBatch(sample_rate, jobs, mics, chan_job, chan_order, batch, bool(padded), draws)


@dataclass
class BatchResult:
    """Device outputs of one batch.

    ``full``/``early`` are flat float32 tensors; channel ``m`` of job ``j`` is
    ``full[jobs['out_off'][j] + m * jobs['out_stride'][j]:][:jobs['n2'][j]]``.
    """

    prepared: PreparedBatch
    full: torch.Tensor
    early: torch.Tensor | None
    direct_index: torch.Tensor

    def job_view(self, j: int, kind: str = "full") -> torch.Tensor:
        J = self.prepared.jobs[j]
        buf = self.full if kind == "full" else self.early
        m, stride, n2, off = int(J["n_mics"]), int(J["out_stride"]), int(J["n2"]), int(J["out_off"])
        return buf[off: off + m * stride].view(m, stride)[:, :n2]


class DeviceBatch:
    """Device-resident copy of a prepared batch plus its workspace."""

    def __init__(self, pb: PreparedBatch, device=None, stream=None, workspace: bool = True):
        require_cuda()
        self.pb = pb
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index)
        self.device = dev
        self.plan = get_plan(pb.sample_rate, dev)
        u8 = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1))
        self.jobs = u8(pb.jobs).to(dev, non_blocking=False)
        self.chan_job = torch.from_numpy(pb.chan_job).to(dev)
        self.chan_order = torch.from_numpy(pb.chan_order).to(dev)
        self.mics = torch.from_numpy(pb.mics.reshape(-1)).to(dev)
        self.draws = None
        if pb.draws is not None:
            self.draws = [torch.from_numpy(d).to(dev) for d in pb.draws]
        b = _abi.FrirBatch()
        ctypes.memmove(ctypes.byref(b), ctypes.byref(pb.batch), ctypes.sizeof(b))
        b.jobs = self.jobs.data_ptr()
        b.chan_job = self.chan_job.data_ptr()
        b.chan_order = self.chan_order.data_ptr()
        b.mics = self.mics.data_ptr()
        if self.draws is not None:
            b.draw_dist, b.draw_az, b.draw_el, b.draw_refl = (d.data_ptr() for d in self.draws)
        self.batch = b
        self.workspace_bytes = int(_abi.lib().frir_workspace_size(self.plan.handle, ctypes.byref(b)))
        # workspace=False: the caller passes one to launch() (shared / double-buffered)
        self.workspace = (torch.empty(self.workspace_bytes, dtype=torch.uint8, device=dev) if workspace
                          else None)
        self._ws_done, self._ws_stream = None, None

    def alloc_outputs(self, include_early: bool = True, stream=None):
        """Output tensors, allocated (and, for padded layouts, zeroed) on
        `stream` (default: current) so they are ordered with a launch there."""
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        with torch.cuda.stream(st):
            n = int(self.batch.total_out)
            full = torch.empty(n, dtype=torch.float32, device=self.device)
            early = torch.empty(n, dtype=torch.float32, device=self.device) if include_early else None
            if self.pb.padded:
                full.zero_()
                if early is not None:
                    early.zero_()
            direct = torch.empty(int(self.batch.total_channels), dtype=torch.int32, device=self.device)
        return full, early, direct

    def launch(self, full, early, direct, stream=None, stages: int = _abi.STAGE_ALL, workspace=None) -> None:
        """Enqueue the render of the whole batch on `stream` (default: current),
        using `workspace` (uint8 device tensor >= workspace_bytes) if given."""
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        ws = self.workspace if workspace is None else workspace
        if ws is None or ws.numel() < self.workspace_bytes:
            raise ValueError(f"workspace too small: need {self.workspace_bytes} bytes")
        own = workspace is None  # the batch's own workspace may be in use on another stream
        if own and self._ws_done is not None and self._ws_stream != st:
            st.wait_event(self._ws_done)
        status = _abi.lib().frir_simulate_stages(
            self.plan.handle, ctypes.byref(self.batch), ws.data_ptr(),
            ws.numel(), full.data_ptr(), early.data_ptr() if early is not None else None,
            direct.data_ptr(), st.cuda_stream, stages,
        )
        _abi.check(status, "frir_simulate_stages")
        if own:
            if self._ws_done is None:
                self._ws_done = torch.cuda.Event()
            self._ws_done.record(st)
            self._ws_stream = st

    def run(self, include_early: bool = True, stream=None) -> BatchResult:
        full, early, direct = self.alloc_outputs(include_early, stream)
        self.launch(full, early, direct, stream)
        return BatchResult(self.pb, full, early, direct)

    def launch_count(self, include_early: bool = True) -> int:
        return int(_abi.lib().frir_launch_count(self.plan.handle, ctypes.byref(self.batch),
                                                int(include_early)))


def simulate_jobs(sample_rate: int, jobs: np.ndarray, mics: np.ndarray, include_early: bool = True,
                  draws=None, padded: bool = False, device=None) -> BatchResult:
    """Validate, upload and render a job table; returns device tensors."""
    pb = prepare(sample_rate, jobs, mics, padded=padded, draws=draws)
    return DeviceBatch(pb, device=device).run(include_early)


class HostPipeline:
    """Batched generation straight into pinned host memory (the e2e path).

    The job table is split into ``chunks`` sub-batches that are validated and
    laid out once; every ``run()`` copies the job tables host->device, renders
    chunk k on a compute stream while chunk k-1's RIRs stream device->host on a
    copy stream, and returns flat float32 host arrays (full, early) plus the
    per-channel direct indices, laid out as ``self.layout`` describes.
    """

    def __init__(self, sample_rate: int, jobs: np.ndarray, mics: np.ndarray,
                 include_early: bool = True, chunks: int = 4, device=None):
        require_cuda()
        n = len(jobs)
        chunks = max(1, min(chunks, n))
        bounds = [n * i // chunks for i in range(chunks + 1)]
        self.sample_rate = sample_rate
        self.include_early = include_early
        self.dev = torch.device("cuda", torch.cuda.current_device() if device is None
                                else torch.device(device).index)
        self.parts = []
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            pb = prepare(sample_rate, jobs[lo:hi], mics)
            db = DeviceBatch(pb, device=self.dev)
            full, early, direct = db.alloc_outputs(include_early)
            nfl = int(pb.batch.total_out)
            host = {
                "jobs": torch.empty(pb.jobs.nbytes, dtype=torch.uint8).pin_memory(),
                # the other per-chunk tables, staged pinned so every H2D is asynchronous
                "chan_job": torch.empty(len(pb.chan_job), dtype=torch.int32).pin_memory(),
                "chan_order": torch.empty(len(pb.chan_order), dtype=torch.int32).pin_memory(),
                "mics": torch.empty(pb.mics.size, dtype=torch.float64).pin_memory(),
                "full": torch.empty(nfl, dtype=torch.float32).pin_memory(),
                "early": torch.empty(nfl, dtype=torch.float32).pin_memory() if include_early else None,
                "direct": torch.empty(int(pb.batch.total_channels), dtype=torch.int32).pin_memory(),
            }
            self.parts.append((lo, hi, pb, db, (full, early, direct), host))
        self.compute = torch.cuda.Stream(self.dev)
        self.copy = torch.cuda.Stream(self.dev)
        self.jobs_src = jobs
        self.mics_src = mics

    @property
    def h2d_bytes(self) -> int:
        return sum(p[2].jobs.nbytes + p[2].chan_job.nbytes + p[2].chan_order.nbytes + p[2].mics.nbytes
                   for p in self.parts)

    @property
    def d2h_bytes(self) -> int:
        v = 2 if self.include_early else 1
        return sum(p[5]["full"].numel() * 4 * v + p[5]["direct"].numel() * 4 for p in self.parts)

    def job_view(self, j: int, kind: str = "full") -> np.ndarray:
        """(M, n2) host view of job j after run()."""
        for lo, hi, pb, _, _, host in self.parts:
            if lo <= j < hi:
                J = pb.jobs[j - lo]
                m, stride, n2, off = int(J["n_mics"]), int(J["out_stride"]), int(J["n2"]), int(J["out_off"])
                return host[kind].numpy()[off: off + m * stride].reshape(m, stride)[:, :n2]
        raise IndexError(j)

    def run(self, revalidate: bool = True):
        """One end-to-end pass; returns the list of per-chunk host buffers."""
        done = []
        for lo, hi, pb, db, (full, early, direct), host in self.parts:
            if revalidate:  # host validation + layout, as a caller with fresh rooms would do
                pb = prepare(self.sample_rate, self.jobs_src[lo:hi], self.mics_src)
            host["jobs"].numpy()[:] = pb.jobs.view(np.uint8).reshape(-1)
            host["chan_job"].numpy()[:] = pb.chan_job
            host["chan_order"].numpy()[:] = pb.chan_order
            host["mics"].numpy()[:] = pb.mics.reshape(-1)
            with torch.cuda.stream(self.compute):
                db.jobs.copy_(host["jobs"], non_blocking=True)
                db.chan_job.copy_(host["chan_job"], non_blocking=True)
                db.chan_order.copy_(host["chan_order"], non_blocking=True)
                db.mics.copy_(host["mics"], non_blocking=True)
                db.launch(full, early, direct, self.compute)
                ev = torch.cuda.Event()
                ev.record(self.compute)
            with torch.cuda.stream(self.copy):
                self.copy.wait_event(ev)
                host["full"].copy_(full, non_blocking=True)
                if early is not None:
                    host["early"].copy_(early, non_blocking=True)
                host["direct"].copy_(direct, non_blocking=True)
            done.append(host)
        self.copy.synchronize()
        self.compute.synchronize()
        return done


def split_jobs(jobs: np.ndarray, mics: np.ndarray, lo: int, hi: int):
    """Jobs [lo, hi) with only the mic rows they reference (mic_off rebased)."""
    part = np.array(jobs[lo:hi], copy=True)
    if len(part) == 0:
        return part, mics[:0]
    m0 = int(part["mic_off"].min())
    m1 = int((part["mic_off"] + part["n_mics"]).max())
    part["mic_off"] -= m0
    return part, np.ascontiguousarray(mics[m0:m1])


class HostStream:
    """Bounded-memory end-to-end generation of a large job table.

    The table is cut into parts of ``part_jobs`` jobs.  Every ``run()``
    validates each part on the host (``frir_jobs_prepare``), copies its job
    tables host->device from pinned memory, renders it on a compute stream and
    copies every RIR device->host into one of ``slots`` pinned host slots on a
    copy stream, so the copy of part k overlaps the render of part k+1.
    Before a slot is reused, ``consumer(part_index, host)`` (if given) sees the
    finished part (``host["full"]``, ``host["early"]``, ``host["direct"]`` flat
    arrays laid out as ``parts[i].jobs`` says).  This is the form a dataloader
    that keeps RIRs on the host uses for workloads larger than host or device
    memory (BASELINE config 5: 65,536 32-channel rooms, 109 GB per pass).
    """

    def __init__(self, sample_rate: int, jobs: np.ndarray, mics: np.ndarray, part_jobs: int = 1024,
                 include_early: bool = True, slots: int = 2, device=None):
        require_cuda()
        self.sample_rate = int(sample_rate)
        self.include_early = include_early
        self.dev = torch.device("cuda", torch.cuda.current_device() if device is None
                                else torch.device(device).index)
        n = len(jobs)
        part_jobs = max(1, int(part_jobs))
        self.src = [split_jobs(jobs, mics, lo, min(n, lo + part_jobs)) for lo in range(0, n, part_jobs)]
        self.parts = [prepare(self.sample_rate, j, m) for j, m in self.src]
        self.dbs = [DeviceBatch(p, device=self.dev, workspace=False) for p in self.parts]
        max_out = max(int(p.batch.total_out) for p in self.parts)
        max_ch = max(int(p.batch.total_channels) for p in self.parts)
        max_ws = max(db.workspace_bytes for db in self.dbs)
        max_jobs = max(p.jobs.nbytes for p in self.parts)
        max_mics = max(p.mics.size for p in self.parts)
        max_chj = max(len(p.chan_job) for p in self.parts)
        self.slots = []
        for _ in range(max(1, min(slots, len(self.parts)))):
            self.slots.append({
                "ws": torch.empty(max_ws, dtype=torch.uint8, device=self.dev),
                "d_full": torch.empty(max_out, dtype=torch.float32, device=self.dev),
                "d_early": torch.empty(max_out, dtype=torch.float32, device=self.dev) if include_early else None,
                "d_direct": torch.empty(max_ch, dtype=torch.int32, device=self.dev),
                "jobs": torch.empty(max_jobs, dtype=torch.uint8).pin_memory(),
                "chan_job": torch.empty(max_chj, dtype=torch.int32).pin_memory(),
                "chan_order": torch.empty(max_chj, dtype=torch.int32).pin_memory(),
                "mics": torch.empty(max_mics, dtype=torch.float64).pin_memory(),
                "full": torch.empty(max_out, dtype=torch.float32).pin_memory(),
                "early": torch.empty(max_out, dtype=torch.float32).pin_memory() if include_early else None,
                "direct": torch.empty(max_ch, dtype=torch.int32).pin_memory(),
                "done": None, "part": -1,
            })
        self.compute = torch.cuda.Stream(self.dev)
        self.copy = torch.cuda.Stream(self.dev)

    @property
    def n_jobs(self) -> int:
        return sum(len(p.jobs) for p in self.parts)

    @property
    def h2d_bytes(self) -> int:
        return sum(p.jobs.nbytes + p.chan_job.nbytes + p.chan_order.nbytes + p.mics.nbytes for p in self.parts)

    @property
    def d2h_bytes(self) -> int:
        v = 2 if self.include_early else 1
        return sum(int(p.batch.total_out) * 4 * v + int(p.batch.total_channels) * 4 for p in self.parts)

    def _retire(self, slot, consumer):
        if slot["done"] is not None:
            slot["done"].synchronize()
            if consumer is not None:
                k = slot["part"]
                nout, nch = int(self.parts[k].batch.total_out), int(self.parts[k].batch.total_channels)
                consumer(k, {"full": slot["full"].numpy()[:nout],
                             "early": slot["early"].numpy()[:nout] if slot["early"] is not None else None,
                             "direct": slot["direct"].numpy()[:nch]})
            slot["done"] = None

    def run(self, consumer=None, revalidate: bool = True) -> None:
        """One end-to-end pass over every part (see the class docstring)."""
        for k, db in enumerate(self.dbs):
            slot = self.slots[k % len(self.slots)]
            self._retire(slot, consumer)
            pb = prepare(self.sample_rate, *self.src[k]) if revalidate else self.parts[k]
            nj, nc, nm = pb.jobs.nbytes, len(pb.chan_job), pb.mics.size
            slot["jobs"].numpy()[:nj] = pb.jobs.view(np.uint8).reshape(-1)
            slot["chan_job"].numpy()[:nc] = pb.chan_job
            slot["chan_order"].numpy()[:nc] = pb.chan_order
            slot["mics"].numpy()[:nm] = pb.mics.reshape(-1)
            nout, nch = int(pb.batch.total_out), int(pb.batch.total_channels)
            with torch.cuda.stream(self.compute):
                db.jobs.copy_(slot["jobs"][:nj], non_blocking=True)
                db.chan_job.copy_(slot["chan_job"][:nc], non_blocking=True)
                db.chan_order.copy_(slot["chan_order"][:nc], non_blocking=True)
                db.mics.copy_(slot["mics"][:nm], non_blocking=True)
                db.launch(slot["d_full"], slot["d_early"], slot["d_direct"], self.compute, workspace=slot["ws"])
                ev = torch.cuda.Event()
                ev.record(self.compute)
            with torch.cuda.stream(self.copy):
                self.copy.wait_event(ev)
                slot["full"][:nout].copy_(slot["d_full"][:nout], non_blocking=True)
                if slot["early"] is not None:
                    slot["early"][:nout].copy_(slot["d_early"][:nout], non_blocking=True)
                slot["direct"][:nch].copy_(slot["d_direct"][:nch], non_blocking=True)
                done = torch.cuda.Event()
                done.record(self.copy)
            # (the slot's buffers are reused only after _retire() has waited for this copy)
            slot["done"], slot["part"] = done, k
        for slot in self.slots:
            self._retire(slot, consumer)


class CallRunner:
    """Low-latency path for one small batch per call (the drop-in
    ``simulate_rir``, called per item by reference dataloaders,
    mixture.py:342): the job tables travel in ONE pinned host→device copy, the
    outputs (full, early, direct indices) come back in ONE device→host copy,
    and the device tables, workspace and outputs are reused across calls
    (grown on demand).  One runner per (sample rate, device); a lock keeps
    concurrent callers from sharing its buffers."""

    _runners: dict = {}
    _runners_lock = threading.Lock()

    @classmethod
    def get(cls, sample_rate: int, device=None) -> "CallRunner":
        require_cuda()
        dev = torch.cuda.current_device() if device is None else torch.device(device).index
        if dev is None:
            dev = torch.cuda.current_device()
        key = (int(sample_rate), dev)
        with cls._runners_lock:
            r = cls._runners.get(key)
            if r is None:
                r = cls._runners[key] = CallRunner(int(sample_rate), dev)
        return r

    def __init__(self, sample_rate: int, device: int):
        self.sample_rate = sample_rate
        self.dev = torch.device("cuda", device)
        self.plan = get_plan(sample_rate, self.dev)
        self.lock = threading.Lock()
        self._bufs = {}

    def _buf(self, name, nbytes, pinned=False):
        b = self._bufs.get(name)
        if b is None or b.numel() < nbytes:
            n = max(int(nbytes), 1 << 16)
            b = (torch.empty(n, dtype=torch.uint8).pin_memory() if pinned
                 else torch.empty(n, dtype=torch.uint8, device=self.dev))
            self._bufs[name] = b
        return b

    def run(self, jobs: np.ndarray, mics: np.ndarray, include_early: bool = True):
        """(prepared batch, full, early or None, direct) with host numpy
        arrays laid out as ``prepared.jobs`` says (copies, safe to keep)."""
        pb = prepare(self.sample_rate, jobs, mics)
        b = _abi.FrirBatch()
        ctypes.memmove(ctypes.byref(b), ctypes.byref(pb.batch), ctypes.sizeof(b))
        parts = [pb.jobs.view(np.uint8).reshape(-1), pb.chan_job.view(np.uint8), pb.chan_order.view(np.uint8),
                 pb.mics.reshape(-1).view(np.uint8)]
        offs, n = [], 0
        for a in parts:
            offs.append(n)
            n = (n + a.nbytes + 255) & ~255
        nout, nch = int(b.total_out), int(b.total_channels)
        v = 2 if include_early else 1
        out_bytes = nout * 4 * v + nch * 4
        with self.lock, torch.cuda.device(self.dev):
            st = torch.cuda.current_stream(self.dev)
            h_in = self._buf("h_in", n, pinned=True)
            d_in = self._buf("d_in", n)
            hv = h_in.numpy()
            for a, o in zip(parts, offs):
                hv[o: o + a.nbytes] = a
            d_in[:n].copy_(h_in[:n], non_blocking=True)
            base = d_in.data_ptr()
            b.jobs, b.chan_job, b.chan_order, b.mics = (base + o for o in offs)
            need = int(_abi.lib().frir_workspace_size(self.plan.handle, ctypes.byref(b)))
            ws = self._buf("ws", need)
            d_out = self._buf("d_out", out_bytes)
            h_out = self._buf("h_out", out_bytes, pinned=True)
            o = d_out.data_ptr()
            status = _abi.lib().frir_simulate(self.plan.handle, ctypes.byref(b), ws.data_ptr(), ws.numel(), o,
                                              o + nout * 4 if include_early else None, o + nout * 4 * v,
                                              st.cuda_stream)
            _abi.check(status, "frir_simulate")
            h_out[:out_bytes].copy_(d_out[:out_bytes], non_blocking=True)
            st.synchronize()
            raw = h_out.numpy()
            full = raw[: nout * 4].view(np.float32).copy()
            early = raw[nout * 4: nout * 8].view(np.float32).copy() if include_early else None
            direct = raw[nout * 4 * v: out_bytes].view(np.int32).copy()
        return pb, full, early, direct
