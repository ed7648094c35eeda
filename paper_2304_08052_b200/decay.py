"""Reverberation-time measurement on the GPU.

Mirrors ``framrir.decay`` (/root/reference/pkg/src/framrir/decay.py:8-49):
``schroeder_curve`` and ``measure_t60`` with the reference's arguments,
defaults and errors, plus batched forms over many channels at once
(``schroeder_batch``, ``measure_t60_batch``) that run on device tensors --
e.g. every channel of a rendered batch -- through libfrir's frir_edc /
frir_t60 kernels.  The energy decay curve is summed in FP64 in the
reference's order, so it is bit-identical to numpy's.
"""

from __future__ import annotations

import numpy as np

from . import _abi

__all__ = ["schroeder_curve", "measure_t60", "schroeder_batch", "measure_t60_batch"]


def _torch():
    import torch

    return torch


def _rows(h, lengths, device):
    """(C, n) device rows, float32 or float64 (kept: float64 input stays FP64;
    other dtypes become float32, the renderer's type)."""
    torch = _torch()
    if not isinstance(h, torch.Tensor):
        a = np.atleast_2d(np.asarray(h))
        a = np.ascontiguousarray(a, dtype=np.float64 if a.dtype == np.float64 else np.float32)
        h = torch.as_tensor(a)
    if h.dim() == 1:
        h = h[None, :]
    dev = torch.device(device) if device is not None else (
        h.device if h.is_cuda else torch.device("cuda", torch.cuda.current_device()))
    h = h.to(dev, torch.float64 if h.dtype == torch.float64 else torch.float32)
    if h.stride(-1) != 1:
        h = h.contiguous()
    C, n = h.shape
    if lengths is None:
        lengths = np.full(C, n, dtype=np.int32)
    lens = torch.as_tensor(np.asarray(lengths, dtype=np.int32).reshape(C), device=dev)
    return h, lens, dev


def _edc(h, lens, dev):
    torch = _torch()
    C, n = h.shape
    edc = torch.empty((C, n), dtype=torch.float64, device=dev)  # frir_edc zero-fills past each length
    amax = torch.empty(C, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    fn = _abi.lib().frir_edc_f64 if h.dtype == torch.float64 else _abi.lib().frir_edc
    _abi.check(fn(h.data_ptr(), h.stride(0), lens.data_ptr(), C, edc.data_ptr(), n, amax.data_ptr(), st),
               "frir_edc")
    return edc, amax


def schroeder_batch(h, lengths=None, device=None):
    """Normalised energy decay curves of C rows (C, n) -> (C, n) FP64 device
    tensor (zeros past each row's length); rows without energy give NaN rows.
    float64 rows are processed in FP64, anything else as float32."""
    h, lens, dev = _rows(h, lengths, device)
    edc, _ = _edc(h, lens, dev)
    return edc / edc[:, :1]


def measure_t60_batch(h, sample_rate: int, lengths=None, max_drop: float = 55.0, floor_margin: float = 5.0,
                      min_drop: float = 25.0, device=None):
    """measure_t60 of every row of (C, n) float32 samples -> (C,) FP64 device
    tensor (NaN where the reference returns NaN or raises for no energy)."""
    torch = _torch()
    h, lens, dev = _rows(h, lengths, device)
    edc, amax = _edc(h, lens, dev)
    C, n = h.shape
    out = torch.empty(C, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    fn = _abi.lib().frir_t60_f64 if h.dtype == torch.float64 else _abi.lib().frir_t60
    _abi.check(fn(h.data_ptr(), h.stride(0), lens.data_ptr(), C, edc.data_ptr(), n, amax.data_ptr(),
                  float(sample_rate), float(max_drop), float(floor_margin), float(min_drop), out.data_ptr(), st),
               "frir_t60")
    return out


def _single(h):
    h = np.asarray(h, dtype=float)
    if h.ndim != 1 or h.size == 0:
        raise ValueError("expected a non-empty single-channel impulse response")
    if not np.any(h != 0):
        raise ValueError("impulse response has no energy")
    return h


def schroeder_curve(h) -> np.ndarray:
    """Backward-integrated squared response normalised to 1 at the first
    sample (decay.py:8-17), in FP64 from the float64 samples like the
    reference (bit-identical)."""
    h = _single(h)
    return schroeder_batch(h[None, :])[0].cpu().numpy()


def measure_t60(h, sample_rate: int, max_drop: float = 55.0, floor_margin: float = 5.0,
                min_drop: float = 25.0) -> float:
    """Decay time from the first crossing of the curve ``drop`` dB below its
    level at the direct path, scaled by 60/drop (decay.py:20-49)."""
    h = _single(h)
    return float(measure_t60_batch(h[None, :], sample_rate, None, max_drop, floor_margin, min_drop)[0])
