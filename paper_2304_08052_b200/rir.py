"""Output containers and rate factors mirrored from the reference
(resample.py:18-71, core.py:78-83)."""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class RateFactors:
    """Integer factors between the high, mid and output rates (resample.py:18-32)."""

    r_h: int
    r_l: int
    sample_rate: int

    @property
    def high_rate(self) -> int:
        return self.r_h * self.sample_rate

    @property
    def mid_rate(self) -> int:
        return self.r_l * self.sample_rate


def rate_factors(sample_rate: int) -> RateFactors:
    """r_h = floor(1e6 / fs), r_l = floor(sqrt(r_h)) (resample.py:59-71)."""
    if sample_rate <= 0:
        raise ValueError(f"sample_rate must be > 0, got {sample_rate}")
    r_h = 1_000_000 // int(sample_rate)
    r_l = math.isqrt(r_h)
    if not (1 < r_l < r_h):
        raise ValueError(
            f"sample_rate {sample_rate} leaves no room for the two-stage "
            f"chain (r_h={r_h}, r_l={r_l})"
        )
    return RateFactors(r_h=r_h, r_l=r_l, sample_rate=int(sample_rate))


@dataclass
class RirFilter:
    """One multi-channel filter at the output rate (resample.py:35-56)."""

    samples: np.ndarray
    direct_path_sample: np.ndarray
    sample_rate: int
    kind: str = "full"
    metadata: dict = field(default_factory=dict)

    def __post_init__(self):
        self.samples = np.atleast_2d(np.asarray(self.samples))
        if not np.isfinite(self.samples).all():
            raise ValueError("RIR contains non-finite samples")

    @property
    def n_channels(self) -> int:
        return self.samples.shape[0]

    @property
    def n_samples(self) -> int:
        return self.samples.shape[1]


@dataclass
class RirResult:
    """Full filter and optional early-reverberation filter of one source."""

    full: RirFilter
    early: RirFilter | None = None
