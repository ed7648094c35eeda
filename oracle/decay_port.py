"""CPU restatement of the reference's decay measurement -- TEST
INFRASTRUCTURE ONLY (tests/ and bench_rows.py's cpu_baseline leg).

Follows /root/reference/pkg/src/framrir/decay.py: schroeder_curve (:8-17,
backward-integrated squared response normalised to its first sample, numpy's
cumsum of the reversed squares) and measure_t60 (:20-49, first crossing of
`drop` dB below the level at the direct arrival, the depth adapting to the
curve's floor, scaled by 60 / drop; NaN below min_drop dB of range).  Pinned
against framrir.decay by tests/test_oracle_golden.py (tests/golden/decay.*).
"""

from __future__ import annotations

import numpy as np


def schroeder(h) -> np.ndarray:
    h = np.asarray(h, dtype=float)
    if h.ndim != 1 or h.size == 0:
        raise ValueError("expected a non-empty single-channel impulse response")
    edc = np.cumsum(h[::-1] ** 2)[::-1]
    if edc[0] <= 0:
        raise ValueError("impulse response has no energy")
    return edc / edc[0]


def t60(h, sample_rate: int, max_drop: float = 55.0, floor_margin: float = 5.0, min_drop: float = 25.0) -> float:
    h = np.asarray(h, dtype=float)
    db = 10.0 * np.log10(np.maximum(schroeder(h), 1e-300))
    direct = int(np.argmax(np.abs(h) >= 0.5 * np.abs(h).max()))
    rel = db[direct:] - db[direct]
    drop = min(max_drop, -float(rel.min()) - floor_margin)
    if drop < min_drop:
        return float("nan")
    crossing = int(np.argmax(rel <= -drop))
    return crossing / float(sample_rate) * (60.0 / drop)
