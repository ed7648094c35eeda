"""CPU restatement of the reference's image-source method -- TEST
INFRASTRUCTURE ONLY (tests/ and bench_rows.py's cpu_baseline leg).

Follows /root/reference/pkg/src/framrir/ism.py: the Eyring reflection
coefficient (:64-78), the shoebox lattice (:80-104: per axis, index m maps to
m L + s for even m and m L + (L - s) for odd m, |m| reflections), and ism_rir
(:106-147): arrivals q = ceil(D / c0 * rate) past the filter end dropped,
amplitudes r**g / D scattered with np.add.at into the (M, L) high-rate train,
then the same decimation chain as the FRAM path (oracle/framrir_port.chain,
resample.py:81-136).  Pinned against framrir.ism.ism_rir by
tests/test_oracle_golden.py (tests/golden/ism.*).
"""

from __future__ import annotations

import math

import numpy as np

from .framrir_port import chain, factors


def eyring(room, t60: float) -> float:
    """ism.py:64-78: r = exp(-0.0805 V / (S T60))."""
    lx, ly, lz = (float(v) for v in room)
    ratio = (lx * ly * lz) / (2.0 * (lx * ly + lx * lz + ly * lz))
    return float(math.exp(-0.0805 * ratio / t60))


def max_order(room, c0: float, duration: float) -> int:
    """IsmConfig.resolved_max_order (ism.py:56-62) when max_order is None."""
    return int(math.ceil(c0 * duration / (2.0 * min(room)))) + 1


def lattice(room, src, order: int):
    """enumerate_images (ism.py:80-104): positions ((2K+1)^3, 3), counts."""
    dims = np.asarray(room, dtype=float)
    s = np.asarray(src, dtype=float)
    m = np.arange(-order, order + 1)
    axis = [np.where(m % 2 == 0, m * dims[k] + s[k], m * dims[k] + (dims[k] - s[k])) for k in range(3)]
    g = np.abs(m)
    px, py, pz = np.meshgrid(axis[0], axis[1], axis[2], indexing="ij")
    pos = np.stack([px.ravel(), py.ravel(), pz.ravel()], axis=1)
    cnt = (g[:, None, None] + g[None, :, None] + g[None, None, :]).ravel()
    return pos, cnt


def render(room, src, mics, t60: float, sample_rate: int = 16000, order: int | None = None,
           duration: float | None = None, c0: float = 343.0, reflection: float | None = None):
    """ism_rir (ism.py:106-147): (samples (M, n2), direct_path_sample (M,))."""
    r_h, _ = factors(sample_rate)
    rate = r_h * sample_rate
    dur = t60 if duration is None else duration
    L = math.ceil(dur * rate)
    r = eyring(room, t60) if reflection is None else reflection
    if not 0.0 < r < 1.0:
        raise ValueError(f"reflection coefficient must be in (0, 1), got {r}")
    k = max_order(room, c0, dur) if order is None else order
    pos, cnt = lattice(room, src, k)
    mics = np.atleast_2d(np.asarray(mics, dtype=float))
    dist = np.sqrt(((pos[:, None, :] - mics[None, :, :]) ** 2).sum(-1))
    sd = np.sqrt(((np.asarray(src, dtype=float)[None, None, :] - mics[None, :, :]) ** 2).sum(-1))[0]
    x = np.zeros((mics.shape[0], L))
    q0 = np.zeros(mics.shape[0], dtype=np.int64)
    for m in range(mics.shape[0]):
        q = np.ceil(dist[:, m] / c0 * rate).astype(np.int64)
        keep = q <= L - 1
        np.add.at(x[m], q[keep], r ** cnt[keep] / dist[keep, m])
        q0[m] = min(int(np.ceil(sd[m] / c0 * rate)), L - 1)
    full = chain(x, sample_rate)
    direct = np.clip(np.round(q0 / r_h).astype(np.int64), 0, full.shape[1] - 1)
    return full, direct
