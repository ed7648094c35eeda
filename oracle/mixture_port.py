"""CPU oracle for spatialise-and-mix -- TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference's consumer of the RIR path,
``framrir.mixture.spatialize_and_mix`` (/root/reference/pkg/src/framrir/
mixture.py:216-332): FP64 ``scipy.signal.fftconvolve`` per (source,
channel), placement at the offsets, reference-channel powers, SIR/SNR gains,
tiled full-utterance point noise, mixture sum.  Offsets, SIR and SNR are
taken as arguments (the reference draws them from the caller's rng before
any arithmetic, :245-263).  Pinned to the reference by
tests/test_oracle_golden.py::test_mixture_port_matches_reference with the
fixtures tools/make_golden.py writes.

Only tests/ and bench_mix.py's CPU-baseline leg may import this module.
"""

from __future__ import annotations

import numpy as np
from scipy.signal import fftconvolve


def _conv(x, rir):
    """(N,) dry signal against (M, L) filter -> (M, N + L - 1), mixture.py:216-218."""
    return fftconvolve(rir, x[None, :], axes=1)


def _power(x):
    return float(np.mean(x**2))


def mix(sources, noise, rirs_full, rirs_early, offsets, sir_db, snr_db, sir_scope="full"):
    """Returns (mixture, placed_full list, placed_early list, noise_img, gains, noise_gain).

    rirs_full: list of (M, R) arrays, one per speaker plus the noise last;
    rirs_early: list of (M, R) arrays or None per speaker (None -> full).
    """
    rir_len = rirs_full[0].shape[1]
    total = max(off + len(s) for off, s in zip(offsets, sources)) + rir_len - 1  # :272
    placed_full, placed_early = [], []
    for k, (src, off) in enumerate(zip(sources, offsets)):  # :274-287
        img = _conv(np.asarray(src, dtype=float), rirs_full[k])
        out = np.zeros((img.shape[0], total))
        out[:, off:off + img.shape[1]] = img
        placed_full.append(out)
        if rirs_early[k] is not None:
            img_e = _conv(np.asarray(src, dtype=float), rirs_early[k])
            out_e = np.zeros((img_e.shape[0], total))
            out_e[:, off:off + img_e.shape[1]] = img_e
            placed_early.append(out_e)
        else:
            placed_early.append(out.copy())
    gains = [1.0]  # :289-305
    p_ref = _power(placed_full[0][0])
    for k in range(1, len(sources)):
        if sir_scope == "overlap":
            lo = offsets[k]
            hi = min(total, offsets[k] + len(sources[k]) + rir_len - 1)
            p_int = _power(placed_full[k][0, lo:hi])
            p_tgt = _power(placed_full[0][0, lo:hi])
        else:
            p_int = _power(placed_full[k][0])
            p_tgt = p_ref
        g = np.sqrt(p_tgt / (p_int * 10.0 ** (sir_db[k - 1] / 10.0)))
        gains.append(float(g))
        placed_full[k] = placed_full[k] * g
        placed_early[k] = placed_early[k] * g
    dry_len = total - rir_len + 1  # :307-312
    reps = int(np.ceil(dry_len / len(noise)))
    noise_dry = np.tile(np.asarray(noise, dtype=float), reps)[:dry_len]
    noise_img = _conv(noise_dry, rirs_full[-1])[:, :total]
    g_noise = float(np.sqrt(p_ref / (_power(noise_img[0]) * 10.0 ** (snr_db / 10.0))))
    noise_img = noise_img * g_noise
    mixture = sum(placed_full) + noise_img
    return mixture, placed_full, placed_early, noise_img, gains, g_noise
