"""The render kernel's formulation, emulated in FP64 numpy from the C
library's design tables, equals the reference chain (no GPU needed).

This isolates the math of csrc/frir_kernels.cu (output-rate composite tables,
LP recursion, modal tail correction of the n1 truncation) from the CUDA
implementation, which tests/test_gpu_parity.py checks on the device.
"""

import numpy as np
import pytest

from _emulate import Tables, render_channel
from oracle import framrir_port as P


def _check(job, tol=1e-9):
    d = P.draw(job)
    q, amp, L, rate = P.delays_gains(job, d)
    full, early, _ = P.render(job, d)
    tab = Tables(job.sample_rate)
    lo, hi = -(-6 * rate // 1000), -(-50 * rate // 1000)
    for m in range(q.shape[1]):
        y = render_channel(tab, q[:, m], amp[:, m], L)
        pk = np.abs(full[m]).max()
        assert np.abs(y - full[m]).max() / pk < tol
        rel = q[:, m] - q[0, m]
        keep = (rel >= -lo) & (rel <= hi)
        ye = render_channel(tab, q[keep, m], amp[keep, m], L)
        assert np.abs(ye - early[m]).max() / np.abs(early[m]).max() < tol


@pytest.mark.parametrize("fs,t60,n,seed", [
    (16000, 0.3, 600, 1), (16000, 0.06, 300, 2), (8000, 0.25, 400, 3), (22050, 0.2, 500, 4),
    (32000, 0.15, 300, 5), (44100, 0.12, 500, 6), (48000, 0.2, 800, 7), (24000, 0.1, 200, 8),
])
def test_formulation_matches_chain(fs, t60, n, seed):
    mics = np.array([[-0.05, 0.0, 0.0], [0.05, 0.01, 0.0], [0.0, 0.07, 0.02]])
    job = P.Job(room=(6.0, 5.0, 3.0), mics=mics, center=mics.mean(axis=0),
                source=(1.3, 0.4 * seed, 0.1), t60=t60, sample_rate=fs, num_images=n, seed=seed)
    _check(job)


def test_formulation_direct_only_and_clamped_tail():
    # I = 0 (direct path only) and a far mic whose arrivals clamp at L - 1
    mics = np.array([[0.0, 0.0, 0.0], [1.5, 0.0, 0.0]])
    job = P.Job(room=(6.0, 5.0, 3.0), mics=mics, center=mics.mean(axis=0), source=(1.0, 1.0, 0.0),
                t60=0.08, num_images=0, seed=0)
    _check(job)
    job.num_images = 500
    _check(job)
