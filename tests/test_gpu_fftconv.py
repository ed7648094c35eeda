"""frir_mix_convolve (libfrir's partitioned overlap-save FFT convolution, the
fftconvolve of reference mixture.py:216-218) against a float64 numpy
convolution of the same placed sources and filter rows.  Shapes cover what
the golden mixes do not: filters of 1 to 5 partitions, per-item filter
lengths, an odd mic count (a noise row without a partner), no early filters,
noise tiled several times, totals that are not whole blocks.  Tolerance: 1e-5
of the largest |y| (FP32 transforms)."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5


def _placed(dry, off, ln, noise, nl, dl):
    """Sources as the kernel sees them: speaker k at its offset, the noise tiled."""
    S = len(off)
    T = max(int(o + n) for o, n in zip(off, ln))
    src = np.zeros((S + 1, T))
    for k in range(S):
        src[k, off[k]:off[k] + ln[k]] = dry[k, :ln[k]]
    reps = -(-dl // nl)
    src[S, :dl] = np.tile(noise[:nl], reps)[:dl]
    return src


def _run(B, S, M, R, rlens, offs, lens, nls, early=True, seed=0):
    from paper_2304_08052_b200 import _abi

    rng = np.random.default_rng(seed)
    N = max(int(o + n) for b in range(B) for o, n in zip(offs[b], lens[b]))
    dry = rng.standard_normal((B, S, N)).astype(np.float32)
    noise = rng.standard_normal((B, max(nls))).astype(np.float32)
    full = np.zeros((B, S + 1, M, R), dtype=np.float32)
    ear = np.zeros((B, S, M, R), dtype=np.float32)
    for b in range(B):
        full[b, :, :, :rlens[b]] = rng.standard_normal((S + 1, M, rlens[b])) * np.exp(-np.arange(rlens[b]) / 3000.0)
        ne = min(rlens[b], 700)
        ear[b, :, :, :ne] = full[b, :S, :, :ne]
    total = [max(o + n for o, n in zip(offs[b], lens[b])) + rlens[b] - 1 for b in range(B)]
    T = max(total)
    dlen = [total[b] - rlens[b] + 1 for b in range(B)]
    dev = torch.device("cuda")
    i32 = lambda a: torch.as_tensor(np.asarray(a, dtype=np.int32), device=dev)  # noqa: E731
    d_dry, d_noise = torch.as_tensor(dry, device=dev), torch.as_tensor(noise, device=dev)
    d_full = torch.as_tensor(full, device=dev)
    d_ear = torch.as_tensor(ear, device=dev) if early else None
    off_d, len_d, nl_d, dl_d, rl_d = i32(offs), i32(lens), i32(nls), i32(dlen), i32(rlens)
    lib = _abi.lib()
    ys = ctypes.c_int64(0)
    nscr = lib.frir_mix_convolve_scratch(B, S, M, R, T, ctypes.byref(ys))
    F = ys.value
    scratch = torch.empty(nscr, dtype=torch.uint8, device=dev)
    J = (2 * S + 1) * M
    y = torch.full((B, J, F), float("nan"), device=dev)

    def call(scr_bytes=nscr, y_stride=F):
        return lib.frir_mix_convolve(
            d_dry.data_ptr(), d_dry.stride(0), d_dry.stride(1), d_noise.data_ptr(), d_noise.stride(0),
            off_d.data_ptr(), len_d.data_ptr(), nl_d.data_ptr(), dl_d.data_ptr(), d_full.data_ptr(),
            d_full.stride(0), d_ear.data_ptr() if early else None, d_ear.stride(0) if early else 0,
            rl_d.data_ptr(), B, S, M, R, T, scratch.data_ptr(), scr_bytes, y.data_ptr(), y_stride,
            torch.cuda.current_stream().cuda_stream)

    _abi.check(call(), "frir_mix_convolve")
    torch.cuda.synchronize()
    got = y.cpu().numpy()
    worst = 0.0
    for b in range(B):
        src = _placed(dry[b].astype(np.float64), offs[b], lens[b], noise[b].astype(np.float64), nls[b], dlen[b])
        rows = []
        for k in range(S):
            for m in range(M):
                rows.append((k, full[b, k, m, :rlens[b]]))
        for k in range(S):
            for m in range(M):
                rows.append((k, (ear if early else full)[b, k, m, :rlens[b]]))
        for m in range(M):
            rows.append((S, full[b, S, m, :rlens[b]]))
        for j, (k, h) in enumerate(rows):
            ref = np.convolve(src[k], h.astype(np.float64))[:total[b]]
            g = got[b, j, :total[b]]
            assert np.isfinite(g).all()
            worst = max(worst, np.abs(g - ref).max() / max(np.abs(ref).max(), 1e-30))
    assert worst < TOL, worst
    return call


@pytest.mark.parametrize("case", [
    # B, S, M, R, rir lengths, offsets, dry lengths, noise lengths, early
    (2, 2, 3, 9000, [9000, 2000], [[0, 1500], [700, 0]], [[20000, 12000], [5000, 9000]], [3000, 9000], True),
    (1, 1, 1, 1, [1], [[0]], [[5000]], [5000], True),
    (1, 2, 4, 20000, [20000], [[0, 4096]], [[8192, 4000]], [1234], False),
    (3, 3, 2, 4097, [4096, 4097, 100], [[0, 10, 20], [5, 0, 9000], [0, 0, 0]],
     [[4096, 4096, 4096], [100, 200, 300], [1, 2, 3]], [4096, 50, 1], True),
])
def test_matches_float64_convolution(case):
    B, S, M, R, rl, offs, lens, nls, early = case
    _run(B, S, M, R, rl, offs, lens, nls, early)


def test_rejects_short_scratch_and_stride():
    from paper_2304_08052_b200 import _abi

    call = _run(1, 1, 2, 300, [300], [[0]], [[5000]], [5000])
    assert call(scr_bytes=1) == _abi.FRIR_EINVAL
    ys = ctypes.c_int64(0)
    _abi.lib().frir_mix_convolve_scratch(1, 1, 2, 300, 5299, ctypes.byref(ys))
    assert call(y_stride=ys.value - 1) == _abi.FRIR_EINVAL
