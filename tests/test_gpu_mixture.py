"""GPU spatialise-and-mix vs the reference's outputs
(tests/golden/mix.*, made by framrir.mixture.spatialize_and_mix) and vs the
CPU oracle port on RIRs rendered by our own simulate_rir.  Tolerance: 1e-5 of
the mixture's peak (FP32 FFT convolution against the reference's FP64)."""

import math

import numpy as np
import pytest

from _mixcases import case

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5


def _rirs(rf, re, sr=16000):
    from paper_2304_08052_b200.rir import RirFilter, RirResult

    out = []
    for k, h in enumerate(rf):
        full = RirFilter(samples=h, direct_path_sample=np.zeros(h.shape[0], dtype=np.int64), sample_rate=sr)
        e = re[k] if k < len(re) else None
        early = (RirFilter(samples=e, direct_path_sample=np.zeros(h.shape[0], dtype=np.int64),
                           sample_rate=sr, kind="early") if e is not None else None)
        out.append(RirResult(full=full, early=early))
    return out


@pytest.mark.parametrize("ci", range(6))
def test_matches_reference_goldens(golden, ci):
    from paper_2304_08052_b200 import mixture as MX

    m, srcs, noise, rf, re, ref = case(golden, ci)
    spec = MX.MixtureSpec(n_speakers=len(srcs), sir_scope=m["scope"], min_overlap_ratio=m["min_overlap_ratio"])
    rng = np.random.default_rng(m["draw_seed"])
    g = m["given"]
    res = MX.spatialize_and_mix(srcs, noise, _rirs(rf, re), spec, rng, sir_db=g["sir_db"],
                                snr_db=g["snr_db"], offsets=g["offsets"])
    pk = m["peak"]
    assert res.mixture.shape == ref["mixture"].shape
    assert np.abs(res.mixture - ref["mixture"]).max() / pk < TOL
    for k in range(len(srcs)):
        assert np.abs(res.sources[k] - ref["sources"][k]).max() / pk < TOL
        assert np.abs(res.early_sources[k] - ref["early"][k]).max() / pk < TOL
    assert np.abs(res.noise - ref["noise"]).max() / pk < TOL
    md = res.metadata
    assert md["offsets"] == m["offsets"] and md["sir_db"] == m["sir_db"] and md["snr_db"] == m["snr_db"]
    assert np.allclose(md["gains"], m["gains"], rtol=1e-5)
    assert math.isclose(md["noise_gain"], m["noise_gain"], rel_tol=1e-5)
    assert np.allclose(md["overlap_ratios"], m["overlap_ratios"])


def _identity(n, channels=2, length=16):
    h = np.zeros((channels, length))
    h[:, 0] = 1.0
    return [h] * n


def test_identity_rir_reduces_to_offset_sum():
    """Reference test_mixture.py:113-133 on the GPU path."""
    from paper_2304_08052_b200 import mixture as MX

    rng = np.random.default_rng(4)
    n = 8000
    srcs = [rng.standard_normal(n), rng.standard_normal(n)]
    noise = rng.standard_normal(n)
    spec = MX.MixtureSpec()
    res = MX.spatialize_and_mix(srcs, noise, _rirs(_identity(3), _identity(2)), spec, rng, sir_db=[0.0],
                                snr_db=100.0, offsets=[0, 1000])
    g = res.metadata["gains"][1]
    expected = np.concatenate([srcs[0], np.zeros(res.mixture.shape[1] - n)])
    shifted = np.zeros_like(expected)
    shifted[1000:1000 + n] = g * srcs[1]
    assert np.allclose(res.mixture[0], expected + shifted, atol=1e-4)


@pytest.mark.parametrize("sir", [-6.0, 0.0, 6.0])
def test_sir_and_snr_exact(sir):
    from paper_2304_08052_b200 import mixture as MX

    rng = np.random.default_rng(5)
    srcs = [rng.standard_normal(8000), rng.standard_normal(8000)]
    res = MX.spatialize_and_mix(srcs, rng.standard_normal(4000), _rirs(_identity(3), _identity(2)),
                                MX.MixtureSpec(), rng, sir_db=[sir], snr_db=12.0)
    p0 = np.mean(res.sources[0][0] ** 2)
    p1 = np.mean(res.sources[1][0] ** 2)
    pn = np.mean(res.noise[0] ** 2)
    assert 10 * np.log10(p0 / p1) == pytest.approx(sir, abs=0.01)
    assert 10 * np.log10(p0 / pn) == pytest.approx(12.0, abs=0.01)


def test_batched_equals_single_items(golden):
    """mix_device over a batch of utterances == one utterance at a time."""
    from paper_2304_08052_b200 import mixture as MX

    dev = torch.device("cuda")
    cases = [case(golden, ci) for ci in (0, 1)]  # same S, M, R
    B = len(cases)
    S = len(cases[0][1])
    M, R = cases[0][3][0].shape
    N = max(len(s) for c in cases for s in c[1])
    dry = torch.zeros((B, S, N), device=dev)
    nz = torch.zeros((B, max(len(c[2]) for c in cases)), device=dev)
    rf = torch.zeros((B, S + 1, M, R), device=dev)
    re = torch.zeros((B, S, M, R), device=dev)
    lens, nls = [], []
    for b, (m, srcs, noise, rfl, rel, ref) in enumerate(cases):
        for k, s in enumerate(srcs):
            dry[b, k, :len(s)] = torch.as_tensor(s, dtype=torch.float32)
        nz[b, :len(noise)] = torch.as_tensor(noise, dtype=torch.float32)
        for k in range(S + 1):
            rf[b, k] = torch.as_tensor(rfl[k], dtype=torch.float32)
        for k in range(S):
            re[b, k] = torch.as_tensor(rel[k], dtype=torch.float32)
        lens.append([len(s) for s in srcs])
        nls.append(len(noise))
    offs = [c[0]["offsets"] for c in cases]
    sir = [c[0]["sir_db"] for c in cases]
    snr = [c[0]["snr_db"] for c in cases]
    # scope differs between the two cases: run each scope as its own batch of two
    for scope in ("full", "overlap"):
        out = MX.mix_device(dry, lens, offs, nz, nls, rf, re, [R] * B, sir, snr, sir_scope=scope)
        for b in range(B):
            one = MX.mix_device(dry[b:b + 1], lens[b:b + 1], offs[b:b + 1], nz[b:b + 1], nls[b:b + 1],
                                rf[b:b + 1], re[b:b + 1], [R], sir[b:b + 1], snr[b:b + 1], sir_scope=scope)
            T = int(one["total"][0])
            a = out["mixture"][b, :, :T].cpu().numpy()
            c = one["mixture"][0, :, :T].cpu().numpy()
            assert np.abs(a - c).max() <= 1e-5 * np.abs(c).max()
            assert torch.all(out["mixture"][b, :, T:] == 0)


def test_with_rendered_rirs_vs_oracle_port():
    """End to end: RIRs from our simulate_rir (2 speakers + noise), mixed on the
    GPU, against the CPU port of the reference mixer on the same RIRs."""
    from oracle import mixture_port as MP
    from paper_2304_08052_b200 import SimParams, Scene, linear_array, simulate_rir
    from paper_2304_08052_b200 import mixture as MX

    scene = Scene(room_dims=(6.0, 5.0, 3.0), mic_positions=linear_array([0.04, 0.08, 0.04]),
                  sources=[(1.5, 0.3, 0.1), (2.5, 2.0, -0.2), (3.0, 4.0, 0.0)])
    rirs = simulate_rir(SimParams(t60=0.4, num_images=1024, seed=11), scene)
    rng = np.random.default_rng(12)
    srcs = [rng.standard_normal(16000), rng.standard_normal(12000)]
    noise = rng.standard_normal(16000)
    res = MX.spatialize_and_mix(srcs, noise, rirs, MX.MixtureSpec(), rng)
    md = res.metadata
    mix, pf, pe, nimg, gains, gn = MP.mix(srcs, noise, [r.full.samples for r in rirs],
                                          [r.early.samples for r in rirs[:2]], md["offsets"],
                                          md["sir_db"], md["snr_db"])
    pk = np.abs(mix).max()
    assert np.abs(res.mixture - mix).max() / pk < TOL
    assert np.abs(res.early_sources[1] - pe[1]).max() / pk < TOL
    assert np.allclose(md["gains"], gains, rtol=1e-5)


def test_generate_batch_matches_reference(golden_dir):
    """generate_batch end to end (host draws in the reference's order, RIRs
    and mixing on the device) vs framrir.mixture.generate_batch."""
    import json

    from paper_2304_08052_b200 import mixture as MX

    ref = dict(np.load(golden_dir / "genbatch.npz"))
    meta = json.loads((golden_dir / "genbatch.json").read_text())
    spec = MX.MixtureSpec(num_images=64, utterance_seconds=0.15, speaker_distance=(0.5, 2.0),
                          room_length=(4.0, 6.0), room_width=(4.0, 6.0), t60_range=(0.1, 0.15))
    res = MX.generate_batch(2, spec, seed=5)
    for i, r in enumerate(res):
        m = meta[i]
        for k in ("offsets", "sir_db", "snr_db", "index", "seed", "sim_seed", "t60", "room_dims", "doas_deg",
                  "distances", "overlap_ratios"):
            assert r.metadata[k] == m[k], k
        assert np.allclose(r.metadata["gains"], m["gains"], rtol=1e-5)
        assert r.metadata["noise_gain"] == pytest.approx(m["noise_gain"], rel=1e-5)
        pk = np.abs(ref[f"i{i}_mixture"]).max()
        assert r.mixture.dtype == np.float32 or r.mixture.shape == ref[f"i{i}_mixture"].shape
        assert np.abs(r.mixture - ref[f"i{i}_mixture"]).max() / pk < TOL
    assert np.abs(res[0].sources[1] - ref["i0_src1"]).max() / np.abs(ref["i0_mixture"]).max() < TOL
    assert np.abs(res[1].early_sources[0] - ref["i1_early0"]).max() / np.abs(ref["i1_mixture"]).max() < TOL
