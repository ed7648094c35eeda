"""The reference's stage functions (framrir/__init__.py:15-28) on the device,
against the oracle port of the reference (oracle/framrir_port.py), which is
pinned to the unmodified reference by tests/test_oracle_golden.py.

Tolerances: FP64 stage values within a few ulp of numpy (CUDA cbrt / pow /
sincos are <= 2 ulp), integer delays exact, the dense train equal to
np.add.at's; filters from downsample_highpass_downsample within 1e-5 of peak
(FP32 output), direct indices exact.
"""

import numpy as np
import pytest
import torch

import paper_2304_08052_b200 as F
from oracle import framrir_port as P

pytestmark = pytest.mark.gpu
TOL = 1e-5

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _scene():
    return F.Scene(room_dims=(6.0, 5.0, 3.0), mic_positions=F.linear_array([0.05, 0.05, 0.05]),
                   sources=[(1.4456832294801, 2.356194490192345, 0.20903329903452), (2.0, -0.5, 0.1)])


def _rel(a, b):
    return float(np.abs(np.asarray(a, float) - b).max() / np.abs(b).max())


def test_elementwise_stages_match_numpy():
    rng = np.random.default_rng(3)
    got = F.quadratic_ratio_sample(np.random.default_rng(11), 5000, 0.1, 1.0)
    u = np.random.default_rng(11).random(5000)
    ref = np.cbrt(0.1**3 + (1.0 - u) * (1.0**3 - 0.1**3))
    assert got.shape == (5000,) and np.allclose(got, ref, rtol=4e-16, atol=0)
    x = rng.uniform(0.1, 1.0, (7, 9))
    got = F.rescale_distance_ratio(x, 0.1, 1.0, 120.0)
    ref = 1.0 + (0.1 / (1.0 - 0.1)) * (x / 0.1 - 1.0) * (120.0 - 1.0)
    assert got.shape == x.shape and np.array_equal(got, ref)


@pytest.mark.parametrize("k", [0, 1])
def test_image_geometry_and_reflections_match_oracle(k):
    params = F.SimParams(t60=0.5, num_images=2048, seed=7)
    scene = _scene()
    im = F.sample_image_geometry(params, scene, k)
    job = P.jobs_from_scene(params, scene)[k]
    dr = P.draw(job)
    assert im.n_images == 2048 and im.source_index == k and im.direct_distance == scene.sources[k][0]
    assert np.array_equal(im.azimuths, dr.azimuths) and np.array_equal(im.elevations, dr.elevations)
    assert np.allclose(im.distances, dr.distances, rtol=1e-15, atol=0)
    assert im.distance_ratios[0] == 1.0 and np.all(np.isnan(im.reflections[1:])) and im.reflections[0] == 0.0
    P.positions(job, dr)
    q, amp, L, rate = P.delays_gains(job, dr)
    assert np.allclose(im.mic_distances, dr.mic_distances, rtol=1e-15, atol=0)
    r = F.reflection_coefficient(scene.room_dims, params.t60)
    rr = F.max_reflections(params.t60, im.direct_distance, r, params.sound_speed)
    F.sample_reflection_counts(im, params, rr)  # device stage-1 stream
    assert np.allclose(im.reflections, dr.reflections, rtol=1e-14, atol=0)
    with pytest.raises(ValueError, match="rr_max must be >= 1"):
        F.sample_reflection_counts(im, params, 0.5)
    # a caller-supplied rng is consumed exactly like the reference does
    im2 = F.sample_reflection_counts(F.sample_image_geometry(params, scene, k), params, rr,
                                     rng=np.random.default_rng(5))
    p = np.random.default_rng(5).uniform(params.perturb_lo, params.perturb_hi, 2048)
    g = 1.0 + (dr.distances[1:] / (params.sound_speed * params.t60)) ** 2 * (rr - 1.0) + p * im2.distance_ratios[1:] ** 0.25
    assert np.allclose(im2.reflections[1:], np.clip(g, 1.0, rr), rtol=1e-14, atol=0)


def test_train_early_window_and_chain_match_oracle():
    params = F.SimParams(t60=0.5, num_images=2048, seed=0)
    scene = _scene()
    r = F.reflection_coefficient(scene.room_dims, params.t60)
    im = F.sample_image_geometry(params, scene, 0)
    F.sample_reflection_counts(im, params, F.max_reflections(params.t60, im.direct_distance, r))
    tr = F.build_impulse_train(im, params, r)
    job = P.jobs_from_scene(params, scene)[0]
    dr = P.draw(job)
    q, amp, L, rate = P.delays_gains(job, dr)
    x = P.dense_train(q, amp, L)
    assert tr.rate == rate and tr.length == L and np.array_equal(tr.direct_index, q[0])
    assert np.array_equal(tr.channels != 0, x != 0)  # same delays, same collisions
    assert np.allclose(tr.channels, x, rtol=1e-14, atol=0)
    ear = F.early_reverb_train(tr, params)
    xe = P.early_only(x, q[0], rate)
    assert np.array_equal(ear.channels != 0, xe != 0) and np.allclose(ear.channels, xe, rtol=1e-14, atol=0)
    fac = F.rate_factors(16000)
    full = F.downsample_highpass_downsample(tr, fac, kind="full", metadata={"seed": 0})
    early = F.downsample_highpass_downsample(ear, fac, kind="early")
    ref_full, ref_early = P.chain(x, 16000), P.chain(xe, 16000)
    assert full.samples.shape == ref_full.shape and _rel(full.samples, ref_full) <= TOL
    assert _rel(early.samples, ref_early) <= TOL
    assert np.array_equal(full.direct_path_sample, np.clip(np.round(q[0] / 62).astype(np.int64), 0, 7999))
    assert full.kind == "full" and full.metadata["seed"] == 0 and full.metadata["r_h"] == 62
    # the staged chain equals simulate_rir's batched render
    res = F.simulate_rir(params, F.Scene(room_dims=scene.room_dims, mic_positions=scene.mic_positions,
                                         sources=scene.sources[:1]))[0]
    assert _rel(full.samples, res.full.samples) <= 1e-6 and _rel(early.samples, res.early.samples) <= 1e-6


def test_downsample_of_arbitrary_arrays():
    """Any (M, L) high-rate array, including negative samples and dense rows,
    through the same kernels (sign +1 minus sign -1)."""
    rng = np.random.default_rng(1)
    fac = F.rate_factors(16000)
    L = 62 * 900
    x = np.zeros((3, L))
    idx = rng.integers(0, L, 400)
    x[0, idx] = rng.standard_normal(400)          # sparse, both signs
    x[1, 5000:5600] = rng.uniform(0.0, 1e-2, 600)  # a dense positive run
    x[2, :] = 0.0
    x[2, L - 1] = 0.5                              # one arrival at the last sample
    got = F.downsample_highpass_downsample(x, fac)
    ref = P.chain(x, 16000)
    for m in range(2):
        assert _rel(got.samples[m], ref[m]) <= TOL, m
    assert np.abs(got.samples[2] - ref[2]).max() <= TOL * np.abs(ref[2]).max()
    assert np.array_equal(got.direct_path_sample, np.zeros(3, np.int64))
    with pytest.raises(ValueError, match="empty train"):
        F.downsample_highpass_downsample(np.zeros((0, 0)), fac)


def test_py_generate_batch_matches_generate_batch():
    from paper_2304_08052_b200 import binding

    cfg = {"mixture": {"n_speakers": 2, "utterance_seconds": 0.5, "t60_range": [0.2, 0.4], "num_images": 256}}
    b = binding.py_generate_batch(cfg, 3, seed=4)
    assert len(b) == 3 and all(m.dtype == np.float32 and m.flags.c_contiguous for m in b.mixtures)
    items = F.generate_batch(3, F.config_mixture_spec(cfg), seed=4)
    for i in range(3):
        assert np.array_equal(b.mixtures[i], items[i].mixture.astype(np.float32))
        assert len(b.sources[i]) == 2 and b.metadata[i]["index"] == i
    with pytest.raises(binding.BindingError):
        binding.py_generate_batch({"mixture": {"n_speakers": 0}}, 1)
    assert len(binding.py_generate_batch(cfg, 0)) == 0
