"""Host-side API surface mirrored from the reference (no GPU): dataclass
validation, geometry helpers, config handling, error types.  Cases follow
/root/reference/pkg/tests/test_core.py:350-393 and binding tests."""

import numpy as np
import pytest

import paper_2304_08052_b200 as F
from paper_2304_08052_b200 import _abi, api, binding

ARRAY = F.linear_array([0.04, 0.08, 0.04])


def test_linear_array_centered():
    a = F.linear_array([0.04, 0.08, 0.04])
    assert np.allclose(a[:, 0], [-0.08, -0.04, 0.04, 0.08])
    assert np.all(a[:, 1:] == 0)


def test_simparams_invariants():
    for kw in (dict(t60=0.0), dict(t60=0.5, alpha=0.5, beta=0.5), dict(t60=0.5, alpha=-0.1),
               dict(t60=0.5, beta=1.2), dict(t60=0.5, perturb_lo=1.0, perturb_hi=-1.0),
               dict(t60=0.5, tau=0.0), dict(t60=0.5, sound_speed=0.0), dict(t60=0.5, num_images=-1)):
        with pytest.raises(ValueError):
            F.SimParams(**kw)
    F.SimParams(t60=0.5, alpha=0.0)  # legal here, rejected at sampling


def test_scene_invariants():
    with pytest.raises(ValueError):
        F.Scene(room_dims=(5, 4, 0), mic_positions=ARRAY, sources=[(1, 0, 0)])
    with pytest.raises(ValueError):
        F.Scene(room_dims=(5, 4, 3), mic_positions=ARRAY, sources=[(-1, 0, 0)])
    with pytest.raises(ValueError):
        F.Scene(room_dims=(5, 4, 3), mic_positions=ARRAY, sources=[])
    with pytest.raises(ValueError, match="aperture"):
        F.Scene(room_dims=(1.0, 4, 3), mic_positions=[[-1.0, 0, 0], [1.0, 0, 0]], sources=[(0.5, 0, 0)])


def test_distant_source_warns():
    with pytest.warns(UserWarning, match="diagonal"):
        F.Scene(room_dims=(3, 3, 2.5), mic_positions=ARRAY, sources=[(6.0, 0, 0)])


def test_centroid_reference_point():
    s = F.Scene(room_dims=(5, 4, 3), mic_positions=ARRAY, sources=[(1.5, 0, 0)])
    assert np.allclose(F.array_center(s), 0)
    s2 = F.Scene(room_dims=(5, 4, 3), mic_positions=ARRAY, sources=[(1.5, 0, 0)],
                 reference_point=(0.5, 0.5, 0.0))
    assert np.array_equal(F.array_center(s2), [0.5, 0.5, 0.0])
    assert np.allclose(F.source_position(s2, 0), [2.0, 0.5, 0.0])


def test_reflection_and_rr_max():
    r = F.reflection_coefficient((5.0, 4.0, 3.0), 0.5)
    assert r == pytest.approx(0.98279, abs=1e-5)
    assert F.max_reflections(0.5, 1.5, r) == pytest.approx(124.896, abs=0.01)
    for dims, t60 in [((0, 4, 3), 0.5), ((5, 4, 3), 0.0), ((5, 4, 3), -1.0)]:
        with pytest.raises(ValueError):
            F.reflection_coefficient(dims, t60)
    for bad in (0.0, 1.0, 1.5, -0.2):
        with pytest.raises(ValueError):
            F.max_reflections(0.5, 1.5, bad)


def test_reflection_kat(golden):
    for e in golden["kat"]["reflection"]:
        assert F.reflection_coefficient(e["dims"], e["t60"]) == float.fromhex(e["r"])


def test_rate_factors():
    assert (F.rate_factors(16000).r_h, F.rate_factors(16000).r_l) == (62, 7)
    assert F.rate_factors(16000).high_rate == 992000 and F.rate_factors(16000).mid_rate == 112000
    for fs in (0, -1, 1_000_000, 400_000):
        with pytest.raises(ValueError):
            F.rate_factors(fs)


def test_fingerprint_matches_reference(golden):
    sc = F.Scene(room_dims=(5.0, 4.0, 3.0), mic_positions=ARRAY, sources=[(1.5, 0.5235987755982988, 0.0)])
    assert F.scene_fingerprint(sc) == golden["kat"]["fingerprints"]["binding"]


def test_rir_filter_rejects_nonfinite():
    with pytest.raises(ValueError, match="finite"):
        F.RirFilter(samples=np.array([[0.0, np.inf]]), direct_path_sample=np.array([0]), sample_rate=16000)
    f = F.RirFilter(samples=np.zeros((3, 100)), direct_path_sample=np.zeros(3, int), sample_rate=16000)
    assert f.n_channels == 3 and f.n_samples == 100


def test_validation_precedes_compute():
    scene = F.Scene(room_dims=(5.0, 4.0, 3.0), mic_positions=ARRAY, sources=[(1.5, 0.0, 0.0)])
    with pytest.raises(ValueError, match="direct distance"):
        F.simulate_rir(F.SimParams(t60=0.004, num_images=8), scene)
    with pytest.raises(ValueError, match="alpha"):
        F.simulate_rir(F.SimParams(t60=0.4, num_images=8, alpha=0.0), scene)
    near = F.Scene(room_dims=(5.0, 4.0, 3.0), mic_positions=ARRAY, sources=[(0.05, 0.0, 0.0)])
    with pytest.raises(ValueError, match="rr_max"):
        F.simulate_rir(F.SimParams(t60=1.5, num_images=8), near)


def test_config_validation():
    cfg = {"sim": {"t60": 0.3}, "scene": {"room_dims": [5, 4, 3], "mic_spacings": [0.04],
                                          "sources": [[1.0, 0, 0]]}}
    assert F.validate_config(cfg) is cfg
    with pytest.raises(ValueError, match="unknown config sections"):
        F.validate_config({"bogus": {}})
    with pytest.raises(ValueError, match="unknown keys"):
        F.validate_config({"sim": {"order": 4}})
    with pytest.raises(ValueError, match="must be an object"):
        F.validate_config({"sim": 3})
    sc = F.config_scene(cfg)
    assert sc.n_mics == 2


def test_binding_typed_errors():
    bad = {"sim": {"t60": 0.3, "alpha": 0.9, "beta": 0.2},
           "scene": {"room_dims": [5, 4, 3], "mic_spacings": [0.04], "sources": [[1.5, 0, 0]]}}
    with pytest.raises(binding.BindingError, match="alpha"):
        binding.py_simulate_rir(bad)
    with pytest.raises(binding.BindingError, match="unknown"):
        binding.py_simulate_rir({"sim": {"t60": 0.3, "order": 4}})


def test_product_has_no_cpu_fallback(monkeypatch):
    # the engine refuses to run without a GPU instead of computing on the host
    import torch

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    scene = F.Scene(room_dims=(5.0, 4.0, 3.0), mic_positions=ARRAY, sources=[(1.5, 0.0, 0.0)])
    with pytest.raises(_abi.FrirLibraryError):
        F.simulate_rir(F.SimParams(t60=0.3, num_images=16), scene)


def test_product_never_imports_oracle():
    import pathlib

    pkg = pathlib.Path(api.__file__).parent
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "from oracle" not in text and "import oracle" not in text, f


# The reference's public names (framrir/__init__.py:43-83, framrir_binding/__init__.py:35-42):
REFERENCE_ALL = [
    "__version__", "SimParams", "Scene", "linear_array", "array_center", "source_position", "sph_to_cart",
    "ImageSet", "HighRateTrain", "RirResult", "RirFilter", "RateFactors", "quadratic_ratio_sample",
    "rescale_distance_ratio", "reflection_coefficient", "sample_image_geometry", "max_reflections",
    "sample_reflection_counts", "build_impulse_train", "early_reverb_train", "simulate_rir", "rate_factors",
    "downsample_highpass_downsample", "IsmConfig", "enumerate_images", "eyring_reflection_coefficient", "ism_rir",
    "schroeder_curve", "measure_t60", "MixtureSpec", "MixtureResult", "CurriculumState", "SyntheticPool",
    "WavDirectoryPool", "sample_scene", "spatialize_and_mix", "curriculum_step", "generate_batch",
]
BINDING_ALL = ["__version__", "__core_version__", "BindingError", "BindingBatch", "py_simulate_rir",
               "py_generate_batch"]


def test_every_reference_name_is_exported():
    import paper_2304_08052_b200 as F
    from paper_2304_08052_b200 import binding

    assert [n for n in REFERENCE_ALL if not hasattr(F, n)] == []
    assert [n for n in BINDING_ALL if not hasattr(binding, n)] == []
    assert set(REFERENCE_ALL) <= set(F.__all__)


def test_stage_dataclasses_and_binding_batch():
    import numpy as np

    import paper_2304_08052_b200 as F

    im = F.ImageSet(distances=np.array([1.0, 2.0, 3.0]), azimuths=np.zeros(3), elevations=np.zeros(3),
                    distance_ratios=np.array([1.0, 2.0, 3.0]), mic_distances=np.ones((3, 2)),
                    reflections=np.zeros(3), direct_distance=1.0)
    assert im.n_images == 2 and np.array_equal(im.direct_mic_distances, [1.0, 1.0])
    tr = F.HighRateTrain(channels=np.zeros((2, 7)), direct_index=np.array([1, 2]), rate=992000)
    assert tr.length == 7
    b = F.BindingBatch()
    assert len(b) == 0 and b.metadata == []
    with pytest.raises(NotImplementedError):
        F.downsample_highpass_downsample(tr, F.rate_factors(16000), highpass_hz=100.0)


def test_config_mixture_sections():
    from paper_2304_08052_b200 import config

    cfg = config.validate_config({"mixture": {"n_speakers": 1, "t60_range": [0.2, 0.4]},
                                  "curriculum": {"epoch": 0}})
    spec = config.config_mixture_spec(cfg)
    assert spec.n_speakers == 1 and spec.t60_range == (0.2, 0.4)
    assert config.config_curriculum(cfg).epoch == 0 and config.config_curriculum({}) is None
    with pytest.raises(ValueError):
        config.validate_config({"mixture": {"bogus": 1}})
