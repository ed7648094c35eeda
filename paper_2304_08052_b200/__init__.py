"""B200-native FRAM-RIR generator (arXiv 2304.08052), drop-in for the
reference's batched RIR hot path.

Reference-shaped API: every name of ``framrir.__all__``
(/root/reference/pkg/src/framrir/__init__.py:43-83) with its arguments,
defaults and errors -- ``simulate_rir`` and its stage functions
(``stages``: ``ImageSet`` ... ``downsample_highpass_downsample``), the
image-source method (``ism``), decay measurement (``decay``), the mixture
generator (``mixture``) -- plus the binding's ``py_simulate_rir`` /
``py_generate_batch`` / ``BindingBatch`` / ``BindingError``.

Batched device API: ``engine.simulate_jobs`` / ``engine.DeviceBatch`` over job
tables (see ``workloads`` for the seeded BASELINE configs).  All arithmetic
runs in the CUDA library ``lib/libfrir.so`` (sources in ``csrc/``); there is no
CPU fallback.
"""

__version__ = "0.1.0"

from .api import max_reflections, reflection_coefficient, scene_fingerprint, simulate_rir
from .binding import BindingBatch, BindingError, py_generate_batch, py_simulate_rir
from .config import config_curriculum, config_mixture_spec, config_scene, config_sim_params, validate_config
from .decay import measure_t60, schroeder_curve
from .ism import IsmConfig, enumerate_images, eyring_reflection_coefficient, ism_rir
from .mixture import (
    CurriculumState,
    MixtureResult,
    MixtureSpec,
    SyntheticPool,
    WavDirectoryPool,
    curriculum_step,
    generate_batch,
    sample_scene,
    spatialize_and_mix,
)
from .rir import RateFactors, RirFilter, RirResult, rate_factors
from .scene import (
    Scene,
    SimParams,
    array_center,
    distances_to_mics,
    linear_array,
    source_position,
    sph_to_cart,
)
from .stages import (
    HighRateTrain,
    ImageSet,
    build_impulse_train,
    downsample_highpass_downsample,
    early_reverb_train,
    quadratic_ratio_sample,
    rescale_distance_ratio,
    sample_image_geometry,
    sample_reflection_counts,
)

__all__ = [
    "__version__", "SimParams", "Scene", "linear_array", "array_center", "source_position", "sph_to_cart",
    "distances_to_mics", "ImageSet", "HighRateTrain", "RirResult", "RirFilter", "RateFactors",
    "quadratic_ratio_sample", "rescale_distance_ratio", "reflection_coefficient", "sample_image_geometry",
    "max_reflections", "sample_reflection_counts", "build_impulse_train", "early_reverb_train", "simulate_rir",
    "rate_factors", "downsample_highpass_downsample", "IsmConfig", "enumerate_images",
    "eyring_reflection_coefficient", "ism_rir", "schroeder_curve", "measure_t60", "MixtureSpec", "MixtureResult",
    "CurriculumState", "SyntheticPool", "WavDirectoryPool", "sample_scene", "spatialize_and_mix",
    "curriculum_step", "generate_batch", "scene_fingerprint", "py_simulate_rir", "py_generate_batch",
    "BindingBatch", "BindingError", "validate_config", "config_sim_params", "config_scene",
    "config_mixture_spec", "config_curriculum",
]
