"""B200-native FRAM-RIR generator (arXiv 2304.08052), drop-in for the
reference's batched RIR hot path.

Reference-shaped API (framrir names, arguments, defaults and errors):
``SimParams``, ``Scene``, ``simulate_rir``, ``RirResult``, ``RirFilter``,
``rate_factors``, ``linear_array``, ``array_center``, ``source_position``,
``sph_to_cart``, ``reflection_coefficient``, ``max_reflections`` and the
binding's ``py_simulate_rir`` / ``BindingError``.

Batched device API: ``engine.simulate_jobs`` / ``engine.DeviceBatch`` over job
tables (see ``workloads`` for the seeded BASELINE configs).  All arithmetic
runs in the CUDA library ``lib/libfrir.so`` (sources in ``csrc/``); there is no
CPU fallback.
"""

__version__ = "0.1.0"

from .api import max_reflections, reflection_coefficient, scene_fingerprint, simulate_rir
from .binding import BindingError, py_simulate_rir
from .config import config_scene, config_sim_params, validate_config
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

__all__ = [
    "__version__", "SimParams", "Scene", "linear_array", "array_center", "source_position",
    "sph_to_cart", "distances_to_mics", "RirResult", "RirFilter", "RateFactors", "rate_factors",
    "reflection_coefficient", "max_reflections", "scene_fingerprint", "simulate_rir",
    "py_simulate_rir", "BindingError", "validate_config", "config_sim_params", "config_scene",
]
