"""Dataloader veneer mirroring ``framrir_binding.py_simulate_rir``
(/root/reference/pkg/binding/src/framrir_binding/__init__.py:44-94).

``py_simulate_rir`` returns host float32 arrays exactly shaped like the
reference's; ``py_simulate_rir_device`` returns the same data as CUDA tensors
without the host round trip (the form a GPU training loop wants).
"""

from __future__ import annotations

import numpy as np

from .api import simulate_rir
from .config import config_scene, config_sim_params, validate_config

__version__ = "0.1.0"


class BindingError(ValueError):
    """Any configuration or simulation error from the core."""


def py_simulate_rir(config: dict, include_early: bool = True):
    """``(full, early, metadata)`` for a ``{"sim": ..., "scene": ...}`` mapping.

    ``full``/``early``: contiguous float32 (n_sources, n_channels, n_samples);
    ``early`` is None without ``include_early``; one metadata dict per source.
    """
    try:
        cfg = validate_config(dict(config))
        results = simulate_rir(config_sim_params(cfg), config_scene(cfg), include_early=include_early)
    except (ValueError, TypeError) as exc:
        raise BindingError(str(exc)) from exc

    def stack(kind):
        return np.ascontiguousarray(np.stack([getattr(r, kind).samples for r in results]),
                                    dtype=np.float32)

    full = stack("full")
    early = stack("early") if include_early else None
    metadata = []
    for r in results:
        meta = dict(r.full.metadata)
        meta["direct_path_sample"] = [int(v) for v in r.full.direct_path_sample]
        meta["sample_rate"] = r.full.sample_rate
        metadata.append(meta)
    return full, early, metadata
