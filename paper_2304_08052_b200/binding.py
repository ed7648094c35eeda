"""Dataloader veneer mirroring ``framrir_binding``
(/root/reference/pkg/binding/src/framrir_binding/__init__.py): ``py_simulate_rir``
(:66-94), ``py_generate_batch`` and ``BindingBatch`` (:48-59, :97-124).

``py_simulate_rir`` returns host float32 arrays exactly shaped like the
reference's; ``py_simulate_rir_device`` returns the same data as CUDA tensors
without the host round trip (the form a GPU training loop wants).
"""

from __future__ import annotations

import numpy as np

from dataclasses import dataclass, field

from . import __version__ as _core_version
from .api import simulate_rir
from .config import config_curriculum, config_mixture_spec, config_scene, config_sim_params, validate_config

__version__ = "0.1.0"
__core_version__ = _core_version
__all__ = ["__version__", "__core_version__", "BindingError", "BindingBatch", "py_simulate_rir",
           "py_generate_batch"]


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


@dataclass
class BindingBatch:
    """One generated batch; every array is contiguous float32 (channels x samples)."""

    mixtures: list = field(default_factory=list)
    sources: list = field(default_factory=list)        # per item: list per speaker
    early_sources: list = field(default_factory=list)  # per item: list per speaker
    noises: list = field(default_factory=list)
    metadata: list = field(default_factory=list)

    def __len__(self) -> int:
        return len(self.mixtures)


def _as_f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def py_generate_batch(config: dict, batch_size: int, seed: int = 0, workers: int = 1) -> BindingBatch:
    """A reproducible mixture batch from a ``{"mixture": ..., "curriculum": ...}``
    mapping (framrir_binding/__init__.py:97-124): (seed, item index) fixes
    every sample for any worker count; all RIRs render in one device launch
    and the mixing runs on the device (``mixture.generate_batch``)."""
    from .mixture import generate_batch

    try:
        cfg = validate_config(dict(config))
        spec = config_mixture_spec(cfg)
        curriculum = config_curriculum(cfg)
        items = generate_batch(batch_size, spec, curriculum=curriculum, seed=seed, workers=workers)
    except (ValueError, TypeError) as exc:
        raise BindingError(str(exc)) from exc
    batch = BindingBatch()
    for item in items:
        batch.mixtures.append(_as_f32(item.mixture))
        batch.sources.append([_as_f32(s) for s in item.sources])
        batch.early_sources.append([_as_f32(s) for s in item.early_sources])
        batch.noises.append(_as_f32(item.noise))
        batch.metadata.append(dict(item.metadata))
    return batch

