"""Strict JSON-style config handling for the simulate path.

Key sets and messages follow the reference's ``framrir.io`` (io.py:110-160):
unknown sections or keys are rejected before any value is looked at; value
checks happen in the SimParams / Scene constructors.
"""

from __future__ import annotations

from .scene import Scene, SimParams, linear_array

KNOWN_KEYS = {
    "sim": frozenset({"t60", "sample_rate", "num_images", "alpha", "beta", "perturb_lo",
                      "perturb_hi", "tau", "sound_speed", "seed"}),
    "scene": frozenset({"room_dims", "mic_positions", "mic_spacings", "sources", "reference_point"}),
    # accepted for compatibility with shared configs; the mixture pipeline is out of scope
    "mixture": frozenset({"n_speakers", "sir_db", "snr_db", "min_overlap_ratio", "speaker_distance",
                          "t60_range", "room_length", "room_width", "room_height",
                          "elevation_range", "mic_spacings", "sample_rate", "num_images",
                          "utterance_seconds", "sir_scope"}),
    "curriculum": frozenset({"epoch", "lower_ms", "upper_ms", "step_ms", "max_ms"}),
}


def validate_config(cfg: dict) -> dict:
    if not isinstance(cfg, dict):
        raise ValueError("config root must be an object")
    extra = set(cfg) - set(KNOWN_KEYS)
    if extra:
        raise ValueError(f"unknown config sections: {sorted(extra)}")
    for name, allowed in KNOWN_KEYS.items():
        if name not in cfg:
            continue
        section = cfg[name]
        if not isinstance(section, dict):
            raise ValueError(f"config section {name!r} must be an object")
        bad = set(section) - allowed
        if bad:
            raise ValueError(f"unknown keys in {name!r}: {sorted(bad)}")
    return cfg


def config_sim_params(cfg: dict, **overrides) -> SimParams:
    return SimParams(**{**cfg.get("sim", {}), **overrides})


def config_scene(cfg: dict) -> Scene:
    section = dict(cfg.get("scene", {}))
    if "mic_spacings" in section:
        section["mic_positions"] = linear_array(section.pop("mic_spacings"))
    return Scene(**section)


def config_mixture_spec(cfg: dict):
    """MixtureSpec from the "mixture" section, lists as tuples (io.py:163-168)."""
    from .mixture import MixtureSpec

    section = {k: tuple(v) if isinstance(v, list) else v for k, v in cfg.get("mixture", {}).items()}
    return MixtureSpec(**section)


def config_curriculum(cfg: dict):
    """CurriculumState from the "curriculum" section, or None (io.py:171-174)."""
    if "curriculum" not in cfg:
        return None
    from .mixture import CurriculumState

    return CurriculumState(**cfg["curriculum"])

