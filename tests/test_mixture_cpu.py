"""Host logic of the spatialise-and-mix drop-in (no GPU): spec validation and
the rng draws of offsets / SIR / SNR, against the reference's texts and the
golden cases' drawn values (mixture.py:38-80, :245-263)."""

import numpy as np
import pytest

from paper_2304_08052_b200 import mixture as MX


def test_spec_defaults_mirror_reference():
    s = MX.MixtureSpec()
    assert (s.n_speakers, s.sir_db, s.snr_db, s.min_overlap_ratio) == (2, (-6.0, 6.0), (10.0, 20.0), 0.5)
    assert (s.sample_rate, s.num_images, s.utterance_seconds, s.sir_scope) == (16000, 2048, 4.0, "full")


@pytest.mark.parametrize("kw,msg", [
    ({"n_speakers": 0}, "need at least one speaker"),
    ({"sir_db": (3.0, 1.0)}, "sir_db range is empty"),
    ({"t60_range": (0.7, 0.1)}, "t60_range range is empty"),
    ({"min_overlap_ratio": 1.5}, "min_overlap_ratio must be in"),
    ({"sir_scope": "partial"}, "sir_scope must be"),
])
def test_spec_validation(kw, msg):
    with pytest.raises(ValueError, match=msg):
        MX.MixtureSpec(**kw)


def test_convolve_scratch_sizes():
    """frir_mix_convolve_scratch (host-side sizing, no GPU): spectra of every
    4096-sample block of each source plus every filter partition of each row
    pair (mics 2h, 2h + 1 of each filter group), 8192 complex64 bins each, and
    the partitions' non-zero flags; y rows padded to whole blocks."""
    import ctypes

    from paper_2304_08052_b200 import _abi

    lib = _abi.lib()
    ys = ctypes.c_int64(0)
    B, S, M, R, T = 3, 2, 4, 9000, 70000
    got = lib.frir_mix_convolve_scratch(B, S, M, R, T, ctypes.byref(ys))
    nb, q, pairs = -(-T // 4096), -(-R // 4096), (2 * S + 1) * ((M + 1) // 2)
    assert ys.value == nb * 4096
    flags = (B * pairs * q * 4 + 255) // 256 * 256  # one int32 per filter partition: non-zero taps
    assert got == (B * (S + 1) * nb + B * pairs * q) * 8192 * 8 + flags
    lib.frir_mix_convolve_scratch(1, 1, 3, 1, 1, ctypes.byref(ys))
    assert ys.value == 4096
    assert lib.frir_mix_convolve_scratch(1, 0, 4, 10, 10, None) == -1
    assert lib.frir_mix_convolve_scratch(1, 1, 4, 0, 10, None) == -1


@pytest.mark.parametrize("ci", [4, 5])
def test_drawn_offsets_sir_snr_match_reference(golden, ci):
    """Same rng consumption order as the reference: offsets, then SIR, then SNR."""
    m = golden["mix_meta"][ci]
    rng = np.random.default_rng(m["draw_seed"])
    spec = MX.MixtureSpec(n_speakers=len(m["lens"]), sir_scope=m["scope"],
                          min_overlap_ratio=m["min_overlap_ratio"])
    srcs = [np.zeros(n) for n in m["lens"]]
    offs = MX._draw_offsets(srcs, spec, rng)
    sir = [float(rng.uniform(*spec.sir_db)) for _ in range(len(srcs) - 1)]
    snr = float(rng.uniform(*spec.snr_db))
    assert offs == m["offsets"] and sir == m["sir_db"] and snr == m["snr_db"]


def test_short_source_rejected_before_compute():
    rng = np.random.default_rng(8)
    spec = MX.MixtureSpec(min_overlap_ratio=0.9, utterance_seconds=1.0)
    srcs = [np.zeros(8000), np.zeros(500)]
    with pytest.raises(ValueError, match="overlap"):
        MX.spatialize_and_mix(srcs, np.zeros(8000), [None] * 3, spec, rng, sir_db=[0.0], snr_db=15.0,
                              offsets=[0, 7800])
    with pytest.raises(ValueError, match="one RIR"):
        MX.spatialize_and_mix([np.zeros(100)], np.zeros(100), [None] * 3, spec, rng)


def test_sample_scene_matches_reference():
    """Same draws, order and types as framrir.mixture.sample_scene (golden KAT)."""
    import json
    from pathlib import Path

    kat = json.loads((Path(__file__).parent / "golden" / "scene_kat.json").read_text())
    cur = MX.curriculum_step(MX.curriculum_step(MX.CurriculumState()))
    assert [cur.upper_ms, cur.epoch] == kat["curriculum_upper_ms"]
    for c in kat["cases"]:
        rng = np.random.default_rng(c["seed"])
        sc, pr = MX.sample_scene(MX.MixtureSpec(n_speakers=c["n_speakers"]), rng, cur if c["curriculum"] else None)
        assert list(sc.room_dims) == c["room"] and pr.t60 == c["t60"] and pr.seed == c["sim_seed"]
        assert np.asarray(sc.sources).tolist() == c["sources"]
        assert np.asarray(sc.mic_positions).tolist() == c["mics"]
        assert float(rng.random()) == c["next_u"]  # same number of draws consumed
