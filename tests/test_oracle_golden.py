"""Pin the CPU oracle (oracle/framrir_port.py) to the reference's own outputs.

The fixtures come from running the unmodified reference
(tools/make_golden.py); the reference's tests hold no stored vectors, so
these plus its closed-form KATs (test_core.py) are the parity anchor.
"""

import math

import numpy as np
import pytest

from oracle import framrir_port as P


def _case_job(golden, ci):
    m = golden["cases_meta"][ci]
    mics = golden["cases"][f"c{ci}_mics"]
    return P.Job(room=tuple(m["room"]), mics=mics, center=mics.mean(axis=0),
                  source=tuple(m["source"]), t60=m["t60"], sample_rate=m["fs"],
                  num_images=m["num_images"], seed=m["seed"])


def test_philox_stream_kat(golden):
    # numpy Philox4x64-10 + SeedSequence as the reference keys them (core.py:86-91)
    for e in golden["kat"]["philox"]:
        g = P._gen(int(e["seed"]), e["k"], e["stage"])
        got = g.random(e["first"] + 8)[e["first"]:]
        assert [float(x).hex() for x in got] == e["doubles"]


def test_rate_factors_kat(golden):
    for fs, (r_h, r_l) in golden["kat"]["rate_factors"].items():
        assert P.factors(int(fs)) == (r_h, r_l)


def test_reflection_coefficient_kat(golden):
    for e in golden["kat"]["reflection"]:
        assert P.wall_reflection(e["dims"], e["t60"]) == float.fromhex(e["r"])
    # test_core.py:32-35 closed form
    assert P.wall_reflection((5.0, 4.0, 3.0), 0.5) == pytest.approx(0.98279, abs=1e-5)


def test_rr_limit_kat():
    # test_core.py:90-93
    r = P.wall_reflection((5.0, 4.0, 3.0), 0.5)
    assert P.rr_limit(0.5, 1.5, r, 343.0) == pytest.approx(124.896, abs=0.01)


def test_cfg1_matches_reference(golden):
    g = golden["cfg1"]
    job = P.Job(room=tuple(g["room"]), mics=g["mics"], center=g["mics"].mean(axis=0),
                source=tuple(g["source"][0]), t60=0.5, num_images=2048, seed=0)
    full, early, direct = P.render(job)
    assert np.array_equal(direct, g["direct"])
    for m in range(4):
        assert np.abs(full[m] - g["full"][m]).max() / g["full_peak"][m] < 1e-6
        assert np.abs(early[m] - g["early"][m]).max() / g["early_peak"][m] < 1e-6
    # direct arrivals and peak
    assert list(direct) == [65, 67, 68, 70]
    assert np.abs(full).max() == pytest.approx(1.122455176007e-02, rel=1e-10)


def test_cfg1_draws_match_reference(golden):
    g = golden["cfg1"]
    job = P.Job(room=tuple(g["room"]), mics=g["mics"], center=g["mics"].mean(axis=0),
                source=tuple(g["source"][0]), t60=0.5, num_images=2048, seed=0)
    d = P.draw(job)
    for name, key in (("distances", "dist"), ("azimuths", "az"), ("elevations", "el"),
                      ("reflections", "refl")):
        assert np.array_equal(getattr(d, name), g[key]), name
    P.delays_gains(job, d)
    assert np.array_equal(d.mic_distances, g["mic_distances"])


@pytest.mark.parametrize("ci", range(11))
def test_cases_match_reference(golden, ci):
    job = _case_job(golden, ci)
    full, early, direct = P.render(job)
    pk = golden["cases"][f"c{ci}_peak"]
    assert np.array_equal(direct, golden["cases"][f"c{ci}_direct"])
    assert np.abs(full - golden["cases"][f"c{ci}_full"]).max() / pk[0] < 1e-6
    assert np.abs(early - golden["cases"][f"c{ci}_early"]).max() / pk[1] < 1e-6


def test_early_window_offsets():
    # test_core.py:282-285
    rate = 62 * 16000
    assert -(-6 * rate // 1000) == 5952 and -(-50 * rate // 1000) == 49600


def test_index_arithmetic():
    # test_core.py:210-212
    assert math.ceil(3.43 / 343.0 * 62 * 16000) == 9920


@pytest.mark.parametrize("ci", range(6))
def test_mixture_port_matches_reference(golden, ci):
    """oracle/mixture_port.py vs framrir.mixture.spatialize_and_mix outputs."""
    from _mixcases import case
    from oracle import mixture_port as MP

    m, srcs, noise, rf, re, ref = case(golden, ci)
    mix, pf, pe, nimg, gains, gn = MP.mix(srcs, noise, rf, re, m["offsets"], m["sir_db"], m["snr_db"],
                                          m["scope"])
    pk = m["peak"]
    assert np.abs(mix - ref["mixture"]).max() / pk < 1e-6
    for k in range(len(srcs)):
        assert np.abs(pf[k] - ref["sources"][k]).max() / pk < 1e-6
        assert np.abs(pe[k] - ref["early"][k]).max() / pk < 1e-6
    assert np.abs(nimg - ref["noise"]).max() / pk < 1e-6
    assert np.allclose(gains, m["gains"], rtol=1e-12) and math.isclose(gn, m["noise_gain"], rel_tol=1e-12)


@pytest.mark.parametrize("ci", range(5))
def test_ism_port_matches_reference(golden, ci):
    """oracle/ism_port vs framrir.ism.ism_rir (tests/golden/ism.*)."""
    from oracle import ism_port as IP

    m = golden["ism_meta"][ci]
    c = m["cfg"]
    full, direct = IP.render(c["room_dims"], c["source_position"], c["mic_positions"], c["t60"],
                             sample_rate=c.get("sample_rate", 16000), order=c.get("max_order"),
                             duration=c.get("duration"), reflection=c.get("reflection"))
    ref = golden["ism"][f"c{ci}_samples"]
    assert full.shape == ref.shape
    assert np.abs(full.astype(np.float32) - ref).max() <= 1e-6 * m["peak"]
    assert np.array_equal(direct, golden["ism"][f"c{ci}_direct"])
    assert IP.eyring(c["room_dims"], c["t60"]) == m["metadata"]["reflection_coefficient"] or "reflection" in c


def test_decay_port_matches_reference(golden):
    """oracle/decay_port vs framrir.decay (tests/golden/decay.*): EDC values
    bit for bit, T60 exactly."""
    from _decaycases import rows

    from oracle import decay_port as DP

    d = golden["decay"]
    for i, r in enumerate(rows(golden)):
        c = DP.schroeder(r)
        assert np.array_equal(c[d[f"edc_idx{i}"]], d[f"edc{i}"]), i
        t = DP.t60(r, 16000)
        ref = golden["decay_meta"]["t60"][i]
        assert (ref is None and math.isnan(t)) or t == ref, i
