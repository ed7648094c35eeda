"""Host side of the GPU image-source method (ism.py:19-103 mirrors)."""

import math

import numpy as np
import pytest

from paper_2304_08052_b200 import ism as I


@pytest.mark.parametrize("kw,msg", [
    (dict(room_dims=(4, 3, -1)), "room_dims must be 3 positive lengths"),
    (dict(t60=0.0), "t60 must be > 0"),
    (dict(source_position=(5.0, 1.0, 1.0)), "source must lie strictly inside the room"),
    (dict(mic_positions=[(1.0, 1.0, 0.0)]), "all mics must lie strictly inside the room"),
    (dict(max_order=-1), "max_order must be >= 0"),
])
def test_config_validation(kw, msg):
    base = dict(room_dims=(4.0, 3.0, 2.5), source_position=(1.0, 1.0, 1.0), mic_positions=[(2.0, 2.0, 1.2)],
                t60=0.2)
    base.update(kw)
    with pytest.raises(ValueError, match=msg):
        I.IsmConfig(**base)


def test_resolved_order_and_duration():
    c = I.IsmConfig(room_dims=(4.0, 3.0, 2.5), source_position=(1.0, 1.0, 1.0),
                    mic_positions=[(2.0, 2.0, 1.2)], t60=0.2)
    assert c.effective_duration == 0.2
    assert c.resolved_max_order() == int(math.ceil(343.0 * 0.2 / 5.0)) + 1
    c2 = I.IsmConfig(room_dims=(4.0, 3.0, 2.5), source_position=(1.0, 1.0, 1.0),
                     mic_positions=[(2.0, 2.0, 1.2)], t60=0.2, duration=0.05, max_order=4)
    assert c2.effective_duration == 0.05 and c2.resolved_max_order() == 4


def test_reflection_coefficient_matches_reference_metadata(golden):
    for m in golden["ism_meta"]:
        cfg = m["cfg"]
        if "reflection" in cfg:
            assert m["metadata"]["reflection_coefficient"] == cfg["reflection"]
        else:
            assert I.eyring_reflection_coefficient(cfg["room_dims"], cfg["t60"]) == \
                m["metadata"]["reflection_coefficient"]


def test_lattice():
    c = I.IsmConfig(room_dims=(4.0, 3.0, 2.5), source_position=(1.0, 1.2, 0.7),
                    mic_positions=[(2.0, 2.0, 1.2)], t60=0.2, max_order=2)
    pos, g = I.enumerate_images(c)
    assert pos.shape == (125, 3) and g.shape == (125,)
    # the source itself (m = 0, 0, 0) sits in the middle with g = 0
    assert np.array_equal(pos[62], [1.0, 1.2, 0.7]) and g[62] == 0
    # odd index mirrors: m = 1 on x -> L + (L - s)
    assert pos[3 * 25 + 2 * 5 + 2][0] == 1 * 4.0 + (4.0 - 1.0)
    assert g.max() == 6 and (g == 0).sum() == 1
