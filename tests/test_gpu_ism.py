"""GPU image-source method vs framrir.ism.ism_rir
(tests/golden/ism.*), plus the reference's oracle-equivalence property:
FRAM-RIR with zero images == order-0 ISM, bit for bit on the same chain."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5


def _cfg(m):
    from paper_2304_08052_b200.ism import IsmConfig

    kw = dict(m["cfg"])
    kw["room_dims"] = tuple(kw["room_dims"])
    kw["source_position"] = tuple(kw["source_position"])
    return IsmConfig(**kw)


@pytest.mark.parametrize("ci", range(5))
def test_matches_reference(golden, ci):
    from paper_2304_08052_b200.ism import ism_rir

    m = golden["ism_meta"][ci]
    out = ism_rir(_cfg(m))
    ref = golden["ism"][f"c{ci}_samples"]
    assert out.samples.shape == ref.shape
    assert np.abs(out.samples - ref).max() / m["peak"] < TOL
    assert np.array_equal(out.direct_path_sample, golden["ism"][f"c{ci}_direct"])
    for k, v in m["metadata"].items():
        assert out.metadata[k] == v, k
    assert out.kind == "full"


def test_batch_equals_single(golden):
    from paper_2304_08052_b200.ism import ism_batch, ism_rir

    cfgs = [_cfg(golden["ism_meta"][ci]) for ci in (0, 1, 2, 4)]  # all 16 kHz
    outs = ism_batch(cfgs)
    for c, o in zip(cfgs, outs):
        assert np.array_equal(o.samples, ism_rir(c).samples)


def test_zero_images_equals_order_zero():
    """Reference test_acceptance.py:184-212 on the GPU path: bit-exact."""
    from paper_2304_08052_b200 import Scene, SimParams, simulate_rir, source_position
    from paper_2304_08052_b200.ism import IsmConfig, ism_rir

    rng = np.random.default_rng(104)
    array = np.array([[-0.08, 0, 0], [-0.04, 0, 0], [0.04, 0, 0], [0.08, 0, 0]])
    for _ in range(8):
        room = tuple(rng.uniform([4, 4, 2.8], [10, 10, 4]))
        mics = array + np.asarray(room) / 2.0
        d0 = rng.uniform(0.4, 1.3)
        scene = Scene(room_dims=room, mic_positions=mics,
                      sources=[(d0, rng.uniform(0, 2 * np.pi), rng.uniform(-0.5, 0.5))])
        params = SimParams(t60=rng.uniform(0.15, 0.6), num_images=0, seed=int(rng.integers(2**31)))
        fram = simulate_rir(params, scene, include_early=False)[0].full
        cfg = IsmConfig(room_dims=room, source_position=tuple(source_position(scene, 0)), mic_positions=mics,
                        t60=params.t60, max_order=0)
        ism = ism_rir(cfg)
        assert np.array_equal(fram.samples, ism.samples)
        assert np.array_equal(fram.direct_path_sample, ism.direct_path_sample)


def test_dropped_arrivals_and_duration():
    """Short duration: most of the lattice lands past the train end and is dropped."""
    from oracle import framrir_port as P
    from paper_2304_08052_b200.ism import IsmConfig, enumerate_images, ism_rir

    cfg = IsmConfig(room_dims=(5.0, 4.0, 3.0), source_position=(1.0, 1.5, 1.0),
                    mic_positions=[(3.5, 2.0, 1.4), (3.6, 2.0, 1.4)], t60=0.4, max_order=4, duration=0.03)
    out = ism_rir(cfg)
    # CPU restatement: the same train through the oracle chain
    r_h, _ = P.factors(16000)
    rate = r_h * 16000
    L = int(np.ceil(0.03 * rate))
    pos, g = enumerate_images(cfg)
    mics = np.asarray(cfg.mic_positions)
    r = out.metadata["reflection_coefficient"]
    x = np.zeros((2, L))
    for m in range(2):
        d = np.sqrt(((pos - mics[m]) ** 2).sum(-1))
        q = np.ceil(d / 343.0 * rate).astype(np.int64)
        keep = q <= L - 1
        np.add.at(x[m], q[keep], r ** g[keep] / d[keep])
    ref = P.chain(x, 16000)
    assert out.samples.shape == ref.shape
    assert np.abs(out.samples - ref).max() / np.abs(ref).max() < TOL


def test_device_lattice_equals_host_lattice(golden):
    """The kernel's own lattice enumeration (job field `lattice`) renders the
    same samples, bit for bit, as the host-enumerated, culled rows."""
    from paper_2304_08052_b200.ism import ism_batch

    cfgs = [_cfg(golden["ism_meta"][ci]) for ci in (0, 1, 2, 4)]
    dev = ism_batch(cfgs, device_lattice=True)
    host = ism_batch(cfgs, device_lattice=False)
    for a, b in zip(dev, host):
        assert np.array_equal(a.samples, b.samples)
        assert np.array_equal(a.direct_path_sample, b.direct_path_sample)
        assert a.metadata == b.metadata


@pytest.mark.parametrize("fs,room,t60", [(16000, (3.2, 2.8, 2.5), 0.4), (48000, (4.0, 3.5, 2.8), 0.25)])
def test_large_lattice_segmented_matches_port(fs, room, t60):
    """Lattices large enough that every channel renders as several segments
    (K3 units joined by the seam kernel K4) and about half of the images
    arrive after the train end (the dropped-arrival bucket); vs oracle/ism_port
    (the reference's dense np.add.at + scipy chain)."""
    from oracle import ism_port as IP
    from paper_2304_08052_b200.ism import IsmConfig, ism_rir

    src = (0.9, 1.1, 1.3)
    mics = [(2.1, 1.4, 1.2), (2.15, 1.4, 1.2), (2.2, 1.45, 1.25)]
    cfg = IsmConfig(room_dims=room, source_position=src, mic_positions=mics, t60=t60, sample_rate=fs)
    n_img = (2 * cfg.resolved_max_order() + 1) ** 3
    assert n_img > 2 * 16384  # about half arrive in time: more than 16384 kept, so segmented
    out = ism_rir(cfg)
    ref, direct = IP.render(room, src, mics, t60, sample_rate=fs)
    assert out.samples.shape == ref.shape
    for m in range(len(mics)):
        assert np.abs(out.samples[m] - ref[m]).max() / np.abs(ref[m]).max() < TOL, m
    assert np.array_equal(out.direct_path_sample, direct)
