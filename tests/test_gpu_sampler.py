"""On-device scene sampler vs the host mirror of
framrir.mixture.sample_scene (itself pinned to the reference by a KAT)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _host(spec, seed, first, count, curriculum=None):
    from paper_2304_08052_b200 import engine
    from paper_2304_08052_b200 import mixture as MX

    scenes, params = [], []
    for i in range(first, first + count):
        rng = np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, i))))
        sc, pr = MX.sample_scene(spec, rng, curriculum)
        scenes.append(sc)
        params.append(pr)
    jobs, mics = MX.scene_batch_jobs(scenes, params)
    return engine.prepare(spec.sample_rate, jobs, mics, padded=True)


@pytest.mark.parametrize("curr", [False, True])
def test_device_jobs_equal_host_draws(curr):
    from paper_2304_08052_b200 import mixture as MX
    from paper_2304_08052_b200.sampler import DeviceSceneSampler

    spec = MX.MixtureSpec(n_speakers=2, num_images=256)
    cur = MX.curriculum_step(MX.CurriculumState()) if curr else None
    smp = DeviceSceneSampler(spec, cur)
    jobs_d, chan_job = smp.jobs(seed=7, first=100, count=48)
    dj = smp.host_jobs(jobs_d)
    hj = _host(spec, 7, 100, 48, cur).jobs
    for f in ("room", "center", "d0", "az", "el", "t60", "c0", "alpha", "beta", "perturb_lo", "perturb_hi", "tau",
              "seed", "source_index", "n_images", "n_mics", "L", "n1", "n2", "e_lo", "e_hi", "key", "alpha3",
              "b3a3"):
        assert np.array_equal(dj[f], hj[f]), f
    for f in ("r", "rr_max", "log2r"):  # device exp/log10 vs glibc: within an ulp or two
        assert np.allclose(dj[f], hj[f], rtol=1e-14, atol=0), f
    assert np.array_equal(chan_job.cpu().numpy(), np.repeat(np.arange(48 * 3), 4))


def test_device_render_equals_host_prepared():
    from paper_2304_08052_b200 import engine
    from paper_2304_08052_b200 import mixture as MX
    from paper_2304_08052_b200.sampler import DeviceSceneSampler

    spec = MX.MixtureSpec(num_images=512, t60_range=(0.1, 0.4))
    smp = DeviceSceneSampler(spec)
    full, early, direct = smp.render(seed=3, first=0, count=16)
    pb = _host(spec, 3, 0, 16)
    res = engine.DeviceBatch(pb).run()
    d_host = res.direct_index.cpu().numpy()
    for j in range(16 * 3):
        b, k = divmod(j, 3)
        n2 = int(pb.jobs[j]["n2"])
        ref = res.job_view(j).cpu().numpy()
        got = full[b, k, :, :n2].cpu().numpy()
        assert np.abs(got - ref).max() <= 1e-6 * np.abs(ref).max(), j
        ref_e = res.job_view(j, "early").cpu().numpy()
        assert np.abs(early[b, k, :, :n2].cpu().numpy() - ref_e).max() <= 1e-6 * np.abs(ref_e).max(), j
        assert torch.all(full[b, k, :, n2:] == 0)
        ch = int(pb.jobs[j]["chan_off"])
        assert np.array_equal(direct[b, k].cpu().numpy(), d_host[ch: ch + 4])


def test_sampler_rules_raise():
    from paper_2304_08052_b200 import mixture as MX
    from paper_2304_08052_b200.sampler import DeviceSceneSampler

    spec = MX.MixtureSpec(mic_spacings=(1.5, 1.5), room_length=(2.6, 2.7), room_width=(2.6, 2.7),
                          room_height=(2.5, 2.6))
    with pytest.raises(ValueError, match="aperture"):
        DeviceSceneSampler(spec).jobs(seed=0, first=0, count=4)
