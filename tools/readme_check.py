import sys
sys.path.insert(0, '/root/repo')
import paper_2304_08052_b200 as frir
params = frir.SimParams(t60=0.5, num_images=2048, seed=0)
scene = frir.Scene(room_dims=(6.0, 5.0, 3.0), mic_positions=frir.linear_array([0.05] * 3),
                   sources=[(1.4457, 2.3562, 0.2090)])
full_and_early = frir.simulate_rir(params, scene)
from paper_2304_08052_b200 import engine, workloads
w = workloads.config2(1024)
res = engine.DeviceBatch(engine.prepare(w.sample_rate, w.jobs, w.mics)).run()
from paper_2304_08052_b200 import mixture, ism, decay, container
from paper_2304_08052_b200.sampler import DeviceSceneSampler
batch = mixture.generate_batch(64, mixture.MixtureSpec(), seed=0, workers=16)
full, early, direct = DeviceSceneSampler(mixture.MixtureSpec()).render(seed=0, first=0, count=1024)
h = ism.ism_rir(ism.IsmConfig(room_dims=(5, 4, 3), source_position=(1, 1.5, 1.2),
                              mic_positions=[(3.5, 2, 1.4)], t60=0.3))
t60 = decay.measure_t60_batch(full.flatten(0, 2), 16000)
container.write_rir_container("/tmp/rirs.frir", [container.RirRecord(h.samples, 16000)])
print("README ok", len(batch), full.shape, h.samples.shape, float(t60.nanmedian()))
