"""Write tests/golden/* by running the UNMODIFIED reference in place.

    PYTHONPATH=/root/reference/pkg/src python tools/make_golden.py

Imports ``framrir`` from /root/reference (read-only, never copied).  The
fixtures are small (< 1 MB total) and committed; the GPU box never needs the
reference.  Cases:

* kat.json            numpy Philox/SeedSequence words, rate factors,
                      reflection coefficients and SURVEY Appendix C values.
* cfg1.npz            BASELINE config 1 (simulate_rir full + early, float32),
                      its direct indices and the reference ImageSet draws.
* cases.npz           small scenes over 8/16/22.05/44.1/48 kHz with their
                      draws and reference outputs (float32) and FP64 peaks.
* mix.npz / mix.json  framrir.mixture.spatialize_and_mix on small seeded
                      inputs (explicit and rng-drawn offsets/SIR/SNR, both
                      SIR scopes, 1-3 speakers, missing early filters, tiled
                      noise): inputs and reference outputs (float32).
* scene_kat.json      framrir.mixture.sample_scene draws.
* ism.npz / ism.json  framrir.ism.ism_rir outputs (float32) and metadata on
                      small rooms.
* decay.npz / .json   framrir.decay.schroeder_curve / measure_t60 on float32
                      rows (cfg 1 RIRs, exponential decays, edge cases).
* container.frir      a framrir.io.write_rir_container file (2 records).
* genbatch.npz/.json  framrir.mixture.generate_batch (2 items, small spec).
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
import framrir as F  # noqa: E402
from framrir.core import (  # noqa: E402
    max_reflections,
    reflection_coefficient,
    sample_image_geometry,
    sample_reflection_counts,
)

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"


def cfg1_scene():
    ctr = np.array([3.0, 2.5, 1.2])
    src = np.array([2.0, 3.5, 1.5])
    v = src - ctr
    d = float(np.linalg.norm(v))
    az = math.atan2(v[1], v[0])
    el = math.asin(v[2] / d)
    mics = F.linear_array([0.05, 0.05, 0.05])
    return F.Scene(room_dims=(6.0, 5.0, 3.0), mic_positions=mics, sources=[(d, az, el)])


def draws_of(params, scene, k):
    im = sample_image_geometry(params, scene, k)
    if params.num_images > 0:
        r = reflection_coefficient(scene.room_dims, params.t60)
        rr = max_reflections(params.t60, im.direct_distance, r, params.sound_speed)
        im = sample_reflection_counts(im, params, rr)
    return im


def kat():
    out = {"philox": [], "rate_factors": {}, "reflection": []}
    for seed, k, stage, first in [(0, 0, 0, 0), (17, 2, 1, 5), (2**63 - 5, 1, 0, 1021),
                                  (123456789012, 0, 1, 3), (91, 0, 0, 4095)]:
        g = np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, k, stage))))
        words = g.random(first + 8)[first:]
        key = np.random.SeedSequence((seed, k, stage)).generate_state(2, np.uint64)
        out["philox"].append({"seed": str(seed), "k": k, "stage": stage, "first": first,
                              "doubles": [float(x).hex() for x in words],
                              "key": [str(int(x)) for x in key]})
    for fs in (8000, 11025, 16000, 22050, 24000, 32000, 44100, 48000, 96000):
        f = F.rate_factors(fs)
        out["rate_factors"][str(fs)] = [f.r_h, f.r_l]
    for dims, t60 in [((5.0, 4.0, 3.0), 0.5), ((6.0, 5.0, 3.0), 0.5), ((8.0, 7.0, 3.5), 1.2)]:
        out["reflection"].append({"dims": dims, "t60": t60,
                                  "r": float(reflection_coefficient(dims, t60)).hex()})
    p = F.SimParams(t60=0.5, num_images=2048, seed=0)
    sc = cfg1_scene()
    im = draws_of(p, sc, 0)
    r = reflection_coefficient(sc.room_dims, 0.5)
    from framrir.params import scene_fingerprint

    def summary(params, scene):
        res = F.simulate_rir(params, scene, include_early=True)
        return [{
            "full_energy": [float(v).hex() for v in (x.full.samples ** 2).sum(axis=1)],
            "early_energy": [float(v).hex() for v in (x.early.samples ** 2).sum(axis=1)],
            "full_peak": float(np.abs(x.full.samples).max()).hex(),
            "direct": [int(v) for v in x.full.direct_path_sample],
            "shape": list(x.full.samples.shape),
            "metadata": {k: (v if not isinstance(v, float) else float(v).hex())
                         for k, v in x.full.metadata.items()},
        } for x in res]

    # binding/tests/test_binding.py:15-22 configuration
    bind_scene = F.Scene(room_dims=(5.0, 4.0, 3.0), mic_positions=F.linear_array([0.04, 0.08, 0.04]),
                         sources=[(1.5, 0.5235987755982988, 0.0)])
    out["binding"] = summary(F.SimParams(t60=0.3, num_images=256, seed=17), bind_scene)
    # CLI KAT (pkg/test_output.txt:136): simulate --t60 0.25 --images 64 --seed 11 --source 1.2,0,0
    cli_scene = F.Scene(room_dims=(5.0, 4.0, 3.0), mic_positions=F.linear_array([0.04, 0.08, 0.04]),
                        sources=[(1.2, 0.0, 0.0)])
    out["cli"] = summary(F.SimParams(t60=0.25, num_images=64, seed=11), cli_scene)
    # two sources, multi-source ordering and per-source streams
    two = F.Scene(room_dims=(6.0, 5.0, 3.0), mic_positions=F.linear_array([0.04, 0.08, 0.04]),
                  sources=[(1.0, 0.5, 0.0), (2.0, 2.0, 0.1)])
    out["two_sources"] = summary(F.SimParams(t60=0.2, num_images=512, seed=3), two)
    out["fingerprints"] = {"cfg1": scene_fingerprint(sc), "binding": scene_fingerprint(bind_scene)}
    out["cfg1"] = {
        "r": float(r).hex(),
        "rr_max": float(max_reflections(0.5, im.direct_distance, r)).hex(),
        "direct_mic_distances": [float(x).hex() for x in im.mic_distances[0]],
    }
    return out


def cfg1():
    p = F.SimParams(t60=0.5, num_images=2048, seed=0)
    sc = cfg1_scene()
    res = F.simulate_rir(p, sc, include_early=True)[0]
    im = draws_of(p, sc, 0)
    np.savez_compressed(
        OUT / "cfg1.npz",
        full=res.full.samples.astype(np.float32), early=res.early.samples.astype(np.float32),
        full_peak=np.abs(res.full.samples).max(axis=1), early_peak=np.abs(res.early.samples).max(axis=1),
        direct=res.full.direct_path_sample.astype(np.int64),
        dist=im.distances, az=im.azimuths, el=im.elevations, refl=im.reflections,
        mic_distances=im.mic_distances, mics=np.asarray(sc.mic_positions, float),
        source=np.asarray(sc.sources, float), room=np.asarray(sc.room_dims, float),
    )


CASES = [
    # fs, t60, images, seed, mics spacings, source (d, az, el), room
    (16000, 0.1, 256, 3, [0.04, 0.08, 0.04], (1.5, 0.3, 0.1), (5.0, 4.0, 3.0)),
    (16000, 0.25, 64, 11, [0.08], (1.2, 0.0, 0.0), (5.0, 4.0, 3.0)),
    (16000, 0.05, 32, 5, [0.05], (0.9, 2.0, -0.3), (4.0, 3.5, 2.8)),
    (16000, 0.15, 0, 7, [0.05, 0.05], (2.0, 1.0, 0.0), (6.0, 5.0, 3.0)),
    (8000, 0.2, 200, 13, [0.1], (1.7, 4.0, 0.2), (7.0, 6.0, 3.0)),
    (22050, 0.12, 300, 17, [0.03, 0.03], (1.1, 5.5, 0.0), (5.0, 5.0, 3.0)),
    (44100, 0.08, 400, 19, [0.02], (1.4, 0.7, 0.4), (6.0, 4.0, 3.0)),
    (48000, 0.06, 512, 23, [0.04, 0.04], (1.2, 3.3, -0.2), (9.0, 8.0, 4.0)),
    # sources a few cm from a mic: stage-1 taps before mid index 0 (head truncation)
    (16000, 0.1, 64, 4, [0.04], (0.045, 0.0, 0.0), (4.0, 3.5, 2.8)),
    (48000, 0.12, 128, 4, [0.1], (0.07, 0.0, 0.0), (4.0, 3.5, 2.8)),
    (16000, 0.05, 0, 9, [0.04], (0.03, 0.0, 0.0), (4.0, 3.5, 2.8)),
]


def cases():
    blobs = {}
    meta = []
    for ci, (fs, t60, n, seed, sp, src, room) in enumerate(CASES):
        p = F.SimParams(t60=t60, sample_rate=fs, num_images=n, seed=seed)
        sc = F.Scene(room_dims=room, mic_positions=F.linear_array(sp), sources=[src])
        res = F.simulate_rir(p, sc, include_early=True)[0]
        im = draws_of(p, sc, 0)
        pre = f"c{ci}_"
        blobs[pre + "full"] = res.full.samples.astype(np.float32)
        blobs[pre + "early"] = res.early.samples.astype(np.float32)
        blobs[pre + "peak"] = np.array([np.abs(res.full.samples).max(), np.abs(res.early.samples).max()])
        blobs[pre + "direct"] = res.full.direct_path_sample.astype(np.int64)
        blobs[pre + "dist"] = im.distances
        blobs[pre + "az"] = im.azimuths
        blobs[pre + "el"] = im.elevations
        blobs[pre + "refl"] = im.reflections
        blobs[pre + "mics"] = np.asarray(sc.mic_positions, float)
        meta.append({"fs": fs, "t60": t60, "num_images": n, "seed": seed, "spacings": sp,
                     "source": list(src), "room": list(room)})
    np.savez_compressed(OUT / "cases.npz", **blobs)
    (OUT / "cases.json").write_text(json.dumps(meta, indent=1))


def _decaying_filters(rng, m, r, fs=16000):
    t = np.arange(r) / fs
    h = rng.standard_normal((m, r)) * np.exp(-t / 0.004)[None, :]
    h[:, 0] += 1.0
    return h.astype(np.float32).astype(np.float64)  # stored as float32, exactly


def mix_cases():
    from framrir.mixture import MixtureSpec, spatialize_and_mix
    from framrir.resample import RirFilter

    specs = [
        # (seed, M, R, lengths, noise_len, offsets, sir, snr, scope, early?, overlap_ratio)
        (1, 2, 120, [900, 700], 900, [0, 250], [3.0], 15.0, "full", True, 0.5),
        (2, 2, 120, [900, 700], 900, [0, 250], [-4.0], 12.0, "overlap", True, 0.5),
        (3, 3, 100, [800], 300, [0], [], 10.0, "full", False, 0.5),
        (4, 3, 110, [700, 600, 500], 700, [0, 150, 300], [2.0, -1.0], 18.0, "full", True, 0.3),
        (5, 2, 100, [800, 800], 800, None, None, None, "full", True, 0.5),
        (6, 2, 100, [800, 600], 400, None, None, None, "overlap", True, 0.6),
    ]
    blobs, meta = {}, []
    for i, (seed, m, r, lens, nl, offs, sir, snr, scope, has_early, ovr) in enumerate(specs):
        rng = np.random.default_rng(seed)
        f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731 (stored as float32)
        srcs = [f32(rng.standard_normal(n)) for n in lens]
        noise = f32(rng.standard_normal(nl))
        rirs = []
        for k in range(len(lens) + 1):
            hf = _decaying_filters(rng, m, r)
            he = hf * (np.arange(r) < r // 4)[None, :]
            full = RirFilter(samples=hf, direct_path_sample=np.zeros(m, dtype=int), sample_rate=16000)
            early = RirFilter(samples=he, direct_path_sample=np.zeros(m, dtype=int), sample_rate=16000,
                              kind="early") if (has_early and k < len(lens)) else None
            rirs.append(F.RirResult(full=full, early=early))
        spec = MixtureSpec(n_speakers=len(lens), sir_scope=scope, min_overlap_ratio=ovr)
        draw_rng = np.random.default_rng(100 + seed)
        res = spatialize_and_mix(srcs, noise, rirs, spec, draw_rng, sir_db=sir, snr_db=snr, offsets=offs)
        pre = f"c{i}_"
        for k, s_ in enumerate(srcs):
            blobs[pre + f"src{k}"] = s_.astype(np.float32)
        blobs[pre + "noise"] = noise.astype(np.float32)
        for k, rr in enumerate(rirs):
            blobs[pre + f"rirf{k}"] = rr.full.samples.astype(np.float32)
            if rr.early is not None:
                blobs[pre + f"rire{k}"] = rr.early.samples.astype(np.float32)
        blobs[pre + "mixture"] = res.mixture.astype(np.float32)
        for k in range(len(lens)):
            blobs[pre + f"out_src{k}"] = res.sources[k].astype(np.float32)
            blobs[pre + f"out_early{k}"] = res.early_sources[k].astype(np.float32)
        blobs[pre + "out_noise"] = res.noise.astype(np.float32)
        md = res.metadata
        meta.append({"seed": seed, "M": m, "R": r, "lens": lens, "noise_len": nl, "scope": scope,
                     "has_early": has_early, "min_overlap_ratio": ovr, "draw_seed": 100 + seed,
                     "given": {"offsets": offs, "sir_db": sir, "snr_db": snr},
                     "offsets": [int(o) for o in md["offsets"]], "gains": md["gains"],
                     "noise_gain": md["noise_gain"], "sir_db": md["sir_db"], "snr_db": md["snr_db"],
                     "overlap_ratios": md["overlap_ratios"],
                     "peak": float(np.abs(res.mixture).max())})
    np.savez_compressed(OUT / "mix.npz", **blobs)
    (OUT / "mix.json").write_text(json.dumps(meta, indent=1))


def scene_kat():
    """framrir.mixture.sample_scene draws (plus a curriculum-capped one)."""
    from framrir.mixture import CurriculumState, MixtureSpec, curriculum_step, sample_scene

    out = []
    cur = curriculum_step(curriculum_step(CurriculumState()))
    for seed in range(6):
        rng = np.random.default_rng(seed)
        spec = MixtureSpec(n_speakers=1 + seed % 3)
        sc, pr = sample_scene(spec, rng, cur if seed % 2 else None)
        out.append({"seed": seed, "n_speakers": spec.n_speakers, "curriculum": bool(seed % 2),
                    "room": list(sc.room_dims), "t60": pr.t60, "sim_seed": int(pr.seed),
                    "sources": np.asarray(sc.sources).tolist(),
                    "mics": np.asarray(sc.mic_positions).tolist(), "next_u": float(rng.random())})
    return {"cases": out, "curriculum_upper_ms": [cur.upper_ms, cur.epoch]}


def ism_cases():
    """framrir.ism.ism_rir on small rooms (explicit and default orders,
    duration and reflection overrides, 16 and 48 kHz)."""
    from framrir.ism import IsmConfig, ism_rir

    specs = [
        dict(room_dims=(4.0, 3.5, 2.6), source_position=(1.2, 2.0, 1.3),
             mic_positions=[(2.5, 1.5, 1.2), (2.55, 1.5, 1.2)], t60=0.12, max_order=3),
        dict(room_dims=(3.0, 3.2, 2.5), source_position=(0.8, 1.1, 1.4),
             mic_positions=[(2.0, 2.1, 1.0), (2.0, 2.15, 1.0), (2.05, 2.1, 1.0)], t60=0.08),
        dict(room_dims=(5.0, 4.0, 3.0), source_position=(3.9, 0.7, 2.2),
             mic_positions=[(1.0, 3.0, 1.5)], t60=0.3, max_order=2, duration=0.05, reflection=0.85),
        dict(room_dims=(4.0, 3.5, 2.6), source_position=(1.2, 2.0, 1.3),
             mic_positions=[(2.5, 1.5, 1.2), (2.54, 1.5, 1.2)], t60=0.1, max_order=2, sample_rate=48000),
        dict(room_dims=(6.0, 5.0, 3.0), source_position=(2.0, 3.5, 1.5),
             mic_positions=[(2.925, 2.5, 1.2), (3.075, 2.5, 1.2)], t60=0.2, max_order=0),
    ]
    blobs, meta = {}, []
    for i, kw in enumerate(specs):
        out = ism_rir(IsmConfig(**kw))
        blobs[f"c{i}_samples"] = out.samples.astype(np.float32)
        blobs[f"c{i}_direct"] = out.direct_path_sample
        meta.append({"cfg": {k: (list(map(list, v)) if k == "mic_positions" else (list(v) if isinstance(v, tuple)
                                                                                  else v)) for k, v in kw.items()},
                     "peak": float(np.abs(out.samples).max()),
                     "metadata": {k: (float(v) if isinstance(v, (np.floating,)) else v)
                                  for k, v in out.metadata.items()}})
    np.savez_compressed(OUT / "ism.npz", **blobs)
    (OUT / "ism.json").write_text(json.dumps(meta, indent=1))


def decay_cases():
    """framrir.decay on float32-representable rows: the cfg 1 reference RIRs,
    exponential decays, leading silence, a short (NaN) tail."""
    from framrir.decay import measure_t60, schroeder_curve

    g = np.load(OUT / "cfg1.npz")
    rows = [g["full"][m].astype(np.float64) for m in range(g["full"].shape[0])]
    rows += [g["early"][0].astype(np.float64)]
    rng = np.random.default_rng(3)
    for t60 in (0.2, 0.5, 0.9):
        n = int(1.2 * t60 * 16000)
        env = 10.0 ** (-3.0 * np.arange(n) / (t60 * 16000))
        rows.append((rng.standard_normal(n) * env).astype(np.float32).astype(np.float64))
    sil = np.concatenate([np.zeros(300), rows[-1][:4000]])
    rows.append(sil)
    rows.append((rng.standard_normal(500) * 10.0 ** (-np.arange(500) / 400.0)).astype(np.float32).astype(np.float64))
    out = {"t60": []}
    blobs = {}
    for i, r in enumerate(rows):
        if i >= 5:  # rows 0-4 are cfg1.npz full[0..3], early[0]
            blobs[f"r{i}"] = r.astype(np.float32)
        out["t60"].append(measure_t60(r, 16000))
        c = schroeder_curve(r)
        idx = np.unique(np.linspace(0, len(c) - 1, 97).astype(np.int64))
        blobs[f"edc_idx{i}"] = idx
        blobs[f"edc{i}"] = c[idx]  # exact FP64 checkpoints of the normalised curve
    np.savez_compressed(OUT / "decay.npz", **blobs)
    (OUT / "decay.json").write_text(json.dumps({"t60": [None if math.isnan(x) else x for x in out["t60"]],
                                                "n": len(rows)}, indent=1))


def container_case():
    """A small container written by framrir.io.write_rir_container."""
    from framrir.io import RirRecord, write_rir_container

    rng = np.random.default_rng(9)
    recs = [RirRecord(samples=rng.standard_normal((2, 17)).astype(np.float32), sample_rate=16000, kind="full",
                      seed=123),
            RirRecord(samples=rng.standard_normal((3, 5)), sample_rate=48000, kind="early", seed=2**63 - 5)]
    write_rir_container(OUT / "container.frir", recs)


def generate_case():
    """framrir.mixture.generate_batch on a small spec (2 items)."""
    from framrir.mixture import MixtureSpec, generate_batch

    spec = MixtureSpec(num_images=64, utterance_seconds=0.15, speaker_distance=(0.5, 2.0),
                       room_length=(4.0, 6.0), room_width=(4.0, 6.0), t60_range=(0.1, 0.15))
    res = generate_batch(2, spec, seed=5)
    blobs, meta = {}, []
    for i, r in enumerate(res):
        blobs[f"i{i}_mixture"] = r.mixture
        blobs[f"i{i}_" + ("src1" if i == 0 else "early0")] = r.sources[1] if i == 0 else r.early_sources[0]
        meta.append({k: (list(map(float, v)) if isinstance(v, (list, tuple)) and k != "offsets" else
                         (int(v) if isinstance(v, (np.integer,)) else v)) for k, v in r.metadata.items()})
    np.savez_compressed(OUT / "genbatch.npz", **blobs)
    (OUT / "genbatch.json").write_text(json.dumps(meta, indent=1, default=float))


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    if "--gen-only" in sys.argv:
        generate_case()
        return
    if "--decay-only" in sys.argv:
        decay_cases()
        container_case()
        return
    if "--ism-only" in sys.argv:
        ism_cases()
        return
    if "--mix-only" in sys.argv:
        mix_cases()
        (OUT / "scene_kat.json").write_text(json.dumps(scene_kat(), indent=1))
        return
    (OUT / "kat.json").write_text(json.dumps(kat(), indent=1))
    cfg1()
    cases()
    mix_cases()
    (OUT / "scene_kat.json").write_text(json.dumps(scene_kat(), indent=1))
    ism_cases()
    decay_cases()
    container_case()
    generate_case()
    for f in sorted(OUT.iterdir()):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
