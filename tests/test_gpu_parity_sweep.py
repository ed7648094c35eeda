"""Parity sweep at the survey's size (SURVEY §8(d) "Parity checks"): >= 64
rooms of each of BASELINE configs 2-5, every channel, full + early, native
device draws, against the oracle port of the reference (oracle/framrir_port.py,
run on all host cores).  Config 4 adds two rooms whose sources draw the maximum
image count (16,384 images = 16,385 rows > the 16,384-row segmentation
threshold), so the segmented render and its seam kernel are covered at 48 kHz.
Configs 2 and 5 also run in oracle mode: the reference's own host draws
(ImageSet rows) are uploaded and the kernels render from them.

Tolerance (north_star): max |y - y_ref| / max |y_ref| <= 1e-5 per (room,
source, variant) over all channels; direct-path indices exact.  With
FRIR_PARITY_OUT=path the per-config record (max error, mismatches, sizes) is
written there as JSON (profiles/parity_r02.json comes from this test), in the
style of the reference's recorded acceptance criteria
(/root/reference/pkg/tests/test_acceptance.py:184-212).
"""

import json
import os
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest
import torch

from oracle import framrir_port as P
from paper_2304_08052_b200 import engine, workloads

pytestmark = pytest.mark.gpu
TOL = 1e-5
ROOMS = 64
SEG_ROWS = 16384  # csrc/frir_kernels.cu kSegRows

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

_RECORD = {}


def _check(args):
    """Oracle render of one job and its errors against the GPU's output."""
    kw, full, early, direct = args
    full_o, early_o, direct_o = P.render(P.Job(**kw), include_early=True)
    out = {}
    for name, got, ref in (("full", full, full_o), ("early", early, early_o)):
        peak = float(np.abs(ref).max())
        err = np.abs(got.astype(np.float64) - ref).max(axis=1) / peak
        out[name] = float(err.max())
        out[name + "_chan"] = int(err.argmax())
    out["direct_mismatch"] = int((np.asarray(direct) != direct_o).sum())
    out["channels"] = int(full_o.shape[0])
    return out


def _job_kw(w, j):
    J = w.jobs[j]
    mics = w.mics[J["mic_off"]: J["mic_off"] + J["n_mics"]].copy()
    return dict(room=tuple(float(x) for x in J["room"]), mics=mics, center=np.array(J["center"]),
                source=(float(J["d0"]), float(J["az"]), float(J["el"])), t60=float(J["t60"]),
                sample_rate=w.sample_rate, num_images=int(J["n_images"]), seed=int(J["seed"]),
                source_index=int(J["source_index"]))


def _workload(cfg):
    w = workloads.build(cfg, ROOMS)
    if cfg == 4:  # two more rooms at the maximum image count: segmented channels
        extra = workloads.build(4, 2, start=ROOMS)
        extra.jobs["n_images"] = 16384
        extra.jobs["mic_off"] += len(w.mics)
        w = workloads.Workload("cfg4+seg", w.sample_rate, np.concatenate([w.jobs, extra.jobs]),
                               np.concatenate([w.mics, extra.mics]), ROOMS + 2)
    return w


def _draws(kw):
    """The reference's own ImageSet rows of one job (oracle: core.py:131-221)."""
    d = P.draw(P.Job(**kw))
    return d.distances, d.azimuths, d.elevations, d.reflections


@pytest.mark.parametrize("cfg,mode", [(2, "native"), (3, "native"), (4, "native"), (5, "native"),
                                      (2, "oracle"), (5, "oracle")])
def test_config_sweep_matches_oracle(cfg, mode):
    w = _workload(cfg)
    t0 = time.perf_counter()
    draws = None
    if mode == "oracle":  # the host draws uploaded as the kernels' input (oracle mode)
        with ProcessPoolExecutor(max_workers=len(os.sched_getaffinity(0))) as ex:
            rows = list(ex.map(_draws, [_job_kw(w, j) for j in range(len(w.jobs))], chunksize=4))
        draws = tuple(np.concatenate([r[k] for r in rows]) for k in range(4))
    res = engine.simulate_jobs(w.sample_rate, w.jobs, w.mics, include_early=True, draws=draws)
    full = res.full.cpu().numpy()
    early = res.early.cpu().numpy()
    direct = res.direct_index.cpu().numpy()
    pj = res.prepared.jobs
    args = []
    for j in range(len(pj)):
        m, stride, n2, off, ch = (int(pj[j][f]) for f in ("n_mics", "out_stride", "n2", "out_off", "chan_off"))
        sl = slice(off, off + m * stride)
        args.append((_job_kw(w, j), full[sl].reshape(m, stride)[:, :n2].copy(),
                     early[sl].reshape(m, stride)[:, :n2].copy(), direct[ch: ch + m].copy()))
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    with ProcessPoolExecutor(max_workers=len(os.sched_getaffinity(0))) as ex:
        stats = list(ex.map(_check, args, chunksize=1))
    worst_f = max(range(len(stats)), key=lambda j: stats[j]["full"])
    worst_e = max(range(len(stats)), key=lambda j: stats[j]["early"])
    rec = {
        "rooms": int(w.rooms), "rirs": len(stats), "channels": int(sum(s["channels"] for s in stats)),
        "max_err_full": stats[worst_f]["full"], "max_err_early": stats[worst_e]["early"],
        "worst_full": {"job": worst_f, "channel": stats[worst_f]["full_chan"]},
        "worst_early": {"job": worst_e, "channel": stats[worst_e]["early_chan"]},
        "direct_mismatches": int(sum(s["direct_mismatch"] for s in stats)),
        "max_rows": int(pj["n_images"].max()) + 1,
        "segmented_channels": int(sum(int(pj[j]["n_mics"]) for j in range(len(pj))
                                      if pj[j]["n_images"] + 1 > SEG_ROWS)),
        "tolerance": TOL,
        "mode": ("native device draws" if mode == "native" else "oracle mode: the reference's host draws")
        + " vs oracle/framrir_port.py (numpy+scipy)",
        "wall_s": time.perf_counter() - t0,
    }
    _RECORD[f"cfg{cfg}" + ("" if mode == "native" else "_oracle_mode")] = rec
    out = os.environ.get("FRIR_PARITY_OUT")
    if out:
        with open(out, "w") as f:
            json.dump(_RECORD, f, indent=1)
    assert rec["direct_mismatches"] == 0, rec
    assert rec["max_err_full"] <= TOL and rec["max_err_early"] <= TOL, rec
    if cfg == 4:
        assert rec["segmented_channels"] >= 32, rec
