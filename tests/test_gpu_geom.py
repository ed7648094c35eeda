"""K1 (geom_kernel) item lists against the reference's own delay and gain
arithmetic (core.py:238-246): every (image, mic) item's integer high-rate
delay q = min(ceil(D / c0 * rate), L - 1) must be EXACT, and its FP32 gain
r**g / D within FP32 rounding.  The render's parity tests would not notice a
single image shifted by one high-rate sample (1 us at 16 kHz), so the delays
are checked here item by item, straight from the raw item list in the
workspace (stage GEOM only).  The kernel computes D from a one-step Newton
FP64 reciprocal square root and falls back to the reference's sqrt/div only
inside a guard band around the integers; this is the test that pins it.
"""

import numpy as np
import pytest
import torch

from oracle import framrir_port as P
from paper_2304_08052_b200 import _abi, engine, workloads

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

K_EXT, K_SP_BIAS = 32, 64  # csrc/frir_internal.h


def _raw_items(w):
    pb = engine.prepare(w.sample_rate, w.jobs, w.mics)
    db = engine.DeviceBatch(pb)
    full, early, direct = db.alloc_outputs(True)
    db.launch(full, early, direct, stages=1)  # K1 only: the raw (image-order) item list
    torch.cuda.synchronize()
    n = int(pb.batch.total_items)
    off = (n * 8 + 255) // 256 * 256  # carve(): sorted list, then the raw list
    raw = db.workspace[off: off + 8 * n].cpu().numpy().view(np.int32).reshape(n, 2)
    return pb, raw


@pytest.mark.parametrize("cfg,rooms", [(2, 64), (5, 24), (4, 2)])
def test_geom_item_delays_exact_and_gains(cfg, rooms):
    w = workloads.build(cfg, rooms)
    pb, raw = _raw_items(w)
    d = _abi.design_describe(w.sample_rate)
    checked = 0
    for j in range(len(pb.jobs)):
        J = pb.jobs[j]
        kw = dict(room=tuple(float(x) for x in J["room"]),
                  mics=w.mics[J["mic_off"]: J["mic_off"] + J["n_mics"]].copy(), center=np.array(J["center"]),
                  source=(float(J["d0"]), float(J["az"]), float(J["el"])), t60=float(J["t60"]),
                  sample_rate=w.sample_rate, num_images=int(J["n_images"]), seed=int(J["seed"]),
                  source_index=int(J["source_index"]))
        job = P.Job(**kw)
        q_ref, amp_ref, _, _ = P.delays_gains(job, P.draw(job))
        rows, M = int(J["n_images"]) + 1, int(J["n_mics"])
        it = raw[int(J["item_off"]): int(J["item_off"]) + rows * M].reshape(M, rows, 2)
        x = it[..., 0].astype(np.int64) & 0xFFFFFFFF
        s = (x & 0xFFFFF) - K_EXT - K_SP_BIAS
        q = d.r_h * s - d.t0 - ((x >> 20) & 0x3FF)
        bad = np.argwhere(q != q_ref.T)
        assert bad.size == 0, (j, bad[:5], q[tuple(bad[0])], q_ref.T[tuple(bad[0])])
        gain = np.abs(it[..., 1].view(np.float32)).astype(np.float64)
        np.testing.assert_allclose(gain, amp_ref.T, rtol=1e-6, atol=0)
        checked += rows * M
    assert checked == int(pb.batch.total_items)
