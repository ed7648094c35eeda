"""C-ABI library checks that need no GPU: loading, exported symbols, struct
layouts, the host-side Philox/SeedSequence restatement and the filter design."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest
from scipy import signal

from paper_2304_08052_b200 import _abi, engine, rate_factors

HEADER = Path(__file__).resolve().parents[1] / "include" / "frir.h"


def test_library_exports_every_declared_symbol():
    lib = _abi.lib()
    decl = set(re.findall(r"^(?:int|int32_t|int64_t|size_t|const char\*)\s+(frir_[a-z0-9_]+)\(",
                          HEADER.read_text(), flags=re.M))
    assert decl, "no declarations parsed"
    for name in sorted(decl):
        assert hasattr(lib, name), name
    assert decl == {s[0] for s in _abi.SIGNATURES}


def test_struct_layouts_match():
    lib = _abi.lib()
    assert lib.frir_struct_size(0) == ctypes.sizeof(_abi.FrirJob) == _abi.JOB_DTYPE.itemsize
    assert lib.frir_struct_size(1) == ctypes.sizeof(_abi.FrirBatch)
    assert lib.frir_struct_size(2) == ctypes.sizeof(_abi.FrirPlanDesc)


def test_philox_restatement_bit_exact(golden):
    for e in golden["kat"]["philox"]:
        got = _abi.philox_doubles(int(e["seed"]), e["k"], e["stage"], e["first"], 8)
        assert [float(x).hex() for x in got] == e["doubles"]


@pytest.mark.parametrize("seed,k,stage", [(0, 0, 0), (1, 2, 1), (2**63 - 1, 7, 0), (2**64 - 1, 0, 1),
                                          (4294967296, 3, 1), (12345, 65536, 0)])
def test_philox_random_streams(seed, k, stage):
    g = np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, k, stage))))
    ref = g.random(2053)
    got = _abi.philox_doubles(seed, k, stage, 0, 2053)
    assert np.array_equal(ref, got)
    assert np.array_equal(ref[1001:1050], _abi.philox_doubles(seed, k, stage, 1001, 49))


@pytest.mark.parametrize("fs", [8000, 11025, 16000, 22050, 24000, 32000, 44100, 48000, 96000])
def test_design_matches_scipy(fs):
    f = rate_factors(fs)
    d = _abi.design_describe(fs)
    assert (d.r_h, d.r_l) == (f.r_h, f.r_l)
    m = max(f.r_l, f.r_h)
    h1 = signal.firwin(20 * m + 1, 1.0 / m, window=("kaiser", 7.0))
    h2 = signal.firwin(20 * f.r_l + 1, 1.0 / f.r_l, window=("kaiser", 7.0))
    sos = signal.butter(2, 80.0, btype="highpass", fs=f.mid_rate, output="sos")[0]
    assert np.abs(_abi.design_table(fs, _abi.TAB_H1) - h1).max() < 1e-15
    assert np.abs(_abi.design_table(fs, _abi.TAB_H2) - h2).max() < 1e-15
    assert np.allclose(_abi.design_table(fs, _abi.TAB_SOS), sos, rtol=1e-13, atol=0)
    assert list(d.sos) == list(_abi.design_table(fs, _abi.TAB_SOS))


@pytest.mark.parametrize("fs", [8000, 16000, 44100, 48000])
def test_composite_tables_equal_chain_response(fs):
    """T_D(t) is the chain (without HP) response at output n=0 to a unit
    impulse at high-rate index -t: check against scipy resample_poly twice."""
    f = rate_factors(fs)
    d = _abi.design_describe(fs)
    comp = _abi.design_table(fs, _abi.TAB_COMP_D)
    m = max(f.r_l, f.r_h)
    h1 = signal.firwin(20 * m + 1, 1.0 / m, window=("kaiser", 7.0))
    h2 = signal.firwin(20 * f.r_l + 1, 1.0 / f.r_l, window=("kaiser", 7.0))
    rng = np.random.default_rng(fs)
    for q in rng.integers(60 * f.r_h, 90 * f.r_h, size=3):
        x = np.zeros(150 * f.r_h)
        x[q] = 1.0
        y = signal.resample_poly(x, f.r_l, f.r_h, window=h1)
        y = signal.resample_poly(y, 1, f.r_l, window=h2)
        n = np.arange(len(y))
        t = f.r_h * n - q - d.t0
        ok = (t >= 0) & (t < len(comp))
        pred = np.zeros(len(y))
        pred[ok] = comp[t[ok]]
        assert np.abs(pred - y)[40:-40].max() < 1e-12


def test_invalid_rates_rejected():
    for fs in (0, -1, 1_000_000, 400_000):
        with pytest.raises(ValueError):
            _abi.design_describe(fs)


def _one_job(**kw):
    jobs = engine.new_jobs(1)
    jobs["room"] = (5.0, 4.0, 3.0)
    jobs["d0"] = 1.5
    jobs["t60"] = 0.5
    jobs["n_images"] = 64
    jobs["n_mics"] = 4
    for k, v in kw.items():
        jobs[k] = v
    return jobs


MICS = np.zeros((4, 3))


def test_jobs_prepare_layout_and_derived():
    jobs = engine.new_jobs(3)
    jobs["room"] = (5.0, 4.0, 3.0)
    jobs["d0"] = 1.5
    jobs["t60"] = [0.5, 0.25, 0.3]
    jobs["n_images"] = [100, 0, 7]
    jobs["n_mics"] = [4, 2, 3]
    jobs["mic_off"] = [0, 4, 6]
    pb = engine.prepare(16000, jobs, np.zeros((9, 3)))
    j = pb.jobs
    assert list(j["img_off"]) == [0, 101, 102]
    assert list(j["item_off"]) == [0, 404, 406]
    assert list(j["chan_off"]) == [0, 4, 6]
    assert list(j["L"]) == [496000, 248000, 297600]
    assert list(j["n2"]) == [8000, 4000, 4800]
    assert list(j["out_off"]) == [0, 32000, 40000]
    assert pb.batch.total_out == 40000 + 3 * 4800
    assert list(pb.chan_job) == [0, 0, 0, 0, 1, 1, 2, 2, 2]
    assert sorted(pb.chan_order) == list(range(9))
    assert j["r"][0] == pytest.approx(0.98279, abs=1e-5)
    assert j["rr_max"][0] == pytest.approx(124.896, abs=0.01)
    assert j["rr_max"][1] == 0.0  # no images: RR_max never evaluated (core.py:295)
    # keys are the SeedSequence((seed, k, stage)) words
    ss = np.random.SeedSequence((0, 0, 0)).generate_state(2, np.uint64)
    assert [int(x) for x in j["key"][0][:2]] == [int(x) for x in ss]
    padded = engine.prepare(16000, jobs, np.zeros((9, 3)), padded=True)
    assert list(padded.jobs["out_stride"]) == [8000] * 3
    odd = engine.prepare(16000, _one_job(t60=0.30001), MICS)
    assert odd.jobs["n2"][0] == 4801 and odd.jobs["out_stride"][0] == 4804  # 16-byte aligned rows


@pytest.mark.parametrize("kw,msg", [
    ({"t60": 0.0}, "t60 must be > 0"),
    ({"alpha": 0.0}, "alpha must be > 0 to sample image distances"),
    ({"alpha": 0.5, "beta": 0.5}, "need 0 <= alpha < beta <= 1"),
    ({"t60": 0.004}, "must exceed the direct distance"),
    ({"d0": 0.02, "t60": 1.5}, "rr_max must be >= 1"),
    ({"tau": 0.0}, "tau must be > 0"),
    ({"n_mics": 0}, "M >= 1"),
    ({"room": (5.0, 0.0, 3.0)}, "room_dims"),
])
def test_jobs_prepare_rejects_like_reference(kw, msg):
    with pytest.raises(ValueError, match=msg):
        engine.prepare(16000, _one_job(**kw), MICS)


def test_jobs_prepare_rejects_oversized_jobs():
    with pytest.raises(_abi.FrirLibraryError, match="exceeds the supported maximum"):
        engine.prepare(16000, _one_job(n_images=1 << 22), MICS)
    engine.prepare(16000, _one_job(n_images=100000), MICS)  # large (ISM-sized) lists are fine


def test_jobs_prepare_ism_rules():
    j = _one_job()
    j["kind"] = _abi.KIND_ISM
    j["d0"] = 0.0
    j["duration"] = 0.05
    pb = engine.prepare(16000, j, MICS)
    assert pb.jobs[0]["L"] == int(np.ceil(0.05 * 62 * 16000))
    r = pb.jobs[0]["r"]
    lx, ly, lz = j["room"][0]
    assert r == np.exp(-0.0805 * (lx * ly * lz) / (2.0 * (lx * ly + lx * lz + ly * lz)) / j["t60"][0])
    j["reflection"] = 1.5
    with pytest.raises(ValueError, match="reflection coefficient must be in"):
        engine.prepare(16000, j, MICS)
    j["reflection"] = 0.0
    j["kind"] = 7
    with pytest.raises(ValueError, match="unknown job kind"):
        engine.prepare(16000, j, MICS)


def test_jobs_prepare_ism_device_lattice():
    """`lattice` = K + 1: frir_jobs_prepare sizes the job for the (2K+1)^3 - 1
    lattice points (enumerate_images without the origin, ism.py:80-104)."""
    j = _one_job()
    j["kind"] = _abi.KIND_ISM
    j["d0"] = 0.0
    for K in (0, 1, 3):
        j["lattice"] = K + 1
        pb = engine.prepare(16000, j, MICS)
        assert pb.jobs[0]["n_images"] == (2 * K + 1) ** 3 - 1
        assert pb.batch.total_images == (2 * K + 1) ** 3
    j["lattice"] = -1
    with pytest.raises(ValueError, match="max_order must be >= 0"):
        engine.prepare(16000, j, MICS)
    j["lattice"] = 82  # 163^3 points: past the per-job row limit (2^22)
    with pytest.raises(_abi.FrirLibraryError, match="too many points"):
        engine.prepare(16000, j, MICS)


def test_header_compiles_as_c_and_links(tmp_path):
    """include/frir.h is plain C (C99): a C program includes it, links
    libfrir.so and calls the host-only entry points."""
    import shutil
    import subprocess

    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    src = tmp_path / "abi.c"
    src.write_text(r"""
#include <stdio.h>
#include "frir.h"
int main(void) {
  frir_plan_desc d;
  if (frir_abi_version() != FRIR_ABI_VERSION) return 2;
  if (frir_design_describe(16000, &d) != FRIR_OK) return 3;
  if (d.r_h != 62 || d.r_l != 7) return 4;
  if (frir_struct_size(0) != (int64_t)sizeof(frir_job)) return 5;
  if (frir_struct_size(1) != (int64_t)sizeof(frir_batch)) return 6;
  if (frir_design_describe(1000000, &d) == FRIR_OK) return 7;   /* rejected like rate_factors */
  printf("%s\n", frir_last_error());
  return 0;
}
""")
    lib = Path(_abi.LIB_PATH)
    exe = tmp_path / "abi"
    subprocess.run([gcc, "-std=c99", "-Wall", "-Werror", "-I", str(HEADER.parent), str(src), "-o", str(exe),
                    "-L", str(lib.parent), "-lfrir", f"-Wl,-rpath,{lib.parent}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out
    assert out.stdout.strip()  # the rejection left a message
