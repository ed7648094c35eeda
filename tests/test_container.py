"""FRIR container (io.py:26-107 mirror): byte compatibility with a file the
reference wrote, round trips, and the reference's error cases."""

import numpy as np
import pytest

from paper_2304_08052_b200 import container as C


def test_reads_reference_file(golden_dir):
    recs = C.read_rir_container(golden_dir / "container.frir")
    assert len(recs) == 2
    assert recs[0].samples.shape == (2, 17) and recs[0].sample_rate == 16000 and recs[0].kind == "full"
    assert recs[1].samples.shape == (3, 5) and recs[1].kind == "early" and recs[1].seed == 2**63 - 5


def test_writes_reference_bytes(golden_dir, tmp_path):
    recs = C.read_rir_container(golden_dir / "container.frir")
    out = tmp_path / "x.frir"
    C.write_rir_container(out, recs)
    assert out.read_bytes() == (golden_dir / "container.frir").read_bytes()


def test_errors(tmp_path):
    p = tmp_path / "bad.frir"
    p.write_bytes(b"XXXX" + b"\0" * 6)
    with pytest.raises(ValueError, match="bad magic"):
        C.read_rir_container(p)
    p.write_bytes(b"FRIR" + (2).to_bytes(2, "little") + (0).to_bytes(4, "little"))
    with pytest.raises(ValueError, match="unsupported container version"):
        C.read_rir_container(p)
    C.write_rir_container(p, [C.RirRecord(samples=np.ones((2, 8)), sample_rate=16000)])
    raw = p.read_bytes()
    p.write_bytes(raw[:-4])
    with pytest.raises(ValueError, match="payload shorter"):
        C.read_rir_container(p)
    p.write_bytes(raw[:5])
    with pytest.raises(ValueError, match="truncated container header"):
        C.read_rir_container(p)
