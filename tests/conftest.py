import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
TESTS = Path(__file__).resolve().parent
if str(TESTS) not in sys.path:
    sys.path.insert(0, str(TESTS))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    g = ROOT / "tests" / "golden"
    return {
        "kat": json.loads((g / "kat.json").read_text()),
        "cfg1": dict(np.load(g / "cfg1.npz")),
        "cases": dict(np.load(g / "cases.npz")),
        "cases_meta": json.loads((g / "cases.json").read_text()),
        "mix": dict(np.load(g / "mix.npz")),
        "mix_meta": json.loads((g / "mix.json").read_text()),
        "ism": dict(np.load(g / "ism.npz")),
        "ism_meta": json.loads((g / "ism.json").read_text()),
        "decay": dict(np.load(g / "decay.npz")),
        "decay_meta": json.loads((g / "decay.json").read_text()),
    }


@pytest.fixture(scope="session")
def golden_dir():
    return ROOT / "tests" / "golden"


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    # Tests run against the in-tree library; build it if sources changed
    # (nvcc cross-compiles without a GPU).
    from paper_2304_08052_b200 import build

    build.build()


@pytest.fixture(scope="session", autouse=True)
def _debug_bounds_checks():
    """With FRIR_LIB pointing at libfrir_debug.so (build.py --debug), every
    kernel index is bounds-checked; fail the session if any check fired."""
    yield
    import os

    if "debug" in os.environ.get("FRIR_LIB", ""):
        from paper_2304_08052_b200 import _abi

        line = _abi.lib().frir_debug_status()
        assert line == 0, f"a device bounds check failed at frir_kernels.cu:{line}"
