"""Build libfrir.so in-tree with nvcc for sm_100a (no GPU needed)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "lib" / "libfrir.so"
SOURCES = ["frir_abi.cu", "frir_kernels.cu", "frir_mix.cu", "frir_fftconv.cu", "frir_decay.cu", "frir_scene.cu", "frir_stages.cu", "frir_design.cpp"]
HEADERS = ["frir_internal.h", "frir_design.h", "frir_philox.cuh"]
INCLUDE = PKG.parent / "include" / "frir.h"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",  # FP64 geometry keeps numpy's rounding (explicit fmaf/fma stay fused)
    "-Xcompiler", "-fPIC,-O3",
    "-shared", "-cudart", "static",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [INCLUDE]
    return any(p.stat().st_mtime > t for p in deps)


DEBUG_OUT = PKG / "lib" / "libfrir_debug.so"


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> Path:
    """Compile libfrir.so (or, with debug=True, libfrir_debug.so whose kernels
    trap on out-of-range indices; load it with FRIR_LIB=...) if stale."""
    out = DEBUG_OUT if debug else OUT
    if not force and not debug and not _stale():
        return OUT
    out.parent.mkdir(parents=True, exist_ok=True)
    tmp = out.with_suffix(".so.tmp")
    flags = NVCC_FLAGS + (["-DFRIR_DEBUG"] if debug else [])
    cmd = [_nvcc(), *flags, "-o", str(tmp), *[str(CSRC / s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, debug="--debug" in sys.argv))
