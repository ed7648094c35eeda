"""Build libfrir with extra nvcc defines into lib/libfrir_<name>.so (A/B dev tool).

usage: python tools/build_variant.py NAME -DMACRO=VALUE ...
"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_08052_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = B.OUT.parent / f"libfrir_{name}.so"
cmd = [B._nvcc(), *B.NVCC_FLAGS, *defs, "-o", str(out), *[str(B.CSRC / s) for s in B.SOURCES]]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr[-2000:])
print(out)
