"""Rows of the decay golden cases (tests/golden/decay.*)."""

import numpy as np


def rows(golden):
    g = golden["cfg1"]
    out = [g["full"][m] for m in range(g["full"].shape[0])] + [g["early"][0]]
    d = golden["decay"]
    i = len(out)
    while f"r{i}" in d:
        out.append(d[f"r{i}"])
        i += 1
    return [np.asarray(r, dtype=np.float32) for r in out]
