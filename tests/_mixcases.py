"""Unpack the spatialise-and-mix golden cases (tests/golden/mix.*)."""

import numpy as np


def case(golden, i):
    m = golden["mix_meta"][i]
    z = golden["mix"]
    pre = f"c{i}_"
    S = len(m["lens"])
    srcs = [z[pre + f"src{k}"].astype(np.float64) for k in range(S)]
    noise = z[pre + "noise"].astype(np.float64)
    rf = [z[pre + f"rirf{k}"].astype(np.float64) for k in range(S + 1)]
    re = [z[pre + f"rire{k}"].astype(np.float64) if pre + f"rire{k}" in z else None for k in range(S)]
    ref = {
        "mixture": z[pre + "mixture"],
        "sources": [z[pre + f"out_src{k}"] for k in range(S)],
        "early": [z[pre + f"out_early{k}"] for k in range(S)],
        "noise": z[pre + "out_noise"],
    }
    return m, srcs, noise, rf, re, ref
