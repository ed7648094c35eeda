"""numpy emulation of the render kernel's arithmetic (tests only).

Uses the C library's host-side design tables (frir_design_table) and the
same index algebra as csrc/frir_kernels.cu (start s', phase phi, composite
tables, output-rate LP recursion, modal tail fix), in FP64, so the
formulation can be checked against the oracle on a machine without a GPU.
"""

from __future__ import annotations

import numpy as np

from paper_2304_08052_b200 import _abi

EXT = 10


class Tables:
    def __init__(self, fs: int):
        self.d = _abi.design_describe(fs)
        g = lambda w: _abi.design_table(fs, w)
        self.comp_d, self.comp_w = g(_abi.TAB_COMP_D), g(_abi.TAB_COMP_W)
        self.kappa = g(_abi.TAB_KAPPA).reshape(-1, 2)
        self.u = g(_abi.TAB_U)
        z = g(_abi.TAB_ZPHASE).reshape(-1, 2)
        self.zphase = z[:, 0] + 1j * z[:, 1]
        p = g(_abi.TAB_PPOW).reshape(-1, 2)
        self.ppow = p[:, 0] + 1j * p[:, 1]
        lp = g(_abi.TAB_LPCOEF)
        self.c1, self.c2 = lp[0], lp[1]
        self.v0 = np.array([lp[2] + 1j * lp[3], lp[4] + 1j * lp[5]])
        self.h1up = g(_abi.TAB_H1) * self.d.up
        self.h2 = g(_abi.TAB_H2)
        self.gw = g(_abi.TAB_GW)


def render_channel(tab: Tables, q: np.ndarray, a: np.ndarray, L: int) -> np.ndarray:
    d = tab.d
    up, down, r_h, r_l = d.up, d.down, d.r_h, d.r_l
    n1 = -(-L * up // down)
    n2 = -(-n1 // r_l)
    q = np.asarray(q, np.int64)
    a = np.asarray(a, np.float64)
    s = -((-(q + d.t0)) // r_h)
    sp = s + EXT
    phi = r_h * s - q - d.t0
    D = np.zeros(n2 + EXT + d.sup + 64)
    W = np.zeros_like(D)
    for k in range(d.sup):
        idx = sp + k
        ok = idx >= 0
        t = phi + r_h * k
        np.add.at(D, idx[ok], a[ok] * tab.comp_d[t[ok]])
        np.add.at(W, idx[ok], a[ok] * tab.comp_w[t[ok]])
    # head: stage-1 taps at mid index k < 0 do not exist in the reference
    for qi, ai in zip(q, a):
        if up * qi >= d.half1:
            continue
        klo = -((-(up * qi - d.half1)) // down)
        for k in range(klo, 0):
            c = ai * tab.h1up[down * k + d.half1 - up * qi]
            for n in range(-EXT, n2):
                idx = r_l * n + d.half2 - k
                if 0 <= idx < len(tab.h2) and n >= 0:
                    D[n + EXT] -= c * tab.h2[idx]
                if 0 <= idx < len(tab.gw):
                    W[n + EXT] -= c * tab.gw[idx]
    LP = np.zeros(n2 + EXT)
    p1 = p2 = 0.0
    for n in range(n2 + EXT):
        v = W[n] + tab.c1 * p1 + tab.c2 * p2
        LP[n], p2, p1 = v, p1, v
    y = D[EXT:n2 + EXT] - LP[EXT:]
    # tail: state at n1 from images within the horizon, plus taps past n1
    e = up * q + d.half1
    khi = e // down
    zeta = 0j
    xt = np.zeros(d.lt_max)
    for qi, ai, kh, ei in zip(q, a, khi, e):
        if kh < n1 - d.horizon:
            continue
        if kh < n1 and up * qi >= d.half1:
            zeta += ai * tab.ppow[n1 - 1 - kh] * tab.zphase[ei - down * kh]
            continue
        klo = max(0, -((-(up * qi - d.half1)) // down))
        for k in range(klo, kh + 1):
            c = ai * tab.h1up[down * k + d.half1 - up * qi]
            if k < n1:
                if n1 - 1 - k < d.horizon:
                    zeta += c * tab.ppow[n1 - 1 - k]
            else:
                xt[k - n1] += c
    s_state = 2.0 * np.real(tab.v0 * zeta)
    n_c = max(0, -(-(n1 - d.half2) // r_l)) if n1 > d.half2 else 0
    for n in range(n_c, n2):
        ee = r_l * n + d.half2 - n1
        if not (0 <= ee < d.half2):
            continue
        corr = tab.kappa[ee] @ s_state
        for l in range(min(ee + 1, d.lt_max)):
            corr += xt[l] * tab.u[ee - l]
        y[n] -= corr
    return y
