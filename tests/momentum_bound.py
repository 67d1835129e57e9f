"""Per-element tolerance for NEXT-1 momentum commits against the plain definition (R21).

The definition is Eq. 2 applied update by update (oracle.momentum.sequential_f64, float64).
The hot path evaluates the aggregate form of a commit of m updates (two weighted sums) in
fp32.  This module runs the definition in float64 and, alongside it, a first-order forward error
bound of ANY fp32 evaluation of the aggregate form (round to nearest, unit roundoff e = 2^-24),
per element, so that a test can require |w_fp32_i - w64_i| <= ew_i for every element i.

Per commit with members g_1..g_m (exact u_j = -lr*g_j), weights cA_j, cB_j, s_h, g_m, the fp32 path
rounds: lr (once), lr*g_j, each weight, each weight product, the m-1 adds of each fold, s_h*h, the
add of A, the add into w, g_m*h and the add of B.  With A_abs = sum cA_j |u_j|, B_abs = sum cB_j |u_j|:
  eA  = (m + 4) e A_abs                       (lr, lr*g, cA, product, and <= m-1 fold adds)
  eB  = (m + 4) e B_abs
  et  = 3 e s_h |h| + s_h eh + eA + e |t|     (s_h, its product, propagated history error, A, the add)
  ew' = ew + et + e |w'|
  eh' = g_m eh + 3 e g_m |h| + eB + e |h'|
(first order in e; the second-order terms are below 1e-12 of these at the configs' magnitudes,
covered by the factor `slack`).  The bound is what a correct fp32 evaluation in ANY order meets, so
it pins the GPU state to the definition without trusting the pinned order of weighted_f32.
"""
from __future__ import annotations

import numpy as np

EPS32 = 2.0 ** -24


def weights(m: int, gamma: float):
    pw = [1.0]
    for _ in range(m):
        pw.append(pw[-1] * gamma)
    cA = [sum(pw[: m - i + 1]) for i in range(1, m + 1)]
    cB = [pw[m - i] for i in range(1, m + 1)]
    return cA, cB, sum(pw[1:]), pw[m]


def sequential_with_bound(w, h, commits, lr: float, gamma: float, widen, slack: float = 1.01):
    """Eq. 2 per update in float64 over `commits` (lists of member arrays, commit order), plus the
    per-element error bound of an fp32 aggregate-form evaluation.  Returns (w64, h64, bound_w, bound_h)."""
    w = np.asarray(w, dtype=np.float64).copy()
    h = np.asarray(h, dtype=np.float64).copy()
    ew = np.zeros_like(w)
    eh = np.zeros_like(w)
    e = EPS32
    for members in commits:
        m = len(members)
        cA, cB, s_h, g_m = weights(m, gamma)
        A_abs = np.zeros_like(w)
        B_abs = np.zeros_like(w)
        h_before = h.copy()
        w_before = w.copy()
        for j, g in enumerate(members):
            u = -lr * widen(g).astype(np.float64)
            A_abs += cA[j] * np.abs(u)
            B_abs += cB[j] * np.abs(u)
            h = u + gamma * h                      # Eq. 2, one update at a time (the definition)
            w = w + h
        t = w - w_before
        eA = (m + 4) * e * A_abs
        eB = (m + 4) * e * B_abs
        et = 3 * e * s_h * np.abs(h_before) + s_h * eh + eA + e * np.abs(t)
        ew = ew + et + e * np.abs(w)
        eh = g_m * eh + 3 * e * g_m * np.abs(h_before) + eB + e * np.abs(h)
    return w, h, slack * ew, slack * eh
