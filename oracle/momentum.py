"""NEXT-1 — momentum (Eq. 2 with gamma > 0) and its aggregate form.  TEST INFRASTRUCTURE.

Paper passages:
* Server update, Eq. 2: w_{t+1} = w_t + u + gamma (w_t - w_{t-1}); with the
  history h_t = w_t - w_{t-1} this is h <- u + gamma h, w <- w + h, one update at a
  time.  North-star sign (R18): u = -lr * g for the pushed gradient g.
* Aggregators compute the (weighted) sum of incoming updates and an
  aggregate commit must be "consistent to the case with no aggregation"
  (P:1072-1073).  Applying Eq. 2 m times in O(U) order gives, for the group
  u_1..u_m (the same expansion as Eq. 6-9):
      w' = w + (sum_{j=1..m} g^j) h + sum_i (sum_{j=0..m-i} g^j) u_i
      h' = g^m h + sum_i g^(m-i) u_i
  i.e. two weighted sums over the same operands.

Two oracles:
* sequential_f64 — the plain definition: Eq. 2 per update, in float64.
* weighted_f32 — the same two weighted sums evaluated in fp32 in a pinned order (reading
  R21: the model and its history are fp32, the paper fixes no precision): gamma is the
  float64 value of the ABI (the same double the planner's Eq. 9/12 bound uses); the
  coefficients are float64 powers pw[j] = pw[j-1]*gamma summed left to right, each rounded
  once to fp32; per member u_i = -(lr*g_i); A = left fold of (cA_i*u_i), B = left fold of
  (cB_i*u_i); t = s_h*h + A; w' = w + t; h' = g_m*h + B; every product / sum rounded to
  fp32, never fused.  The order is a reading, so weighted_f32 is checked against
  sequential_f64 (the definition) with the tolerance DESIGN.md R21 derives.

Parity: weighted_f32 equals the exact rational value of the sequential definition in
an exact-arithmetic case (gamma = 1/2, dyadic inputs), and is within 1e-6
(norm-relative) of sequential_f64 on random data (tests/test_oracle_momentum.py).
"""
from __future__ import annotations

import numpy as np

from .numerics import widen


def coefficients(m: int, gamma: float):
    """(cA[1..m], cB[1..m], s_h, g_m) in float64, fixed evaluation order."""
    pw = [1.0]
    for _ in range(m):
        pw.append(pw[-1] * gamma)
    cA = []
    for i in range(1, m + 1):
        c = 0.0
        for j in range(0, m - i + 1):
            c += pw[j]
        cA.append(c)
    cB = [pw[m - i] for i in range(1, m + 1)]
    s_h = 0.0
    for j in range(1, m + 1):
        s_h += pw[j]
    return cA, cB, s_h, pw[m]


def sequential_f64(w, h, commits: list, lr: float, gamma: float, boundary: int = -1):
    """Eq. 2 applied update by update in float64.  Returns (w, h, backup or None)."""
    w = np.asarray(w, dtype=np.float64).copy()
    h = np.asarray(h, dtype=np.float64).copy()
    backup = (w.copy(), h.copy()) if boundary == 0 else None
    for c, members in enumerate(commits, start=1):
        for g in members:
            u = -lr * widen(g).astype(np.float64)
            h = u + gamma * h
            w = w + h
        if c == boundary:
            backup = (w.copy(), h.copy())
    return w, h, backup


def weighted_f32(w, h, commits: list, lr: float, gamma: float, boundary: int = -1):
    """The aggregate (weighted-sum) form in fp32, pinned order.  Returns (w, h, backup)."""
    f = np.float32
    gamma = float(gamma)                  # R21: one float64 gamma; each weight rounded once to fp32
    w = np.asarray(w, dtype=np.float32).copy()
    h = np.asarray(h, dtype=np.float32).copy()
    lr32 = f(lr)
    backup = (w.copy(), h.copy()) if boundary == 0 else None
    for c, members in enumerate(commits, start=1):
        cA, cB, s_h, g_m = coefficients(len(members), gamma)
        A = B = None
        for i, g in enumerate(members):
            u = np.negative(np.multiply(lr32, widen(g), dtype=np.float32))
            a = np.multiply(f(cA[i]), u, dtype=np.float32)
            b = np.multiply(f(cB[i]), u, dtype=np.float32)
            A = a if A is None else np.add(A, a, dtype=np.float32)
            B = b if B is None else np.add(B, b, dtype=np.float32)
        t = np.add(np.multiply(f(s_h), h, dtype=np.float32), A, dtype=np.float32)
        w = np.add(w, t, dtype=np.float32)
        h = np.add(np.multiply(f(g_m), h, dtype=np.float32), B, dtype=np.float32)
        if c == boundary:
            backup = (w.copy(), h.copy())
    return w, h, backup
