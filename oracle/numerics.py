"""O6 — ordered commit numerics.  TEST INFRASTRUCTURE.

What the hot path computes, written as its plain definition:
* Server update, Eq. 2 with gamma = 0 and the north-star sign (reading
  R18: u is the raw gradient, the server applies w <- w - lr * u).
* Aggregators compute the sum of their group's updates in O(U)
  order (updates "forwarded to aggregators as per O(U)"), and an
  aggregate commit must be "consistent to the case with no aggregation"
  (P:1072-1073).
* The replica applies the same updates in the exact same order; the
  hot path realises it as a mirror store of w at the plan's boundary commit
  (reading R16).

Reading R17: fp32 model; fp32 or bf16 updates, bf16 widened
exactly (u32 = u16 << 16); in-group LEFT FOLD in O(U) order,
x = (((u1 + u2) + u3) + ...), every add rounded to fp32; commit
w <- w - (lr * x) with the product and the difference each rounded to fp32
(never fused).  numpy float32 elementwise ops are IEEE round-to-nearest and are
never contracted, and np.sum is not used (it is pairwise).

Parity: pinned by the exact-arithmetic special case (synthgen variant "exact":
no rounding anywhere, so the result equals the exact rational value computed
with Python Fractions in tests/test_oracle_numerics.py) and by a hand-worked
rounding example where the two-rounding commit differs from an FMA.
"""
from __future__ import annotations

import numpy as np


def widen(a: np.ndarray) -> np.ndarray:
    """fp32 operand as-is; bf16 bit patterns (uint16) widened exactly (R17, SURVEY §8(c)
    O6): a bf16 value is the upper half of the fp32 with the same sign, exponent and leading
    7 mantissa bits, so the fp32 bit pattern is u32 = u16 << 16 (low half zero)."""
    if a.dtype == np.uint16:
        return (a.astype(np.uint32) << np.uint32(16)).view(np.float32)
    assert a.dtype == np.float32
    return a


def fold(members: list) -> np.ndarray:
    """x = (((m1 + m2) + m3) + ...) in fp32, left to right."""
    x = widen(members[0]).astype(np.float32, copy=True)
    for m in members[1:]:
        x = np.add(x, widen(m), dtype=np.float32)
    return x


def commit_batch(w: np.ndarray, commits: list, lr: float, boundary: int = -1):
    """Apply commits (each a list of member arrays, O(U) order) to w in order.

    boundary b (R16): backup <- w after the b-th commit (b = 0: the loaded w,
    b = -1: no backup write).  Returns (w_new, backup or None).
    """
    lr32 = np.float32(lr)
    w = np.array(w, dtype=np.float32, copy=True)
    backup = w.copy() if boundary == 0 else None
    for c, members in enumerate(commits, start=1):
        x = fold(members)
        prod = np.multiply(lr32, x, dtype=np.float32)     # rounding 1
        w = np.subtract(w, prod, dtype=np.float32)        # rounding 2
        if c == boundary:
            backup = w.copy()
    return w, backup


def commits_from_plan(plan: dict, operand) -> list:
    """Member arrays per server commit: operand(batch_index) -> array."""
    out = []
    for f, k in zip(plan["commit_first"], plan["commit_count"]):
        out.append([operand(plan["order"][p]) for p in range(f, f + k)])
    return out


def execute_plan(w: np.ndarray, plan: dict, operand, lr: float):
    """The whole batch: returns (w_new, backup or None, committed update count)."""
    commits = commits_from_plan(plan, operand)
    w_new, backup = commit_batch(w, commits, lr, plan["replica_boundary_commit"])
    return w_new, backup, plan["n_commit"]
