"""NEXT-1 oracle pinned: the weighted-sum aggregate equals the paper's sequential Eq. 2 exactly
in an exact-arithmetic case, and within 1e-6 otherwise; coefficients reduce to Eq. 9's."""
from fractions import Fraction

import numpy as np

import synthgen as sg
from oracle.momentum import coefficients, sequential_f64, weighted_f32


def F(x):
    return Fraction(float(x))


def test_coefficients_match_eq9_and_limits():
    # m = 2 (Eq. 9): w' - w = (g + g^2) h + (1 + g) u1 + u2
    cA, cB, s_h, g_m = coefficients(2, 0.9)
    assert np.isclose(s_h, 0.9 + 0.81) and np.allclose(cA, [1.9, 1.0]) and np.allclose(cB, [0.9, 1.0])
    assert np.isclose(g_m, 0.81)
    cA, cB, s_h, g_m = coefficients(3, 0.0)          # gamma = 0: plain sum, history forgotten
    assert cA == [1.0, 1.0, 1.0] and cB == [0.0, 0.0, 1.0] and s_h == 0.0 and g_m == 0.0
    cA, cB, s_h, g_m = coefficients(1, 0.5)          # m = 1 is Eq. 2 itself
    assert cA == [1.0] and cB == [1.0] and s_h == 0.5 and g_m == 0.5


def test_weighted_equals_sequential_exactly_in_exact_case():
    # gamma = 1/2, lr = 2^-4, g = int11 * 2^-20, w0 = h0 = 0: every fp32 op is exact,
    # so the aggregate form must equal the exact rational sequential result
    n = 16
    idx = np.arange(n)
    gamma, lr = 0.5, 2.0**-4
    for seed in range(5):
        sizes = [1 + (seed + k) % 4 for k in range(3)]
        commits, w_id = [], 0
        for m in sizes:
            commits.append([sg.update_values(seed, w_id + j, 0, idx, sg.DTYPE_F32, "exact") for j in range(m)])
            w_id += m
        w0 = np.zeros(n, np.float32)
        h0 = np.zeros(n, np.float32)
        w, h, bk = weighted_f32(w0, h0, commits, lr, gamma, boundary=2)
        for e in range(n):
            we, he = Fraction(0), Fraction(0)
            for ci, mem in enumerate(commits, start=1):
                for g in mem:
                    he = -Fraction(lr) * F(g[e]) + Fraction(gamma) * he      # Eq. 2, exact
                    we = we + he
                if ci == 2:
                    assert F(bk[0][e]) == we and F(bk[1][e]) == he
            assert F(w[e]) == we and F(h[e]) == he


def test_weighted_close_to_sequential_f64():
    n = 4096
    idx = np.arange(n)
    for seed, gamma in ((1, 0.9), (2, 0.5), (3, 0.99)):
        rng = np.random.default_rng(seed)
        commits, w_id = [], 0
        for _ in range(6):
            m = int(rng.integers(1, 6))
            commits.append([sg.update_values(seed, w_id + j, 0, idx) for j in range(m)])
            w_id += m
        w0 = sg.w0_values(seed, idx)
        h0 = (sg.w0_values(seed + 100, idx) * np.float32(1e-3)).astype(np.float32)
        w32, h32, _ = weighted_f32(w0, h0, commits, 0.01, gamma)
        w64, h64, _ = sequential_f64(w0, h0, commits, 0.01, gamma)
        assert np.max(np.abs(w32 - w64)) <= 1e-6 * np.max(np.abs(w64))
        assert np.max(np.abs(h32 - h64)) <= 1e-5 * np.max(np.abs(h64))
        # the same updates committed one per commit (no aggregation) agree too
        single = [[g] for mem in commits for g in mem]
        w1, _, _ = weighted_f32(w0, h0, single, 0.01, gamma)
        assert np.max(np.abs(w1 - w64)) <= 1e-6 * np.max(np.abs(w64))


def test_weighted_within_per_element_bound_of_sequential():
    # DESIGN.md R21: every element of the fp32 aggregate form lies within the first-order forward
    # error bound of the plain sequential Eq. 2 (tests/momentum_bound.py); a dropped or wrong
    # weight (e.g. cB with gamma^(m-i+1)) moves elements by ~|u| >> the bound
    from oracle.numerics import widen
    from tests.momentum_bound import sequential_with_bound
    n = 200_000
    idx = np.arange(n)
    for seed, gamma, dt in ((4, 0.9, sg.DTYPE_F32), (5, 0.9, sg.DTYPE_BF16), (6, 0.99, sg.DTYPE_F32)):
        rng = np.random.default_rng(seed)
        commits, w_id = [], 0
        for _ in range(12):
            m = int(rng.integers(1, 9))
            commits.append([sg.update_values(seed, w_id + j, 0, idx, dt) for j in range(m)])
            w_id += m
        w0 = sg.w0_values(seed, idx)
        h0 = (sg.w0_values(seed + 100, idx) * np.float32(1e-3)).astype(np.float32)
        w32, h32, _ = weighted_f32(w0, h0, commits, 0.01, gamma)
        w64, h64, bw, bh = sequential_with_bound(w0, h0, commits, 0.01, gamma, widen)
        assert np.all(np.abs(w32 - w64) <= bw) and np.all(np.abs(h32 - h64) <= bh)
        # the bound is tight enough to matter: a plausible slip in the weights breaks it
        bad = [[g for g in mem] for mem in commits]
        wb, _, _ = weighted_f32(w0, h0, [mem[::-1] for mem in bad], 0.01, gamma)   # members reversed
        assert np.any(np.abs(wb - w64) > bw)
