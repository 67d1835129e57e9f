"""Oracle O6 pinned: exact-arithmetic special case equals the exact rational result;
rounded case equals an independent rational emulation of correctly-rounded fp32 ops."""
from fractions import Fraction

import numpy as np

import synthgen as sg
from oracle.numerics import commit_batch, execute_plan, fold


def round_f32(q: Fraction) -> Fraction:
    """Round a rational to the nearest fp32 value, ties to even (normal + subnormal range)."""
    if q == 0:
        return Fraction(0)
    s = -1 if q < 0 else 1
    a = abs(q)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    ulp = Fraction(2) ** (max(e, -126) - 23)
    m = a / ulp
    n = m.numerator // m.denominator
    rem = m - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    return s * n * ulp


def F(x) -> Fraction:
    return Fraction(float(x))


def random_commits(seed, n_updates, n_elems, variant, dtype=sg.DTYPE_F32):
    key = sg.stream_key(seed, sg.KIND_MISC, 9, 0)
    commits, c, w = [], 0, 0
    while w < n_updates:
        m = 1 + sg.word(key, c) % 4
        c += 1
        commits.append([sg.update_values(seed, w + j, 0, np.arange(n_elems), dtype, variant)
                        for j in range(min(m, n_updates - w))])
        w += m
    return commits


def test_exact_case_equals_exact_rational_result():
    lr = 2.0**-4
    for seed, nu in ((1, 1), (2, 7), (3, 40), (4, 256)):
        n = 33
        w0 = sg.w0_values(seed, np.arange(n), "exact")
        for dtype in (sg.DTYPE_F32, sg.DTYPE_BF16):
            commits = random_commits(seed, nu, n, "exact", dtype)
            b = len(commits) // 2
            w, backup = commit_batch(w0, commits, lr, boundary=b)
            for i in range(n):
                exact = F(w0[i])
                for ci, mem in enumerate(commits, start=1):
                    vals = [F(fold([m[i:i + 1]])[0]) for m in mem]
                    exact -= Fraction(lr) * sum(vals)       # no rounding anywhere in this case
                    if ci == b:
                        assert F(backup[i]) == exact
                assert F(w[i]) == exact
            # any summation order gives the same bits in the exact case
            flat = [[m] for mem in commits for m in mem][::-1]
            w_rev, _ = commit_batch(w0, flat, lr)
            assert np.array_equal(w.view(np.uint32), w_rev.view(np.uint32))


def test_rounded_case_equals_rational_emulation():
    lr = 0.01
    n = 24
    for seed in range(6):
        w0 = sg.w0_values(seed, np.arange(n))
        commits = random_commits(seed, 9, n, "normal")
        w, _ = commit_batch(w0, commits, lr)
        lr32 = F(np.float32(lr))
        for i in range(n):
            wi = F(w0[i])
            for mem in commits:
                x = F(mem[0][i])
                for m in mem[1:]:
                    x = round_f32(x + F(m[i]))              # left fold, each add rounded
                p = round_f32(lr32 * x)                     # rounding 1
                wi = round_f32(wi - p)                      # rounding 2
            assert F(w[i]) == wi


def test_two_roundings_are_not_an_fma():
    # R17: the commit must not be contracted; find elements where an FMA would differ
    n = 4096
    w0 = sg.w0_values(3, np.arange(n))
    x = sg.w0_values(4, np.arange(n))              # an operand of w's magnitude
    w, _ = commit_batch(w0, [[x]], 0.7)
    lr32 = F(np.float32(0.7))
    diff = 0
    for i in range(n):
        fma = round_f32(F(w0[i]) - lr32 * F(x[i]))
        two = round_f32(F(w0[i]) - round_f32(lr32 * F(x[i])))
        assert F(w[i]) == two
        diff += fma != two
    assert diff > 0


def test_plan_driven_execution_and_bf16_widening():
    bits = np.array([0x3F80, 0xBF80, 0x0001, 0x7F7F], dtype=np.uint16)
    f = fold([bits])
    assert f[0] == 1.0 and f[1] == -1.0 and f[2] == np.float32(2.0**-133) and f[3] == np.float32(3.3895314e38)
    plan = {"order": [2, 0, 1], "commit_first": [0, 1], "commit_count": [1, 2],
            "replica_boundary_commit": 1, "n_commit": 3}
    ops = {g: sg.update_values(5, g, 0, np.arange(8)) for g in range(3)}
    w0 = sg.w0_values(5, np.arange(8))
    w, backup, n = execute_plan(w0, plan, lambda g: ops[g], 0.5)
    w_ref, b_ref = commit_batch(w0, [[ops[2]], [ops[0], ops[1]]], 0.5, 1)
    assert n == 3 and np.array_equal(w, w_ref) and np.array_equal(backup, b_ref)
