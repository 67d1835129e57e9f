"""O7 — plan invariants.  TEST INFRASTRUCTURE.

* Delay bound (§3.1): every committed update's delay
  (v_init + p) - v(g) <= tau_max (reading R1, p 1-based commit position).
* O(U) and the drops partition U (Alg. 2: every g is either appended or
  skipped).
* Groups are contiguous runs of O(U) after the first n direct updates
  (§5.2, Fig. 7); aggregator ids <= k (Alg. 3).
These are the paper's invariants themselves; they pin nothing beyond their
own definition.
"""
from __future__ import annotations


def check_plan(plan: dict, versions: list, tau_max: int, v_init: int, k: int) -> None:
    n = len(versions)
    order = plan["order"]
    assert len(order) == plan["n_commit"]
    assert len(set(order)) == len(order)
    kept = set(order)
    for g in range(n):
        if g in kept:
            assert plan["drop_reason"][g] == 0
            assert plan["group"][g] >= 0
        else:
            assert plan["drop_reason"][g] in (1, 2)
            assert plan["group"][g] == -1
    # delay bound
    for p, g in enumerate(order, start=1):
        assert (v_init + p) - versions[g] <= tau_max, "delay bound violated"
    # commits = contiguous runs covering O(U)
    pos = 0
    groups_seen = []
    for ci, (f, c) in enumerate(zip(plan["commit_first"], plan["commit_count"])):
        assert f == pos and c >= 1
        gids = {plan["group"][order[p]] for p in range(f, f + c)}
        assert len(gids) == 1
        gid = gids.pop()
        if gid == 0:
            assert c == 1 and ci < plan["n_direct"]
        else:
            groups_seen.append(gid)
        pos += c
    assert pos == len(order)
    assert groups_seen == list(range(1, len(groups_seen) + 1))
    assert len(groups_seen) == plan["n_groups"]
    assert plan["n_groups"] <= k
    # commit times non-decreasing (R7)
    t = plan["commit_t_ns"]
    assert all(a <= b for a, b in zip(t, t[1:]))
