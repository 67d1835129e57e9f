"""O5 — bounded-divergence replication (§5.3).  TEST INFRASTRUCTURE.

Paper passages:
* §5.3: transfer a prefix of the updates to the replica "in the
  same order as O(U)"; tentative replica schedules come from Alg. 3 on the
  network that already accounts for the tentative server schedules;
  T_last = when the last tentative server transfer commits; check Div_max at
  T_last; if it holds freeze the replica transfers finished by T_last and punt
  the rest to the next batch; otherwise "delay just the last update in the
  tentative server schedule to start after completion of the earliest update in
  the replica schedule (say, a_e) such that the divergence bound is satisfied;
  all replica updates until a_e are then frozen".
* Punted updates are processed with the next batch.
* Divergence (Eq. 6-10; Eq. 11-12): with lead
  u_1..u_m since the last common state and history h0,
  w_s - w_r = (sum_{j=1..m} g^j) h0 + sum_i (sum_{j=0..m-i} g^j) u_i, which for
  m = 2 is Eq. 9's ||(g+g^2) h0 + (1+g) u1 + u2||.  The bound replaces each
  vector by its norm (triangle inequality), computable from the pushed norms
  (Table 1 push(server, update, update_norm)).

Readings: R15 Eq. 12's constants are the momentum coefficients
above (gamma = 0 -> the sum of the lead's norms; a count-based Div_max = unit
norms); divergence is checked at T_last only; the replica order is carried ++
O(U); R16 the hot path realises the replica as a MIRROR: the backup shard
receives w at the smallest server-commit boundary b whose committed set covers
the frozen set (b = 0: the pre-batch w; b = -1: no write).  Items covered by b
are reported as frozen, the rest are punted.  The delayed last server commit
keeps its duration and starts at max(its start, commit time of a_e).

Parity: pinned by Eq. 9's coefficients and the 4.61 example, soundness
||w_s - w_r|| <= bound on true vectors, Div_max = inf -> no delay, Div_max = 0 &
gamma = 0 -> lead 0 at T_last, and a hand-worked delay-last instance at three
Div_max values (tests/test_oracle_replication.py).  The delay-last *reading* (R15b)
is ours: the paper gives no formula for the re-reserved schedule.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .aggregation import chained_commit_times, plan_aggregation


def divergence_bound(lead_norms, gamma: float, hist_norm: float) -> float:
    """Upper bound on ||w_s - w_r|| for a lead of m updates (Eq. 9/12 with R15).

    Fixed evaluation order (the C++ planner does the same, -ffp-contract=off):
    pw[0] = 1, pw[j] = pw[j-1]*gamma; coef_h = sum_{j=1..m} pw[j];
    coef_i = sum_{j=0..m-i} pw[j]; D = coef_h*h0, then D += coef_i*||u_i|| for i = 1..m.
    """
    m = len(lead_norms)
    if m == 0:
        return 0.0
    pw = [1.0]
    for _ in range(m):
        pw.append(pw[-1] * gamma)
    coef_h = 0.0
    for j in range(1, m + 1):
        coef_h += pw[j]
    d = coef_h * hist_norm
    for i in range(1, m + 1):
        c = 0.0
        for j in range(0, m - i + 1):
            c += pw[j]
        d += c * lead_norms[i - 1]
    return d


@dataclass
class ReplicaResult:
    frozen: int = 0                 # items of carried ++ order covered by the mirror
    boundary: int = -1              # mirror boundary commit (R16)
    punted: list = field(default_factory=list)   # indices into carried ++ order
    delayed_last: bool = False
    t_last: int = 0                 # server T_last after any delay
    plan_frozen: int = 0            # frozen prefix before rounding up to a boundary
    bound: float = 0.0              # divergence bound at T_last for the plan's frozen prefix
    replica_case: object = None
    commits: list = field(default_factory=list)  # frozen replica commits: (first, count, group)
    replica_bytes: int = 0          # bytes the frozen replica commits deliver to the replica


def plan_replication(server_commits: list, server_times: list, carried: list, ordered: list,
                     net_after, replicas, weights, raggs, div_max: float, gamma: float,
                     hist_norm: float, mode: str = "mirror") -> ReplicaResult:
    """§5.3 on the tentative server plan.  `server_commits` are aggregation.Commit
    objects over positions of `ordered`; `server_times` their chained commit times.

    mode "mirror" (R16): the frozen prefix is rounded up to a server-commit boundary and
    realised as a mirror store of w.  mode "trees" (NEXT-2): the replica
    applies the frozen replica commits themselves — its own Alg. 3 grouping — and exactly
    the plan's frozen prefix is frozen; the rest is punted."""
    items = list(carried) + list(ordered)
    n_c = len(carried)
    rcase = plan_aggregation(items, net_after, replicas, weights, raggs)
    rtimes = chained_commit_times(rcase.commits)
    t_last = server_times[-1] if server_times else 0

    ends, acc = [], 0                               # item count through each replica commit
    for c in rcase.commits:
        acc += len(c.members)
        ends.append(acc)
    n_pre = 0
    while n_pre < len(rtimes) and rtimes[n_pre] <= t_last:
        n_pre += 1
    frozen = ends[n_pre - 1] if n_pre else 0
    n_fc = n_pre                                    # frozen replica commits
    norms = [it.norm for it in items]
    bound = divergence_bound(norms[frozen:], gamma, hist_norm)
    delayed = False
    if bound > div_max:
        a_e = None
        for c in range(n_pre, len(rcase.commits)):
            if divergence_bound(norms[ends[c]:], gamma, hist_norm) <= div_max:
                a_e = c
                break
        assert a_e is not None, "the full prefix has bound 0 <= div_max"
        frozen = ends[a_e]
        n_fc = a_e + 1
        bound = divergence_bound(norms[frozen:], gamma, hist_norm)
        if server_commits:
            delayed = True
            last = server_commits[-1].send
            shift = max(0, rtimes[a_e] - last.t_st)
            new_end = last.t_en + shift
            prev = server_times[-2] if len(server_times) > 1 else 0
            t_last = max(prev, new_end)

    rcommits, rbytes, pos = [], 0, 0
    for c in rcase.commits[:n_fc]:
        rcommits.append((pos, len(c.members), c.group))
        rbytes += max(items[p].size for p in c.members)    # a direct item, or one aggregate
        pos += len(c.members)
    if mode == "trees":
        punted = list(range(frozen, len(items)))
        return ReplicaResult(frozen, -1, punted, delayed, t_last, frozen, bound, rcase, rcommits, rbytes)

    # R16 mirror boundary
    f_o = max(0, frozen - n_c)
    if frozen == 0:
        boundary, covered = -1, 0
    elif f_o == 0:
        boundary, covered = 0, n_c
    else:
        acc, boundary = 0, None
        for ci, c in enumerate(server_commits, start=1):
            acc += len(c.members)
            if acc >= f_o:
                boundary = ci
                break
        covered = n_c + acc
    punted = list(range(covered, len(items)))
    return ReplicaResult(covered, boundary, punted, delayed, t_last, frozen, bound, rcase, rcommits, rbytes)
