"""O4 — in-network aggregation partition, Alg. 3 DetAgg + enumeration.  TEST INFRASTRUCTURE.

Paper passages:
* §5.2: partition O(U) into k+1 groups; the first group (if
  non-empty) goes directly to the server, later groups are aggregated at one
  aggregator each, members forwarded "as per O(U)", and "update to the model is
  consistent to the case with no aggregation".
* Constraint: "aggregating all updates in the i-th group ... should
  not finish later than the time when all prior i-1 groups' gradient aggregates
  are transferred to the server".
* Alg. 3: DetAgg(n): first n updates direct (t_max from their
  t_en, NetUp each); then while i <= |O(U)|: if t_en(g_i, NW, aid) > t_max:
  t_max <- t_en(a_aid, NW, S), NetUp(a_aid -> S), aid += 1, continue; else
  A(g_i) <- aid, NetUp(g_i -> aid), i += 1.  Enumerate n = 0..|U|, pick argmin.
* "We first randomly pre-assign the aggregator to use for the i-th group".
* |r| < |g3| + |g4|: an aggregate of dense same-shape updates has the
  size of one update.

Readings: R10 every DetAgg(n) starts from the batch-start network
(not Alg. 2's reserved one), which keeps group 1's schedules identical to Alg. 2
(P:1147-1149); R12 t_max is the running max of server-bound t_en; before the
first server-bound transfer (n = 0) no constraint applies, so n = 0 yields one
star group; a group that cannot admit its first update is infeasible; aid > k is
infeasible; the last group is flushed; an aggregate is available at its last
member's arrival and has size max(member sizes); aggregation compute time 0;
R13 the caller passes the pre-assigned aggregator list (group i -> agg[i-1]);
R14 ties over n -> smallest n.

Parity: pinned by the Fig. 7 caption instance (n* = 3, G2 = {u4, u5}, G3 = {u6},
total 5 s; totals 8.5, inf, inf, 5, 5, 6, 6) and the n = |U| degeneracy (equals
Alg. 2's schedules).  Optimality of the heuristic against exhaustive contiguous
partitions is PARITY UNPINNED (it is a heuristic; bruteforce.py reports the
ratio only).
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .netmodel import Net, Unschedulable, component_bytes, send


@dataclass
class Commit:
    members: list          # positions in the ordered item list, in order
    group: int             # 0 = direct to server, i >= 1 = aggregated at agg[i-1]
    send: object           # server-bound Send (direct update or aggregate)


@dataclass
class AggCase:
    n: int
    total: int | None      # None = infeasible
    commits: list = field(default_factory=list)
    member_arrivals: dict = field(default_factory=dict)   # position -> t_en at its aggregator
    member_transfers: dict = field(default_factory=dict)  # position -> its Transfer to the aggregator
    net: Net | None = None


def det_agg(n: int, items: list, net0: Net, servers, weights, aggs) -> AggCase:
    """Alg. 3 Fn DetAgg(n, O(U), NW, A) with readings R10-R12."""
    k = len(aggs)
    nw = net0.fork()
    t_max, have = 0, n > 0
    commits, arrivals, transfers = [], {}, {}
    for i in range(n):                                       # lines 3-7
        it = items[i]
        s, nw = send(nw, it.node, servers, component_bytes(it.size, weights), it.t_avail)
        t_max = max(t_max, s.t_en)
        commits.append(Commit([i], 0, s))
    aid, i = 1, n
    group, group_arr = [], []

    def flush():
        nonlocal nw, t_max, have, aid, group, group_arr
        agg = aggs[aid - 1]
        size = max(items[j].size for j in group)
        avail = max(group_arr)
        s, nw = send(nw, agg, servers, component_bytes(size, weights), avail)   # lines 11-12
        t_max = max(t_max, s.t_en)
        have = True
        commits.append(Commit(list(group), aid, s))
        aid += 1
        group, group_arr = [], []

    try:
        while i < len(items):                                # line 9
            if aid > k:
                return AggCase(n, None)
            it = items[i]
            tr = nw.transfer(it.size, it.node, aggs[aid - 1], it.t_avail)
            if have and tr.t_en > t_max:                     # line 10
                if not group:
                    return AggCase(n, None)
                flush()
                continue
            nw.reserve(tr)                                   # lines 16-18
            group.append(i)
            group_arr.append(tr.t_en)
            arrivals[i] = tr.t_en
            transfers[i] = tr
            i += 1
        if group:
            flush()
    except Unschedulable:
        return AggCase(n, None)
    return AggCase(n, t_max, commits, arrivals, transfers, nw)


def plan_aggregation(items: list, net0: Net, servers, weights, aggs) -> AggCase:
    """Alg. 3 lines 21-24: evaluate DetAgg(n) for n = 0..|O(U)|, argmin total (R14)."""
    best = None
    for n in range(len(items) + 1):
        case = det_agg(n, items, net0, servers, weights, aggs)
        if case.total is None:
            continue
        if best is None or case.total < best.total:
            best = case
    assert best is not None, "n = |U| is always feasible"
    return best


def chained_commit_times(commits: list) -> list:
    """R7: commits happen in O(U) order; commit time = max(own t_en, previous commit time)."""
    out, prev = [], 0
    for c in commits:
        prev = max(prev, c.send.t_en)
        out.append(prev)
    return out
