"""O8 — exhaustive search on tiny batches (App. B.1 objectives).  TEST INFRASTRUCTURE.

App. B.1 states the joint problem as an ILP over rates r_g(t) and
next hops dst(g) in {S} u A, with
  obj_sync  = max( max_{dst(g)=S} t_en(g), max_a t_en(a) )                (Eq. 19)
  obj_async = (sum_{dst(g)=S} t_en(g) + sum_a m(a) t_en(a)) / |U|          (Eq. 20)
and calls it intractable.  Here it is enumerated for <= 5 updates
under the same greedy water-filling transfer semantics as netmodel (transfers
are reserved one after another; no arbitrary rate control) — the restriction
SPEC.md S:372 also makes, stated in DESIGN.md.

* best_order_sum / best_order_sum_recursive: minimum of sum t_en over all
  permutations of a batch sent directly to the server (two independent
  enumerators; they must agree).
* partition totals: every split "first n direct, the rest cut into <= k
  contiguous groups, group i at agg[i-1]" evaluated with Alg. 3's reservation
  sequence but WITHOUT its greedy admission rule; the minimum bounds Alg. 3's
  result from below.  Heuristic-vs-optimum ratios are reported, not asserted
  (PARITY UNPINNED: the paper makes no optimality claim for Alg. 3).
"""
from __future__ import annotations

import itertools

from .netmodel import Unschedulable, component_bytes, send


def order_t_ens(net, batch, servers, weights, perm) -> list:
    nw = net.fork()
    out = []
    for g in perm:
        it = batch[g]
        s, nw = send(nw, it.node, servers, component_bytes(it.size, weights), it.t_avail)
        out.append(s.t_en)
    return out


def best_order_sum(net, batch, servers, weights):
    best = None
    for perm in itertools.permutations(range(len(batch))):
        tot = sum(order_t_ens(net, batch, servers, weights, perm))
        if best is None or tot < best[0]:
            best = (tot, perm)
    return best


def best_order_sum_recursive(net, batch, servers, weights):
    """Independent DFS over permutations (branch on the next update to send)."""
    n = len(batch)
    best = [None]

    def dfs(nw, remaining, acc):
        if not remaining:
            if best[0] is None or acc < best[0]:
                best[0] = acc
            return
        for g in sorted(remaining):
            it = batch[g]
            sizes = component_bytes(it.size, weights)
            s, nw2 = send(nw, it.node, servers, sizes, it.t_avail)
            dfs(nw2, remaining - {g}, acc + s.t_en)

    dfs(net.fork(), frozenset(range(n)), 0)
    return best[0]


def eval_partition(items, net0, servers, weights, aggs, n: int, sizes: tuple):
    """Alg. 3's reservation sequence for a fixed partition: n direct, then groups
    of the given sizes at agg[0], agg[1], ...  Returns (obj_sync, obj_async_sum)
    or None if unschedulable."""
    nw = net0.fork()
    sync, asum = 0, 0
    try:
        for i in range(n):
            it = items[i]
            s, nw = send(nw, it.node, servers, component_bytes(it.size, weights), it.t_avail)
            sync = max(sync, s.t_en)
            asum += s.t_en
        pos = n
        for gi, m in enumerate(sizes):
            agg = aggs[gi]
            arr = []
            for j in range(pos, pos + m):
                tr = nw.transfer(items[j].size, items[j].node, agg, items[j].t_avail)
                nw.reserve(tr)
                arr.append(tr.t_en)
            size = max(items[j].size for j in range(pos, pos + m))
            s, nw = send(nw, agg, servers, component_bytes(size, weights), max(arr))
            sync = max(sync, s.t_en)
            asum += m * s.t_en
            pos += m
    except Unschedulable:
        return None
    return sync, asum


def compositions(total: int, max_parts: int):
    """All ordered tuples of positive ints summing to `total` with <= max_parts parts."""
    if total == 0:
        yield ()
        return
    for parts in range(1, max_parts + 1):
        for cuts in itertools.combinations(range(1, total), parts - 1):
            b = (0,) + cuts + (total,)
            yield tuple(b[i + 1] - b[i] for i in range(parts))


def best_partition(items, net0, servers, weights, aggs):
    """Minimum obj_sync over every contiguous partition with <= k groups."""
    best = None
    for n in range(len(items) + 1):
        for sizes in compositions(len(items) - n, len(aggs)):
            r = eval_partition(items, net0, servers, weights, aggs, n, sizes)
            if r is None:
                continue
            if best is None or r[0] < best[0]:
                best = (r[0], n, sizes)
    return best
