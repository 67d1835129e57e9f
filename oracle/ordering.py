"""O3 — update ordering: deadlines, Alg. 1 ShrtUp, Alg. 2 look-ahead drops.  TEST INFRASTRUCTURE.

Paper passages:
* Alg. 1: repeatedly pick g* = argmin_g t_en(g, NW, S), append to
  O(U), NW <- NetUp(NW, g*, S).
* Deadlines (§5.1.2): dl(g) := v(g) + tau_max - v_init; "in iteration
  i if there exists an unscheduled g in U such that dl(g) = i, then we pick g ...
  otherwise we greedily pick the update with the least transfer time".
* Alg. 2 + §5.1.3: after picking g*, look ahead to
  g° = ShrtDline(i+1, U-P, NetUp(NW, g*, S)); if t_en(g*, NW, S) >
  t_en(g°, NetUp(NW, g*, S), S) drop g* ("drop the update g1 at the worker
  itself").
* App. B.2: with |S| shards, t_en(g) = max_j t_en(g^j), all
  components reserved together.

Readings: R1 delay(g) = (v_init + p) - v(g), p = 1-based commit
position, so dl(g) = p is the last legal slot; R3 drops consume no position
(the look-ahead is at p+1); R4 several updates due at p -> the due set's argmin
t_en; any g with dl(g) < p is dropped as expired (includes dl <= 0 at batch
start); R5 the look-ahead is applied to every pick, strict '>', and is skipped
when no candidate with dl >= p+1 remains; R6 ties in t_en -> lowest batch index;
R11 components reserved sequentially in shard order.

Parity: pinned by the Fig. 6 instance (g1 dropped, O(U) = [g2], 0.99 s), the SJF
example of S:156, single-bottleneck SPT optimality vs brute force (1||sum C_j),
the tau = 4 / 6-update instance and the delay-bound invariant on >= 1000 random
batches (tests/test_oracle_ordering.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .netmodel import Net, component_bytes, send

DROP_KEPT, DROP_EXPIRED, DROP_LOOKAHEAD = 0, 1, 2


@dataclass
class Item:
    """One update request (Table 1 push + arrival time), or one carried replica item."""
    node: int
    size: int
    version: int = 0
    t_avail: int = 0
    norm: float = 0.0


@dataclass
class OrderResult:
    order: list                     # batch indices, commit order O(U)
    drop_reason: list               # per batch index: 0 kept, 1 expired, 2 look-ahead
    sends: dict = field(default_factory=dict)   # batch index -> Send (server-bound, Alg. 2 schedule)
    net: Net | None = None          # NW after all reservations


def deadline(version: int, tau_max: int, v_init: int) -> int:
    """dl(g) := v(g) + tau_max - v_init."""
    return version + tau_max - v_init


def t_en_server(net: Net, it: Item, servers, weights):
    """t_en(g, NW, S) for all shard components (App. B.2) and NetUp(NW, g, S)."""
    return send(net, it.node, servers, component_bytes(it.size, weights), it.t_avail)


def shrt_dline(pos: int, cands: list, net: Net, batch: list, dl: list, servers, weights):
    """ShrtDline(it, UU, NW): a g with dl(g) = it if one exists (the due set's
    argmin t_en, R4), otherwise ShrtUp(UU, NW) = argmin t_en (Alg. 1 line 3).
    Returns (g, Send, NetUp(NW, g))."""
    due = [g for g in cands if dl[g] == pos]
    pool = due if due else cands
    best = None
    for g in pool:                                   # batch-index order: ties -> lowest (R6)
        s, nw = t_en_server(net, batch[g], servers, weights)
        if best is None or s.t_en < best[1].t_en:
            best = (g, s, nw)
    return best


def order_final(net: Net, batch: list, servers, weights, tau_max: int, v_init: int) -> OrderResult:
    """Alg. 2 (final update ordering) with readings R1-R6."""
    n = len(batch)
    dl = [deadline(it.version, tau_max, v_init) for it in batch]
    unprocessed = list(range(n))
    reason = [DROP_KEPT] * n
    order, sends = [], {}
    nw = net.fork()
    p = 1
    while True:
        for g in list(unprocessed):                   # R4: missed deadlines expire
            if dl[g] < p:
                reason[g] = DROP_EXPIRED
                unprocessed.remove(g)
        if not unprocessed:
            break
        g_star, s_star, nw_star = shrt_dline(p, unprocessed, nw, batch, dl, servers, weights)
        cands = [g for g in unprocessed if g != g_star and dl[g] >= p + 1]
        if cands:
            _, s_next, _ = shrt_dline(p + 1, cands, nw_star, batch, dl, servers, weights)
            if s_star.t_en > s_next.t_en:             # Alg. 2 line 10: drop g*
                reason[g_star] = DROP_LOOKAHEAD
                unprocessed.remove(g_star)
                continue
        order.append(g_star)
        sends[g_star] = s_star
        nw = nw_star
        unprocessed.remove(g_star)
        p += 1
    return OrderResult(order, reason, sends, nw)


def order_sjf(net: Net, batch: list, servers, weights) -> OrderResult:
    """Alg. 1 alone (no deadlines, no drops)."""
    n = len(batch)
    unprocessed = list(range(n))
    order, sends = [], {}
    nw = net.fork()
    while unprocessed:
        best = None
        for g in unprocessed:
            s, nw2 = t_en_server(nw, batch[g], servers, weights)
            if best is None or s.t_en < best[1].t_en:
                best = (g, s, nw2)
        g, s, nw = best
        order.append(g)
        sends[g] = s
        unprocessed.remove(g)
    return OrderResult(order, [DROP_KEPT] * n, sends, nw)
