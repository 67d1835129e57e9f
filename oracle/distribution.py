"""NEXT-4 — model distribution trees for pulls (App. B.3).  TEST INFRASTRUCTURE.

Paper passage (App. B.3): "if each request for the model is responded
to individually then the down-link at the server will become the bottleneck ... we
use a distribution tree ... requests are batched and responded with same version of
model ... For a batch of requests, k° distributors are earmarked.  Mapping of workers
to distributors is done using a variant of alg. 3 obtained by replacing t_en()s as the
times taken to transfer the model from server-to-distributor and distributor-to-worker.
Once the partitioning is determined, we first transfer the model from the server to the
k°-th distributor and then proceed backwards.  The workers in the first group receive
the model directly from the server."

Readings (R23-R25):
* R23 the "variant of Alg. 3" is Alg. 3 on the time-reversed problem.  Capacities are
  constant within a batch (R9), so a schedule on the TRANSPOSED network (every node's
  up and down caps swapped, pair caps (i, j) <-> (j, i)) that ends at T maps to a
  feasible schedule on the real network by t -> T - t with every transfer reversed:
  a worker's transfer to its aggregator becomes the distributor's transfer to the
  worker, the aggregate's transfer to the servers becomes the servers' transfer of the
  model to the distributor, and "members before the aggregate" becomes "distributor
  before its members".  The last group's distributor is served first and the direct
  group last — "first ... the k°-th distributor and then proceed backwards".
* R24 the request order O is Alg. 1's SJF order (no deadlines: a pull has no
  staleness bound) of the server -> worker transfers, i.e. SJF on the transposed
  network; ties -> lowest request index (R6).  Requests are batched at time 0 (the
  batch boundary, R19), every transfer carries the whole model (model_bytes), split
  into shard components for server transfers (App. B.2, R11).
* R25 a request's model arrival is T - t_st of its reversed transfer (for the direct
  group: the earliest component); a distributor holds the model at T - t_st of its
  reversed aggregate send.

Parity: pinned by closed forms (tests/test_oracle_distribution.py: the one-distributor
star, k° = 0 = Alg. 1's makespan on the transposed network), by symmetry (on a network
with up = down caps and symmetric pairs, the plan equals Alg. 3's aggregation plan of
the same requests), and by feasibility of the real-time schedule it returns (every real
link's summed rate <= capacity at all times, distributor before members, conservation).
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .aggregation import plan_aggregation
from .netmodel import Net
from .ordering import Item, order_sjf


def transpose(net: Net) -> Net:
    """Every node's up and down caps swapped, pair caps transposed (R23)."""
    n = net.n_nodes
    bw = None if net.bw is None else [net.bw[j * n + i] for i in range(n) for j in range(n)]
    return Net(n, list(net.nic_down), list(net.nic_up), bw, list(net.site) if net.site is not None else None)


@dataclass
class DistPlan:
    order: list            # request indices in O (R24)
    group: list            # per request: 0 = direct from the servers, i = via distributor i
    n_direct: int
    group_node: list       # distributor node of group i (1-based i -> [i-1])
    t_total: int           # T: every request has the model by T
    t_recv: list           # per request: model arrival (real time, R25)
    t_start: list          # per request: start of its last hop (real time)
    t_dist: list           # per group: model arrival at its distributor
    schedule: list = field(default_factory=list)   # real transfers: (src, dst, size, t_st, t_en, segs)


def _reverse(tr, T: int):
    """A transposed-network transfer as the real transfer it stands for (R23)."""
    segs = tuple((T - b, T - a, r) for (a, b, r) in reversed(tr.segs))
    return (tr.dst, tr.src, tr.size, T - tr.t_en, T - tr.t_st, segs)


def plan_distribution(net: Net, request_nodes: list, model_bytes: int, servers: list, weights, dists: list) -> DistPlan:
    """Alg. 3 variant for a batch of pull requests (App. B.3, readings R23-R25)."""
    w = list(weights) if weights is not None else [1] * len(servers)
    items = [Item(node, model_bytes) for node in request_nodes]
    nt = transpose(net)
    order = order_sjf(nt, items, servers, w).order
    ordered = [items[g] for g in order]
    case = plan_aggregation(ordered, nt, servers, w, dists)
    T = case.total
    n = len(request_nodes)
    group, t_recv, t_start = [-1] * n, [None] * n, [None] * n
    t_dist, schedule = [], []
    for c in case.commits:
        if c.group == 0:
            (p,) = c.members
            group[order[p]] = 0
            t_recv[order[p]] = T - c.send.t_st
            t_start[order[p]] = T - c.send.t_en
        else:
            t_dist.append(T - c.send.t_st)
            for p in c.members:
                group[order[p]] = c.group
                t_recv[order[p]] = T - case.member_transfers[p].t_st
                t_start[order[p]] = T - case.member_transfers[p].t_en
                schedule.append(_reverse(case.member_transfers[p], T))
        for part in c.send.parts:
            schedule.append(_reverse(part, T))
    n_groups = len(t_dist)
    return DistPlan(list(order), group, case.n, list(dists[:n_groups]), T, t_recv, t_start, t_dist, schedule)


__all__ = ["DistPlan", "plan_distribution", "transpose"]
