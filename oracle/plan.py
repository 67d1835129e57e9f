"""The per-batch planning pipeline: ordering -> aggregation -> replication.  TEST INFRASTRUCTURE.

Mirrors the integer outputs of the C-ABI call mlf_plan (include/mlfabric.h) and
follows §5's decomposition: "We first determine ordering ... Second,
given ordering, we determine the forwarding/aggregation strategy ... Third ...
replica transfers", each step implemented step by step in oracle/ordering.py,
oracle/aggregation.py and oracle/replication.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

from .aggregation import chained_commit_times, plan_aggregation
from .netmodel import Net, component_bytes
from .ordering import Item, OrderResult, order_final
from .replication import plan_replication

# status codes (same numbering as mlf_status, defined independently)
OK, E_INVALID, E_STATE, E_CUDA, E_UNSCHEDULABLE, E_CAPACITY = 0, 1, 2, 3, 4, 5


class PlanError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


@dataclass
class Params:
    servers: list
    aggs: list = field(default_factory=list)
    replicas: list = field(default_factory=list)       # [] = no replica; else one node per shard
    raggs: list = field(default_factory=list)
    v_init: int = 0
    tau_max: int = 1
    div_max: float = math.inf
    gamma: float = 0.0
    hist_norm: float = 0.0
    carried: list = field(default_factory=list)        # Items (node, size, norm), in order
    shard_weights: list | None = None                  # None = equal weights
    replica_mode: int = 0                              # 0 mirror (R16), 1 replica trees (NEXT-2)
    sync_mode: int = 0                                 # 1: MLfabric-S, Alg. 3 over the list (NEXT-3)


def validate(net: Net, batch: list, prm: Params) -> list:
    n = net.n_nodes
    if n < 1:
        raise PlanError(E_INVALID, "n_nodes < 1")
    if len(net.nic_up) != n or len(net.nic_down) != n:
        raise PlanError(E_INVALID, "nic arrays")
    nodes = [it.node for it in batch] + [it.node for it in prm.carried]
    nodes += list(prm.servers) + list(prm.aggs) + list(prm.replicas) + list(prm.raggs)
    if any(not (0 <= x < n) for x in nodes):
        raise PlanError(E_INVALID, "node id out of range")
    if len(prm.servers) < 1:
        raise PlanError(E_INVALID, "no server")
    if prm.replicas and len(prm.replicas) != len(prm.servers):
        raise PlanError(E_INVALID, "replica count must equal server count")
    if prm.replica_mode not in (0, 1):
        raise PlanError(E_INVALID, "replica_mode")
    if prm.sync_mode not in (0, 1):
        raise PlanError(E_INVALID, "sync_mode")
    if prm.tau_max < 0 or not (prm.div_max >= 0) or not (0.0 <= prm.gamma < 1.0):
        raise PlanError(E_INVALID, "tau_max / div_max / gamma")
    if not (prm.hist_norm >= 0 and math.isfinite(prm.hist_norm)):
        raise PlanError(E_INVALID, "hist_norm")
    for it in list(batch) + list(prm.carried):
        if it.size < 0 or it.t_avail < 0 or not (it.norm >= 0 and math.isfinite(it.norm)):
            raise PlanError(E_INVALID, "bad update descriptor")
    w = prm.shard_weights or [1] * len(prm.servers)
    if len(w) != len(prm.servers) or any(x <= 0 for x in w):
        raise PlanError(E_INVALID, "shard weights")
    # unschedulable: a component with bytes whose path is down forever (R9)
    for it in batch:
        for s, b in zip(prm.servers, component_bytes(it.size, w)):
            if b > 0 and net.dead(it.node, s):
                raise PlanError(E_UNSCHEDULABLE, "update path to a server is down")
    if prm.replicas:
        for it in list(prm.carried) + list(batch):
            for r, b in zip(prm.replicas, component_bytes(it.size, w)):
                if b > 0 and net.dead(it.node, r):
                    raise PlanError(E_UNSCHEDULABLE, "update path to a replica is down")
    return w


def plan(net: Net, batch: list, prm: Params) -> dict:
    """Compute the batch plan; returns the integer outputs of mlf_plan as a dict."""
    w = validate(net, batch, prm)
    n = len(batch)
    # 1. ordering (Alg. 2, App. B.2); synchronous mode: "update ordering
    #    does not apply ... aggregation here starts with a list of updates" — the batch in
    #    submission order, nothing dropped (R22)
    if prm.sync_mode:
        ores = OrderResult(list(range(n)), [0] * n)
    else:
        ores = order_final(net, batch, prm.servers, w, prm.tau_max, prm.v_init)
    order = ores.order
    ordered_items = [batch[g] for g in order]
    # 2. aggregation (Alg. 3) on the batch-start network (R10)
    case = plan_aggregation(ordered_items, net, prm.servers, w, prm.aggs)
    times = chained_commit_times(case.commits)
    group = [-1] * n
    commit_first, commit_count = [], []
    pos = 0
    for c in case.commits:
        commit_first.append(pos)
        commit_count.append(len(c.members))
        for p in c.members:
            assert p == pos
            group[order[p]] = c.group
            pos += 1
    n_groups = sum(1 for c in case.commits if c.group > 0)
    out = {
        "n_commit": len(order), "order": list(order), "drop_reason": list(ores.drop_reason),
        "group": group, "n_direct": case.n, "n_groups": n_groups,
        "group_node": [prm.aggs[i] for i in range(n_groups)],
        "n_server_commits": len(case.commits), "commit_first": commit_first,
        "commit_count": commit_count, "commit_t_ns": list(times),
        "replica_frozen": 0, "replica_boundary_commit": -1, "n_punted": 0, "punted": [],
        "delayed_last": 0, "t_total_ns": times[-1] if times else 0,
        "n_replica_commits": 0, "replica_commit_first": [], "replica_commit_count": [],
        "replica_commit_group": [], "replica_bytes": 0, "sync_mode": int(prm.sync_mode),
    }
    # 3. replication (§5.3) on the network after the server plan's reservations
    if prm.replicas:
        rres = plan_replication(case.commits, times, prm.carried, ordered_items, case.net,
                                prm.replicas, w, prm.raggs, prm.div_max, prm.gamma, prm.hist_norm,
                                mode="trees" if prm.replica_mode == 1 else "mirror")
        out["n_replica_commits"] = len(rres.commits)
        out["replica_commit_first"] = [c[0] for c in rres.commits]
        out["replica_commit_count"] = [c[1] for c in rres.commits]
        out["replica_commit_group"] = [c[2] for c in rres.commits]
        out["replica_bytes"] = rres.replica_bytes
        out["replica_frozen"] = rres.frozen
        out["replica_boundary_commit"] = rres.boundary
        out["punted"] = rres.punted
        out["n_punted"] = len(rres.punted)
        out["delayed_last"] = int(rres.delayed_last)
        if rres.delayed_last:
            out["commit_t_ns"][-1] = rres.t_last
        out["t_total_ns"] = rres.t_last
    return out


def make_net(n_nodes, nic_up, nic_down, bw=None, site=None) -> Net:
    return Net(n_nodes, list(nic_up), list(nic_down), list(bw) if bw is not None else None,
               list(site) if site is not None else None)


__all__ = ["Item", "Params", "PlanError", "plan", "make_net", "validate"]
