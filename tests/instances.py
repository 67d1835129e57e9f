"""Seeded random planning instances for the oracle pins and the planner differential tests.

Plain data only (node lists, byte sizes, versions, times, norms) built from
synthgen words; no planning arithmetic lives here.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import synthgen as sg

MB = 1_000_000


@dataclass
class Instance:
    n_nodes: int
    nic_up: list
    nic_down: list
    bw: list | None
    site: list | None
    batch: list                 # dicts: node, size, version, t_avail, norm
    servers: list
    aggs: list
    replicas: list
    raggs: list
    v_init: int
    tau_max: int
    div_max: float
    gamma: float
    hist_norm: float
    carried: list = field(default_factory=list)    # dicts: node, size, norm
    shard_weights: list | None = None
    replica_mode: int = 0
    sync_mode: int = 0


def random_instance(seed: int, idx: int, max_n: int = 8, max_servers: int = 2,
                    replica: bool = True, allow_pair: bool = True, allow_site: bool = True,
                    allow_down: bool = False) -> Instance:
    key = sg.stream_key(seed, sg.KIND_MISC, idx, 0xA11)
    c = [0]

    def ri(lo, hi):
        c[0] += 1
        return sg.randint(key, c[0], lo, hi)

    def rf():
        c[0] += 1
        return sg.uniform01(key, c[0])

    W = ri(1, 6)
    G = ri(1, max_servers)
    k_sep = ri(0, 2)                           # separate aggregator nodes
    has_rep = replica and ri(0, 2) > 0
    n_nodes = W + G + k_sep + (G if has_rep else 0) + (1 if has_rep else 0)
    rates = [1 * MB, 2 * MB, 3 * MB, 5 * MB, 8 * MB, 10 * MB]

    def rate():
        x = ri(0, 9)
        if x == 0:
            return 0                           # uncapped
        if allow_down and x == 9 and ri(0, 4) == 0:
            return -1                          # link down
        return rates[ri(0, len(rates) - 1)]

    nic_up = [rate() for _ in range(n_nodes)]
    nic_down = [rate() for _ in range(n_nodes)]
    servers = list(range(W, W + G))
    for s in servers:                          # servers always have a capped ingress
        nic_down[s] = rates[ri(0, len(rates) - 1)]
    bw = None
    if allow_pair and ri(0, 3) == 0:
        bw = [rates[ri(0, 5)] if ri(0, 4) == 0 else 0 for _ in range(n_nodes * n_nodes)]
    site = None
    if allow_site and ri(0, 4) == 0:
        site = [ri(0, max(1, n_nodes // 2)) for _ in range(n_nodes)]
    agg_pool = list(range(W)) + list(range(W + G, W + G + k_sep))
    k = ri(0, min(3, len(agg_pool)))
    aggs = sg.shuffle(seed ^ idx, agg_pool, salt=1)[:k]
    replicas, raggs = [], []
    if has_rep:
        base = W + G + k_sep
        replicas = list(range(base, base + G))
        kr = ri(0, 2)
        raggs = sg.shuffle(seed ^ idx, list(range(W)) + [base + G], salt=2)[:kr]
    v_init = ri(0, 50)
    tau = ri(1, 8)
    n = ri(0, max_n)
    batch = []
    for _ in range(n):
        size = ri(1, 20) * MB if ri(0, 15) else 0
        if ri(0, 6) == 0:
            size += ri(1, 999_999)            # ragged byte counts
        batch.append(dict(node=ri(0, W - 1), size=size,
                          version=v_init - ri(0, 4) if ri(0, 5) else v_init - ri(0, 12),
                          t_avail=0 if ri(0, 2) else ri(0, 3000) * MB,
                          norm=float(ri(0, 1000)) / 100.0))
    carried = []
    if has_rep:
        for _ in range(ri(0, 3)):
            carried.append(dict(node=ri(0, W - 1), size=ri(1, 10) * MB, norm=float(ri(0, 400)) / 100.0))
    dm = ri(0, 3)
    div_max = [0.0, 5.0, 20.0, math.inf][dm]
    gamma = [0.0, 0.0, 0.5, 0.9][ri(0, 3)]
    hist = float(ri(0, 300)) / 100.0
    weights = None
    if G > 1 and ri(0, 1):
        weights = [ri(1, 9) for _ in range(G)]
    return Instance(n_nodes, nic_up, nic_down, bw, site, batch, servers, aggs, replicas, raggs,
                    v_init, tau, div_max, gamma, hist, carried, weights, replica_mode=ri(0, 1),
                    sync_mode=1 if ri(0, 4) == 0 else 0)


def to_oracle(inst: Instance):
    """(Net, batch Items, Params) for oracle.plan.plan."""
    from oracle.plan import Item, Params, make_net
    net = make_net(inst.n_nodes, inst.nic_up, inst.nic_down, inst.bw, inst.site)
    batch = [Item(b["node"], b["size"], b["version"], b["t_avail"], b["norm"]) for b in inst.batch]
    carried = [Item(c["node"], c["size"], 0, 0, c["norm"]) for c in inst.carried]
    prm = Params(servers=inst.servers, aggs=inst.aggs, replicas=inst.replicas, raggs=inst.raggs,
                 v_init=inst.v_init, tau_max=inst.tau_max, div_max=inst.div_max, gamma=inst.gamma,
                 hist_norm=inst.hist_norm, carried=carried, shard_weights=inst.shard_weights,
                 replica_mode=inst.replica_mode, sync_mode=inst.sync_mode)
    return net, batch, prm
