"""The BASELINE.json workloads as concrete synthetic planner inputs (no method arithmetic).

Each builder returns a plain dict: network (nodes, NIC caps, sites), servers,
aggregators, replicas, tau_max, Div_max, model size S, dtype, worker home GPUs,
plus per-iteration batch draws (versions, t_avail, norms).
"Input recipe" states the same recipe in prose.

Sources for the shapes: SURVEY.md §8(d) table (configs 1-5), the paper's
presets (N1-N3 NIC rate draws P:1422-1430, C1-C3 stragglers P:1413-1419), its
practice tau_max = #workers (delay bound 30 with 30 workers) and the
B200 box model (site = GPU, NIC = NVLink per direction).
"""
from __future__ import annotations

import math

from . import (GBPS, SEED_ROOT, draw_rates, draw_stragglers, shuffle, stream_key, uniform01,
               KIND_MISC)

B_NV_BPS = 770_000_000_000      # measured peer copy per direction (B200_PROFILING.md), NVLink 5


def shard_bounds(S: int, G: int, align: int = 64):
    """Contiguous PS shards (App. B.2), boundaries multiples of `align` elements."""
    per = -(-S // G)
    per = -(-per // align) * align
    out = []
    for j in range(G):
        b = j * per
        if b >= S:
            out.append((S - S % align, 0))       # empty trailing shard, aligned begin
        else:
            out.append((b, min(S, b + per) - b))
    return out


def config(cid: int, *, G: int | None = None, tau: int | None = None, dtype: str = "f32",
           seed: int = SEED_ROOT, scale_S: int | None = None, gamma: float = 0.0,
           replica_mode: int = 0, div_max: float | None = None, with_replica: bool = False,
           workers: int | None = None, replica_aggs: int = 8) -> dict:
    """replica_mode 0 = mirror (R16), 1 = replica trees (NEXT-2).  with_replica adds a replica
    to config 2: a replica server with a 10 Gb/s ingress and k' = replica_aggs replica
    aggregators ("a separate k' aggregators are earmarked for the replica"; the
    paper gives no k'.  8 is the smallest k' with which the replica keeps pace with the server
    on this workload: with k' = 4 the replica's lead grows to Div_max for every Div_max >= 16,
    DESIGN.md "NEXT-2").  `workers` shrinks the worker count of configs 3-5 (tests whose
    oracle plans must be fast)."""
    d = _config(cid, G=G, tau=tau, dtype=dtype, seed=seed, scale_S=scale_S, gamma=gamma,
                with_replica=with_replica, workers=workers, replica_aggs=replica_aggs)
    d["replica_mode"] = replica_mode
    if div_max is not None:
        d["div_max"] = div_max
    return d


def _config(cid: int, *, G, tau, dtype, seed, scale_S, gamma, with_replica, workers, replica_aggs=8) -> dict:
    """Static part of config `cid` (1..5)."""
    if cid == 1:
        W, S, G = 4, 1 << 20, 1
    elif cid == 2:
        W, S, G = 32, 25_600_000, 1
    elif cid == 3:
        W, S, G = 64, 143_667_240, G or 8
    elif cid == 4:
        W, S, G = 128, 25_600_000, 8 if G is None else G
    elif cid == 5:
        W, S, G = 256, 100_000_000, 8 if G is None else G
    else:
        raise ValueError(cid)
    if scale_S is not None:
        S = scale_S
    if workers is not None and cid >= 3:
        W = workers
    d = dict(cid=cid, W=W, S=S, G=G, dtype=dtype, seed=seed, lr=0.01, div_max=math.inf, replica=False,
             preset_net=None, preset_c=None, replan_rates=False, gamma=gamma)
    d["e"] = 2 if dtype == "bf16" else 4
    d["home"] = [w * G // W for w in range(W)]            # block placement of virtual workers
    d["shards"] = shard_bounds(S, G)
    if cid == 1:
        n = W + 1
        d["servers"] = [W]
        ups = [10 * GBPS, 5 * GBPS, int(2.5 * GBPS), 1 * GBPS]
        d["nic_up"] = ups + [0]
        d["nic_down"] = ups + [10 * GBPS]
        d["site"] = None
        d["aggs"] = [0]
        d["tau"] = 2 if tau is None else tau
        d["iterations"] = 3
    elif cid == 2:
        n = W + 1
        d["servers"] = [W]
        d["preset_net"] = "N1"
        d["server_rate"] = 10 * GBPS
        d["site"] = None
        perm = shuffle(seed, list(range(W)), salt=2)
        d["aggs"] = perm[:4]
        d["tau"] = 4 if tau is None else tau
        d["replan_rates"] = True
        if with_replica:
            # a replica server on its own 10 Gb/s machine with k' replica
            # aggregators earmarked among the workers, disjoint from the server's
            n = W + 2
            d["replica"] = True
            d["replicas"] = [W + 1]
            d["raggs"] = perm[4:4 + replica_aggs]
            d["replica_rate"] = 10 * GBPS
    else:
        # box model: planner node g = GPU g.  Its NIC up/down = NVLink egress/ingress per
        # direction, shared by every virtual worker multiplexed on it (as co-located workers
        # share a host NIC); shard j's server is node j; the core
        # (NVSwitch) is congestion-free; same node = zero-time transfer.
        n = G
        d["worker_node"] = list(d["home"])
        d["servers"] = list(range(G))
        d["site"] = None
        d["nic_up"] = [B_NV_BPS] * n
        d["nic_down"] = [B_NV_BPS] * n
        d["aggs"] = shuffle(seed, list(range(G)), salt=3)      # one aggregator per GPU
        d["tau"] = W if tau is None else tau
        if cid == 4:
            d["preset_net"] = "N2"
            d["preset_c"] = "C2"
            d["replan_rates"] = True
        if cid == 5:
            d["replica"] = True
            d["replicas"] = [(j + 1) % G for j in range(G)]   # backup of shard j lives on GPU j+1
            d["raggs"] = []
            d["div_max"] = 0.0
    d["n_nodes"] = n
    d["node_rank"] = list(range(G)) if cid >= 3 else [0] * n
    d.setdefault("worker_node", list(range(W)))
    d.setdefault("replicas", [])
    d.setdefault("raggs", [])
    return d


def network(cfg: dict, iteration: int):
    """(nic_up, nic_down, site) for one iteration (NIC rates resampled when the config says so)."""
    if cfg["cid"] == 2:
        W = cfg["W"]
        ups = draw_rates(cfg["seed"], W, cfg["preset_net"], epoch=iteration, salt=1)
        downs = draw_rates(cfg["seed"], W, cfg["preset_net"], epoch=iteration, salt=2)
        if cfg.get("replica_rate"):
            return ups + [0, 0], downs + [cfg["server_rate"], cfg["replica_rate"]], None
        return ups + [0], downs + [cfg["server_rate"]], None
    if cfg["cid"] == 4:
        # N2: every NIC's NVLink share drawn from the rate set scaled to B_nv
        n = cfg["n_nodes"]
        r_up = draw_rates(cfg["seed"], n, "N2", epoch=iteration, salt=1)
        r_dn = draw_rates(cfg["seed"], n, "N2", epoch=iteration, salt=2)
        scale = B_NV_BPS // (10 * GBPS)
        return [r * scale for r in r_up], [r * scale for r in r_dn], cfg["site"]
    return cfg["nic_up"], cfg["nic_down"], cfg["site"]


def batch_draws(cfg: dict, iteration: int, v_init: int, v_prev: int):
    """Per-worker (version, t_avail_ns, norm) for one batch in which every worker pushes once.

    A worker's update was computed from the model it pulled after the previous
    batch (version v_init); a C-preset straggler is one batch late,
    so its update comes from version v_prev and it arrives later in the window
    (t_avail uniform in [0, 100 ms), the paper's batching period P:1410).
    Norms are the harness's float64 stand-in for ||u|| (same for both planners).
    """
    W = cfg["W"]
    slow = draw_stragglers(cfg["seed"], W, cfg["preset_c"], iteration) if cfg["preset_c"] else [1] * W
    key = stream_key(cfg["seed"], KIND_MISC, 77, iteration)
    out = []
    for w in range(W):
        late = slow[w] > 1
        t = int(uniform01(key, w) * 100_000_000) if late else 0
        out.append(dict(version=v_prev if late else v_init, t_avail=t,
                        norm=1.0 + uniform01(key, W + w)))
    return out
