#!/usr/bin/env python
"""Replica traffic vs Div_max (the paper's Fig. 11 experiment) on the planner.

Runs mlf_plan (replica_mode = 1, replica trees) over a synthetic stream of batches of
config 2 with a replica (32 workers, N1 NIC rates, 10 Gb/s server and replica machines,
k = 4 server and k' = 4 replica aggregators) with a count-based divergence bound (every
update norm = 1, gamma = 0: Div_max = the number of updates the replica may lag, as the
paper measures it).  Reports replica bytes per committed update and the savings
factor against sending every update to the replica on its own (1.0 = no aggregation).
Host-only (the planner); the same plans drive the GPU path in tests/test_gpu_replica_trees.py.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1907_00434_b200 import mlfabric as m  # noqa: E402
from synthgen import configs  # noqa: E402


def run(div_max: float, batches: int, tau: int, kr: int):
    cfg = configs.config(2, tau=tau, with_replica=True, replica_mode=1, div_max=div_max, replica_aggs=kr)
    S_bytes = cfg["S"] * cfg["e"]
    carried, v, vp = [], 0, 0
    rbytes = commits = 0
    lead_max = 0
    for it in range(batches):
        up, down, _ = configs.network(cfg, it)
        draws = configs.batch_draws(cfg, it, v, vp)
        batch = [dict(node=g, size=S_bytes, version=d["version"], t_avail=d["t_avail"], norm=1.0)
                 for g, d in enumerate(draws)]
        p = m.plan(cfg["n_nodes"], up, down, batch, cfg["servers"], aggs=cfg["aggs"], replicas=cfg["replicas"],
                   raggs=cfg["raggs"], v_init=v, tau_max=cfg["tau"], div_max=div_max, carried=carried,
                   replica_mode=1)
        items = carried + [dict(node=g, size=S_bytes, norm=1.0) for g in p["order"]]
        carried = [items[i] for i in p["punted"]]
        lead_max = max(lead_max, len(carried))
        rbytes += p["replica_bytes"]
        commits += p["n_commit"]
        vp, v = v, v + p["n_commit"]
    per_update = rbytes / (commits * S_bytes)
    return {"k_replica_aggs": kr, "div_max": div_max, "replica_bytes_per_update": round(per_update, 4),
            "savings_vs_unaggregated": round(1.0 / per_update, 3), "max_lead": lead_max,
            "final_lead": len(carried)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=40)
    ap.add_argument("--tau", type=int, default=32)
    ap.add_argument("--out", default=None)
    ap.add_argument("--kr", type=int, nargs="+", default=[8, 4], help="replica aggregators k' (P:1178-1179)")
    a = ap.parse_args()
    rows = [run(d, a.batches, a.tau, kr) for kr in a.kr
            for d in (0.0, 1.0, 2.0, 4.0, 8.0, 16.0, 30.0, 60.0, 120.0, 300.0, 600.0)]
    for r in rows:
        print(json.dumps(r))
    if a.out:
        json.dump({"experiment": "replica bytes vs Div_max (Fig. 11 analogue), config 2 + replica, k' in " + str(a.kr) + ", "
                                 f"{a.batches} batches, tau {a.tau}, count-based Div_max", "rows": rows},
                  open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
