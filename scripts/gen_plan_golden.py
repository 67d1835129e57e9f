"""Oracle plans at BASELINE sizes, stored as golden fixtures (tests/golden/plans_*.json).

Calls ONLY oracle/ (plus synthgen for the seeded inputs): the Python oracle needs minutes per
batch at these sizes (O(#U^2 * G) pure-Python water-filling), too slow for the CPU test suite,
so tests/test_planner_baseline_sizes.py compares mlf_plan with these stored oracle outputs.
usage: python scripts/gen_plan_golden.py CID G BATCHES   (writes tests/golden/plans_config{CID}_g{G}.json)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.plan import Item, Params, make_net, plan as oracle_plan  # noqa: E402
from synthgen import configs as cfgs  # noqa: E402


def main():
    cid, G, batches = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    cfg = cfgs.config(cid, G=G)
    v_init = v_prev = 0
    carried = []
    out = {"config": cid, "G": G, "seed": cfg["seed"], "tau": cfg["tau"], "div_max": cfg["div_max"],
           "generator": "scripts/gen_plan_golden.py (oracle.plan.plan only)", "batches": []}
    for it in range(batches):
        draws = cfgs.batch_draws(cfg, it, v_init, v_prev)
        up, down, site = cfgs.network(cfg, it)
        weights = [n for (_, n) in cfg["shards"]] if cfg["G"] > 1 else None
        batch = [Item(cfg["worker_node"][g], cfg["S"] * cfg["e"], d["version"], d["t_avail"], d["norm"])
                 for g, d in enumerate(draws)]
        t0 = time.time()
        p = oracle_plan(make_net(cfg["n_nodes"], up, down, None, site), batch,
                        Params(servers=cfg["servers"], aggs=cfg["aggs"], replicas=cfg["replicas"], raggs=cfg["raggs"],
                               v_init=v_init, tau_max=cfg["tau"], div_max=cfg["div_max"],
                               carried=[Item(c["node"], c["size"], 0, 0, c["norm"]) for c in carried],
                               shard_weights=weights))
        out["batches"].append({"iteration": it, "v_init": v_init, "v_prev": v_prev, "carried": carried, "plan": p,
                               "oracle_seconds": round(time.time() - t0, 1)})
        print(f"config{cid} G={G} batch {it}: {time.time() - t0:.0f} s, {p['n_commit']} committed", flush=True)
        v_prev, v_init = v_init, v_init + p["n_commit"]
        if cfg["replica"]:
            items = list(carried) + [dict(node=cfg["worker_node"][g], size=cfg["S"] * cfg["e"], norm=draws[g]["norm"])
                                     for g in p["order"]]
            carried = [items[i] for i in p["punted"]]
    path = os.path.join(ROOT, "tests", "golden", f"plans_config{cid}_g{G}.json")
    json.dump(out, open(path, "w"), indent=None, separators=(",", ":"))
    print("wrote", path)


if __name__ == "__main__":
    main()
