"""Dump planner instances (BASELINE configs at their sizes + random differential instances) as
text for scripts/planbench/planbench.cpp, with the plan the CURRENT libmlfabric.so returns as the
expected output (the speed work on mlf_plan must keep every plan bit-identical).
usage: python scripts/planbench/dump.py OUTDIR"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1907_00434_b200 import mlfabric as m  # noqa: E402
from synthgen import configs as cfgs  # noqa: E402
from tests.instances import random_instance  # noqa: E402

FIELDS = ["n_commit", "order", "drop_reason", "group", "n_direct", "n_groups", "group_node", "n_server_commits",
          "commit_first", "commit_count", "commit_t_ns", "replica_frozen", "replica_boundary_commit", "n_punted",
          "punted", "delayed_last", "t_total_ns", "n_replica_commits", "replica_commit_first",
          "replica_commit_count", "replica_commit_group", "replica_bytes"]


def canon(p):
    out = []
    for f in FIELDS:
        v = p[f]
        out.append(" ".join(map(str, v)) if isinstance(v, list) else str(v))
    return "|".join(out)


def L(x):
    return " ".join(map(str, x))


def write(f, name, n_nodes, up, down, bw, site, batch, servers, weights, aggs, replicas, raggs, v_init, tau,
          div_max, gamma, hist, carried, rmode, smode):
    f.write(f"instance {name}\n{n_nodes}\n{L(up)}\n{L(down)}\n")
    f.write(("bw " + L(bw) if bw else "bw") + "\n")
    f.write(("site " + L(site) if site else "site") + "\n")
    f.write(f"{len(batch['node'])}\n")
    for k in ("node", "size", "version", "t_avail"):
        f.write(L(batch[k]) + "\n")
    f.write(" ".join(repr(float(x)) for x in batch["norm"]) + "\n")
    f.write(L(servers) + "\n" + ("w " + L(weights) if weights else "w") + "\n")
    f.write(("a " + L(aggs)) + "\n" + ("r " + L(replicas)) + "\n" + ("ra " + L(raggs)) + "\n")
    f.write(f"{v_init} {tau} {repr(float(div_max))} {repr(float(gamma))} {repr(float(hist))} {rmode} {smode}\n")
    f.write(f"{len(carried)}\n" + L([c['node'] for c in carried]) + "\n" + L([c['size'] for c in carried]) + "\n")
    f.write(" ".join(repr(float(c['norm'])) for c in carried) + "\n")
    try:
        p = m.plan(n_nodes, up, down, batch, servers, bw=bw, site=site, aggs=aggs, replicas=replicas, raggs=raggs,
                   v_init=v_init, tau_max=tau, div_max=div_max, gamma=gamma, hist_norm=hist, carried=carried,
                   shard_weights=weights, replica_mode=rmode, sync_mode=smode)
        f.write("expect " + canon(p) + "\n")
        return p
    except m.MlfError as e:
        f.write(f"error {e.code}\n")
        return None


def dump_config(f, cid, G, iters, **kw):
    cfg = cfgs.config(cid, G=G, **kw)
    v_init = v_prev = 0
    carried = []
    for it in range(iters):
        draws = cfgs.batch_draws(cfg, it, v_init, v_prev)
        up, down, site = cfgs.network(cfg, it)
        batch = {"node": cfg["worker_node"], "size": [cfg["S"] * cfg["e"]] * cfg["W"],
                 "version": [d["version"] for d in draws], "t_avail": [d["t_avail"] for d in draws],
                 "norm": [d["norm"] for d in draws]}
        weights = [n for (_, n) in cfg["shards"]] if cfg["G"] > 1 else None
        p = write(f, f"config{cid}_G{cfg['G']}_tau{cfg['tau']}_it{it}", cfg["n_nodes"], up, down, None, site, batch,
                  cfg["servers"], weights, cfg["aggs"], cfg["replicas"], cfg["raggs"], v_init, cfg["tau"],
                  cfg["div_max"], cfg.get("gamma", 0.0), 0.0, carried, cfg.get("replica_mode", 0), 0)
        v_prev, v_init = v_init, v_init + p["n_commit"]
        if cfg["replica"]:
            items = list(carried) + [dict(node=cfg["worker_node"][g], size=cfg["S"] * cfg["e"],
                                          norm=draws[g]["norm"]) for g in p["order"]]
            carried = [items[i] for i in p["punted"]]


def main():
    out = sys.argv[1]
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "configs.txt"), "w") as f:
        dump_config(f, 2, None, 6)
        dump_config(f, 2, None, 6, tau=32)
        dump_config(f, 2, None, 4, with_replica=True, tau=32, div_max=8.0)
        dump_config(f, 3, 8, 3)
        dump_config(f, 3, 4, 2)
        dump_config(f, 4, 8, 8)
        dump_config(f, 4, 4, 3)
        dump_config(f, 5, 8, 2)
    with open(os.path.join(out, "random.txt"), "w") as f:
        for seed in (1, 2, 3, 4):
            for i in range(750):
                inst = random_instance(seed * 1000 + 7, i, max_n=8, allow_down=(i % 5 == 0))
                b = inst.batch
                batch = {k: [x[k] for x in b] for k in ("node", "size", "version", "t_avail", "norm")}
                write(f, f"rand{seed}_{i}", inst.n_nodes, inst.nic_up, inst.nic_down, inst.bw, inst.site, batch,
                      inst.servers, inst.shard_weights, inst.aggs, inst.replicas, inst.raggs, inst.v_init,
                      inst.tau_max, inst.div_max, inst.gamma, inst.hist_norm, inst.carried, inst.replica_mode,
                      inst.sync_mode)
        for i in range(40):
            inst = random_instance(555, i, max_n=48, max_servers=3)
            b = inst.batch
            batch = {k: [x[k] for x in b] for k in ("node", "size", "version", "t_avail", "norm")}
            write(f, f"large_{i}", inst.n_nodes, inst.nic_up, inst.nic_down, inst.bw, inst.site, batch,
                  inst.servers, inst.shard_weights, inst.aggs, inst.replicas, inst.raggs, inst.v_init,
                  inst.tau_max, inst.div_max, inst.gamma, inst.hist_norm, inst.carried, inst.replica_mode,
                  inst.sync_mode)


if __name__ == "__main__":
    main()
