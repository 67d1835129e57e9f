"""Planner latency (mlf_plan, host C++) on a config's batches, no GPU: python scripts/plan_time.py CID G.
With LOCAL_WORLD_SIZE=G the thread pool takes this rank's share of the host's cores, as each
rank of a G-GPU run does."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_00434_b200 import mlfabric as m  # noqa: E402
from synthgen import configs as cfgs  # noqa: E402


def main():
    cid, G = int(sys.argv[1]), int(sys.argv[2])
    cfg = cfgs.config(cid, G=G)
    v_init = v_prev = 0
    ts = []
    for it in range(8):
        draws = cfgs.batch_draws(cfg, it, v_init, v_prev)
        up, down, site = cfgs.network(cfg, it)
        batch = {"node": cfg["worker_node"], "size": [cfg["S"] * cfg["e"]] * cfg["W"],
                 "version": [d["version"] for d in draws], "t_avail": [d["t_avail"] for d in draws],
                 "norm": [d["norm"] for d in draws]}
        weights = [n for (_, n) in cfg["shards"]] if cfg["G"] > 1 else None
        t0 = time.perf_counter()
        p = m.plan(cfg["n_nodes"], up, down, batch, cfg["servers"], site=site, aggs=cfg["aggs"], v_init=v_init,
                   tau_max=cfg["tau"], shard_weights=weights)
        ts.append((time.perf_counter() - t0) * 1e3)
        v_prev, v_init = v_init, v_init + len(p["order"])
    ts.sort()
    print(f"config {cid} G={G} W={cfg['W']} cores={os.cpu_count()} LOCAL_WORLD_SIZE="
          f"{os.environ.get('LOCAL_WORLD_SIZE', '-')}: median {ts[len(ts) // 2]:.2f} ms, min {ts[0]:.2f}, max {ts[-1]:.2f}")


if __name__ == "__main__":
    main()
