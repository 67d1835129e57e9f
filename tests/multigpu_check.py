"""Multi-rank parity check, run under torchrun (one process per rank).

    torchrun --nproc-per-node N tests/multigpu_check.py [--cid 3] [--S 1000003] [--steps 2]

Each rank owns PS shard `rank` (App. B.2); after every batch the shards are
compared bitwise with the oracle at sampled indices (the oracle plans the same
batch from the same inputs and applies it with numpy), and the replica mirror
(stored by rank j into rank (j+1) mod N) is checked where the plan writes it.
If there are fewer GPUs than ranks, ranks share devices (rank % device_count):
the path has no kernel that waits on another kernel, so co-resident ranks are safe.
Prints "MULTIGPU_OK <mode>" on rank 0 when every check passed.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synthgen as sg  # noqa: E402
from oracle.momentum import weighted_f32  # noqa: E402
from oracle.numerics import commit_batch, commits_from_plan, execute_plan  # noqa: E402
from oracle.plan import Item, Params, make_net, plan as oracle_plan  # noqa: E402
from paper_1907_00434_b200.multigpu import ShardedWorkload, init_dist  # noqa: E402
from synthgen import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cid", type=int, default=3)
    ap.add_argument("--S", type=int, default=1_000_003)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--modes", default="fold,tree,staged")
    ap.add_argument("--stage-mib", type=int, default=0, help="staging buffer of the staged mode (0: 4096)")
    ap.add_argument("--kernel", default="bulk")
    ap.add_argument("--gamma", type=float, default=0.0)
    ap.add_argument("--replica-mode", type=int, default=0)
    ap.add_argument("--div-max", type=float, default=None)
    ap.add_argument("--workers", type=int, default=None)
    ap.add_argument("--host", action="store_true", help="host-resident updates (the e2e path)")
    a = ap.parse_args()
    os.environ["MLF_COMMIT_IMPL"] = a.kernel
    rank, world, local, ctrl = init_dist()
    device = local % torch.cuda.device_count()
    torch.cuda.set_device(device)
    dt = sg.DTYPE_BF16 if a.dtype == "bf16" else sg.DTYPE_F32
    for mode in a.modes.split(","):
        if a.gamma and mode != "fold":
            continue                             # momentum runs in fold mode only
        cfg = configs.config(a.cid, G=world, dtype=a.dtype, scale_S=a.S, gamma=a.gamma,
                             replica_mode=a.replica_mode, div_max=a.div_max, workers=a.workers)
        sw = ShardedWorkload(cfg, rank, world, device, ctrl, mode=mode, stage_mib=a.stage_mib)
        b, n = cfg["shards"][rank]
        rng = np.random.default_rng(rank)
        idx = np.unique(np.concatenate([rng.integers(b, b + n, 5000), np.arange(b, min(b + 17, b + n)),
                                        np.arange(max(b, b + n - 17), b + n)]))
        w_ref = sg.w0_values(cfg["seed"], idx)
        h_ref = np.zeros(len(idx), np.float32)
        r_ref = w_ref.copy()                     # replica model of this shard (replica trees)
        carried_ids = []                         # (worker, iteration) of the carried items
        n_punted_total = 0
        carried = []
        v_init = v_prev = 0
        for it in range(a.steps):
            sw.fill(it)
            if a.host:
                # e2e path: the updates live in pinned host memory; every rank stages its own
                # committed ones in phase 1, peers read them in phase 2
                hosts = {}
                for w, t in sw.wl.slots.items():
                    hosts[w] = t.cpu().pin_memory()
                    sw.wl.ctx.set_update_host(w, hosts[w].data_ptr())
                sw.slots_all.zero_()
                torch.cuda.synchronize()
                sw.two_phase = True
                sw.barrier()
            pd, ms = sw.step(it)
            # oracle: same planner inputs
            up, down, site = configs.network(cfg, it)
            draws = configs.batch_draws(cfg, it, v_init, v_prev)
            batch = [Item(cfg["worker_node"][g], cfg["S"] * cfg["e"], d["version"], d["t_avail"], d["norm"])
                     for g, d in enumerate(draws)]
            prm = Params(servers=cfg["servers"], aggs=cfg["aggs"], replicas=cfg["replicas"], raggs=cfg["raggs"],
                         v_init=v_init, tau_max=cfg["tau"], div_max=cfg["div_max"], gamma=cfg["gamma"],
                         carried=[Item(c["node"], c["size"], 0, 0, c["norm"]) for c in carried],
                         shard_weights=[x for (_, x) in cfg["shards"]], replica_mode=cfg["replica_mode"])
            op = oracle_plan(make_net(cfg["n_nodes"], up, down, None, site), batch, prm)
            assert op == pd, f"rank {rank}: plan mismatch"
            operand = lambda g: sg.update_values(cfg["seed"], g, it, idx, dt)  # noqa: E731
            if a.gamma:
                w_ref, h_ref, bk = weighted_f32(w_ref, h_ref, commits_from_plan(op, operand), cfg["lr"],
                                                a.gamma, op["replica_boundary_commit"])
                backup_ref = bk[0] if bk is not None else None
                got_h = sw.wl.h.cpu().numpy()[idx - b]
                assert np.array_equal(got_h.view(np.uint32), h_ref.view(np.uint32)), f"rank {rank}: h mismatch"
            else:
                w_ref, backup_ref, _ = execute_plan(w_ref, op, operand, cfg["lr"])
            got = sw.wl.w.cpu().numpy()[idx - b]
            assert np.array_equal(got.view(np.uint32), w_ref.view(np.uint32)), f"rank {rank} {mode}: w mismatch"
            torch.cuda.synchronize()
            dist.barrier(group=ctrl)
            if cfg["replica"] and cfg["replica_mode"] == 1:
                # the replica applies its own commits over carried ++ O(U) (NEXT-2)
                items = carried_ids + [(g, it) for g in op["order"]]
                rc = [[sg.update_values(cfg["seed"], items[q][0], items[q][1], idx, dt) for q in range(f, f + k)]
                      for f, k in zip(op["replica_commit_first"], op["replica_commit_count"])]
                r_ref, _ = commit_batch(r_ref, rc, cfg["lr"])
                carried_ids = [items[i] for i in op["punted"]]
                n_punted_total += len(carried_ids)
                backup_ref = r_ref
            if op["replica_boundary_commit"] >= 0 or (cfg["replica"] and cfg["replica_mode"] == 1):
                # rank (rank+1) % world holds our mirror: gather it through the control group
                mirrors = [None] * world
                dist.all_gather_object(mirrors, (rank, sw.mirror.cpu().numpy() if sw.mirror is not None else None),
                                       group=ctrl)
                mine = dict(mirrors)[(rank + 1) % world]
                assert np.array_equal(mine[idx - b].view(np.uint32), backup_ref.view(np.uint32)), \
                    f"rank {rank} {mode}: mirror mismatch"
            if cfg["replica"]:
                items = list(carried) + [dict(node=cfg["worker_node"][g], size=cfg["S"] * cfg["e"],
                                              norm=draws[g]["norm"])
                                         for g in op["order"]]
                carried = [items[i] for i in op["punted"]]
            v_prev, v_init = v_init, v_init + op["n_commit"]
        sw.close()
        if rank == 0:
            print(f"MULTIGPU_OK {mode} cid={a.cid} world={world} S={cfg['S']} commits={op['n_commit']} "
                  f"groups={op['n_groups']} boundary={op['replica_boundary_commit']} "
                  f"punted_total={n_punted_total}", flush=True)
    dist.barrier(group=ctrl)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
