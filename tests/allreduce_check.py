"""AllReduce via push/get (NEXT-3) parity, run under torchrun (one process per rank).

    torchrun --nproc-per-node N tests/allreduce_check.py [--S 1000003] [--workers W]

Every rank ends with the full sum of all updates; it must equal, bit for bit at sampled
indices, the oracle's sum in the synchronous plan's fold order (the oracle plans the same
list with sync_mode = 1 and folds with oracle/numerics.commit_batch from zero, lr = -1).
Prints "ALLREDUCE_OK" on rank 0.
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
from oracle.numerics import commit_batch, commits_from_plan  # noqa: E402
from oracle.plan import Item, Params, make_net, plan as oracle_plan  # noqa: E402
from paper_1907_00434_b200.allreduce import MlfAllReduce, allreduce_config  # noqa: E402
from paper_1907_00434_b200.multigpu import init_dist  # noqa: E402
from synthgen import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--S", type=int, default=1_000_003)
    ap.add_argument("--workers", type=int, default=None)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--multicast", action="store_true", help="also the NVLS multicast fused get")
    a = ap.parse_args()
    rank, world, local, ctrl = init_dist()
    device = local % torch.cuda.device_count()
    torch.cuda.set_device(device)
    cfg = allreduce_config(a.S, world, workers=a.workers)
    rng = np.random.default_rng(7)
    idx = np.unique(np.concatenate([rng.integers(0, cfg["S"], 8000), np.arange(cfg["S"] - 11, cfg["S"])]))
    for fused in (True, False):
        check(cfg, rank, world, device, ctrl, idx, a.steps, fused)
    if a.multicast:
        check(cfg, rank, world, device, ctrl, idx, a.steps, True, multicast=True)
    if rank == 0:
        print(f"ALLREDUCE_OK world={world} S={cfg['S']} workers={cfg['W']} multicast={a.multicast}", flush=True)
    dist.barrier(group=ctrl)
    dist.destroy_process_group()


def check(cfg, rank, world, device, ctrl, idx, steps, fused, multicast=False):
    ar = MlfAllReduce(cfg, rank, world, device, ctrl, fused=fused, multicast=multicast)
    v = vp = 0
    for it in range(steps):
        ar.sw.fill(it)
        pd, _, _, _ = ar.run(it)
        up, down, site = configs.network(cfg, it)
        draws = configs.batch_draws(cfg, it, v, vp)
        batch = [Item(cfg["worker_node"][g], cfg["S"] * 4, d["version"], d["t_avail"], d["norm"])
                 for g, d in enumerate(draws)]
        op = oracle_plan(make_net(cfg["n_nodes"], up, down, None, site), batch,
                         Params(servers=cfg["servers"], aggs=cfg["aggs"], v_init=v, tau_max=cfg["tau"],
                                shard_weights=[n for (_, n) in cfg["shards"]], sync_mode=1))
        assert op == pd, "plan mismatch"
        ref, _ = commit_batch(np.zeros(len(idx), np.float32),
                              commits_from_plan(op, lambda g: sg.update_values(cfg["seed"], g, it, idx)), -1.0)
        got = ar.out.cpu().numpy()[idx]
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), \
            f"rank {rank}: allreduce mismatch (fused={fused}, multicast={multicast})"
        vp, v = v, v + 1
    ar.close()


if __name__ == "__main__":
    main()
