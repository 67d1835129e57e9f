"""torchrun: per-rank device time of each batch (fold mode) and each rank's plan-relative
NVLink bytes, to see whether the slowest rank is the one the plan loads most."""
import argparse
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from benchkit.multi import plan_traffic  # noqa: E402
from paper_1907_00434_b200.multigpu import ShardedWorkload, init_dist  # noqa: E402
from synthgen import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cid", type=int, default=4)
    ap.add_argument("--steps", type=int, default=6)
    a = ap.parse_args()
    rank, world, local, ctrl = init_dist()
    torch.cuda.set_device(local)
    cfg = configs.config(a.cid, G=world)
    sw = ShardedWorkload(cfg, rank, world, local, ctrl, mode="fold")
    sw.fill(0)
    for s in range(a.steps):
        pd, ms = sw.step(s)
        allms = [None] * world
        dist.all_gather_object(allms, ms, group=ctrl)
        if rank == 0:
            tr = plan_traffic(cfg, pd, "fold")
            nin = [round(x / 1e9, 2) for x in tr["nv_in"]]
            nout = [round(x / 1e9, 2) for x in tr["nv_out"]]
            print(f"step {s}: ms {[round(x, 3) for x in allms]} nv_in GB {nin} nv_out GB {nout} "
                  f"commits {pd['n_commit']}", flush=True)
    sw.close()


if __name__ == "__main__":
    main()
