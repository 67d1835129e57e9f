"""Debug: staged vs fold on the same batch, full shard compared bitwise (torchrun, N ranks)."""
import argparse
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1907_00434_b200.multigpu import ShardedWorkload, init_dist  # noqa: E402
from synthgen import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--S", type=int, default=143_667_240)
    ap.add_argument("--stage-mib", type=int, default=0)
    ap.add_argument("--workers", type=int, default=None)
    a = ap.parse_args()
    rank, world, local, ctrl = init_dist()
    device = local % torch.cuda.device_count()
    torch.cuda.set_device(device)
    res = {}
    for mode in ("fold", "staged"):
        cfg = configs.config(3, G=world, scale_S=a.S, workers=a.workers)
        sw = ShardedWorkload(cfg, rank, world, device, ctrl, mode=mode, stage_mib=a.stage_mib)
        sw.fill(0)
        sw.step(0)
        res[mode] = sw.wl.w.clone()
        sw.close()
    bad = (res["fold"].view(torch.int32) != res["staged"].view(torch.int32)).nonzero().flatten()
    n = res["fold"].numel()
    msg = f"rank {rank} n={n} mismatches={bad.numel()}"
    if bad.numel():
        msg += f" first={int(bad[0])} last={int(bad[-1])}"
        # histogram over 16 bins of the shard
        h = torch.bincount((bad * 16 // n), minlength=16).tolist()
        msg += f" bins={h}"
        sel = bad[:: max(1, bad.numel() // 6)][:6]
        f, s = res["fold"][sel].tolist(), res["staged"][sel].tolist()
        msg += " samples=" + " ".join(f"{int(i)}:{a:.6e}/{b:.6e}" for i, a, b in zip(sel.tolist(), f, s))
        # runs: how long are the contiguous mismatch stretches
        gaps = (bad[1:] - bad[:-1] != 1).nonzero().flatten()
        msg += f" runs={gaps.numel() + 1}"
    print(msg, flush=True)
    dist.barrier(group=ctrl)


if __name__ == "__main__":
    main()
