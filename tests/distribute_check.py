"""NEXT-4 multi-rank check (torchrun, one process per rank): model distribution trees.

    torchrun --nproc-per-node N tests/distribute_check.py [--S 1000003]

Every rank's view must equal the whole model (w0 drawn by the oracle's generator,
synthgen) bit for bit after mlf_distribute_phase, for (a) the uniform box (Alg. 3 picks
direct pulls), (b) a box whose GPU 0 egress is degraded (the plan routes through
distributors) and (c) a plan with every request in one distributor group.  Each rank's
reported source must follow the plan (earliest hop).  Prints "DISTRIBUTE_OK" on rank 0.
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
from oracle.distribution import plan_distribution as oracle_dist  # noqa: E402
from oracle.netmodel import Net  # noqa: E402
from paper_1907_00434_b200.multigpu import DistributionRun, init_dist  # noqa: E402

B = 770_000_000_000


def expected_source(dplan, reqs, rank):
    """Earliest hop of `rank`'s view in the plan (header: mlf_distribute_phase)."""
    used = {g for g in dplan["group"] if g > 0}
    if any(dplan["group_node"][g - 1] == rank for g in used):
        return -1
    src = None
    for i in dplan["order"]:
        if reqs[i] != rank:
            continue
        g = dplan["group"][i]
        if g == 0:
            return -1
        if src is None:
            src = dplan["group_node"][g - 1]
    if src == rank:
        return -1
    return -2 if src is None else src


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--S", type=int, default=1_000_003)
    a = ap.parse_args()
    rank, world, local, ctrl = init_dist()
    device = local % torch.cuda.device_count()
    torch.cuda.set_device(device)
    run = DistributionRun(a.S, rank, world, device, ctrl)
    want = sg.w0_values(sg.SEED_ROOT, np.arange(a.S)).astype(np.float32)
    G = world
    reqs = [g for g in range(G) for _ in range(8)]
    cases = {
        "uniform": ([B] * G, [B] * G, list(range(G))[::-1]),
        "degraded0": ([B // 10] + [B] * (G - 1), [B] * G, [(j + 1) % G for j in range(G)]),
    }
    for name, (up, down, dists) in cases.items():
        dp = run.plan(up, down, reqs, dists)
        # the C++ plan equals the oracle's on the same box network
        od = oracle_dist(Net(G, up, down, None, list(range(G))), reqs, a.S * 4, list(range(G)),
                         [max(x, 1) for (_, x) in run.shards], dists)
        assert (od.order, od.group, od.group_node, od.t_total) == (dp["order"], dp["group"], dp["group_node"],
                                                                    dp["t_total_ns"]), name
        run.view.fill_(float("nan"))
        src, ms = run.run(dp, reqs)
        assert src == expected_source(dp, reqs, rank), (name, rank, src)
        got = run.view[:a.S].cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), f"rank {rank} {name}: view mismatch"
        if rank == 0:
            print(f"case {name}: groups={dp['n_groups']} n_direct={dp['n_direct']} ms={ms:.3f}", flush=True)
    if G > 1:
        # a hand-made plan: every request through distributor 1 (phase-2 copies on every other GPU)
        dp = {"order": list(range(len(reqs))), "group": [1] * len(reqs), "n_direct": 0, "n_groups": 1,
              "group_node": [1], "t_total_ns": 0}
        run.view.fill_(float("nan"))
        src, _ = run.run(dp, reqs)
        assert src == (-1 if rank == 1 else 1), (rank, src)
        got = run.view[:a.S].cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), f"rank {rank} star: view mismatch"
    run.close()
    if rank == 0:
        print("DISTRIBUTE_OK", flush=True)
    dist.barrier(group=ctrl)


if __name__ == "__main__":
    main()
