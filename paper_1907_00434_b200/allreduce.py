"""AllReduce through MLfabric's push/get — NEXT-3, on one box of GPUs.

"MLfabric would implement AllReduce through successive calls to push(root, update, norm)
and get(root, update), using a synchronous consistency model; root ... acts as the root of
the aggregation topology, which is a dynamically constructed tree".

B200 realisation: the root is the sharded parameter server of multigpu.py (shard j on GPU
j: all NVLink ports of the box serve the root), the plan is a synchronous one (MLfabric-S,
P:1264-1268: Alg. 3 over the list of updates, nothing dropped), and the "model" starts at
zero with lr = -1, so the fused commit computes w = 0 - (-1 * x) = the sum of the updates
in the plan's fold order (push = a plan-driven reduce-scatter fused into the commit
kernel).  get = every GPU gathers all shards over NVLink (mlf_gather, SM peer loads).
Host plumbing only; all bytes move in libmlfabric's kernels.
"""
from __future__ import annotations

import time

import torch
import torch.distributed as dist

from synthgen import configs as cfgs

from . import mlfabric as m
from .multigpu import IpcMapper, ShardedWorkload, max_over_ranks


def allreduce_config(S: int, world: int, dtype: str = "f32", workers: int | None = None) -> dict:
    """One virtual worker per GPU (or `workers`), box model, synchronous plan, lr = -1."""
    W = workers or world
    cfg = cfgs.config(3, G=world, scale_S=S, workers=W, tau=W, dtype=dtype)
    cfg["sync_mode"] = 1
    cfg["lr"] = -1.0
    return cfg


class MlfAllReduce:
    """fused = True: the commit kernel of every shard also stores its final tiles into every
    GPU's result view (push and get in ONE kernel per GPU, NVLink stores overlapped with the
    reduce); fused = False: push, barrier, then get with mlf_gather (peer loads)."""

    def __init__(self, cfg: dict, rank: int, world: int, device: int, ctrl, fused: bool = True,
                 multicast: bool = False):
        """multicast = True (with fused): the get stores through an NVLS multicast address."""
        self.cfg, self.rank, self.world, self.device, self.ctrl = cfg, rank, world, device, ctrl
        self.fused = fused
        self.sw = ShardedWorkload(cfg, rank, world, device, ctrl, mode="fold", fused_get=fused,
                                  multicast=multicast and fused)
        dev = torch.device("cuda", device)
        self.out = self.sw.view[:cfg["S"]] if fused else torch.empty(cfg["S"], dtype=torch.float32, device=dev)
        blobs = [None] * world
        dist.all_gather_object(blobs, (rank, m.ipc_export(device, self.sw.wl.w.data_ptr())), group=ctrl)
        self.mapper = IpcMapper(device)
        self.shard_ptrs = [self.sw.wl.w.data_ptr() if r == rank else self.mapper.open(b) for r, b in sorted(blobs)]
        self.begins = [b for (b, _) in cfg["shards"]]
        self.elems = [n for (_, n) in cfg["shards"]]

    def run(self, iteration: int, flush=None):
        """push (sharded fused reduce) then get (gather).  Returns (plan, push ms, get ms, wall ms),
        device times max over ranks."""
        stream = torch.cuda.current_stream()
        t0 = time.perf_counter()
        self.sw.wl.w.zero_()                      # the root's accumulator
        pd, ms_push = self.sw.step(iteration, flush=flush)
        if self.fused:                            # every view was written by the commits
            wall = (time.perf_counter() - t0) * 1e3
            return pd, max_over_ranks(ms_push, self.ctrl), 0.0, max_over_ranks(wall, self.ctrl)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        m.gather(self.device, self.out.data_ptr(), self.shard_ptrs, self.begins, self.elems, stream=stream.cuda_stream)
        e1.record(stream)
        e1.synchronize()
        self.sw.barrier()                         # nobody zeroes a shard another rank still reads
        wall = (time.perf_counter() - t0) * 1e3
        return pd, max_over_ranks(ms_push, self.ctrl), max_over_ranks(e0.elapsed_time(e1), self.ctrl), \
            max_over_ranks(wall, self.ctrl)

    def close(self):
        self.sw.close()
        self.mapper.close()
