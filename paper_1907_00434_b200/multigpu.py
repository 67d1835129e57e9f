"""Multi-GPU execution: one process per GPU, the model split into PS shards (App. B.2).

PAPER.md App. B.2: the model is split across a set S of servers,
every update has one component per server, all components share the update's
version and deadline and are reserved together.  On one 8xB200 box the servers
are the GPUs: rank j owns the contiguous shard j of w, and the plan (identical
on every rank: mlf_plan is deterministic) is executed by every rank on its own
slice.  The exchange step is the plan's tree edges:

* fold mode (agg_slots = 0): each shard's fused_commit kernel reads its slice of
  every committed update straight from the update's home GPU (NVLink peer loads
  through IPC-mapped pointers), folds groups in registers and applies them in
  commit order: a plan-driven reduce-scatter fused with the apply, one kernel.
* tree mode: groups are first summed on their aggregator's GPU (tree_reduce over
  peer members, fp32 aggregate in scratch), then every shard reads its slice of
  the aggregate — the paper's member -> aggregator -> server path.
The replica mirror of shard j is stored by rank j's commit kernel straight into
rank (j+1) mod G's memory (NVLink remote stores).

Host plumbing only: torch.distributed (gloo control group) exchanges IPC handles
and provides barriers; every byte of the data path moves inside libmlfabric's
kernels.
"""
from __future__ import annotations

import os
import time

import torch
import torch.distributed as dist

from . import mlfabric as m
from .harness import Workload


NV_GUIDE_GBPS = 770.0     # pool-measured peer copy per direction per GPU (B200_PROFILING.md)


def init_dist():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    if rank == 0:
        # rank 0 plans for the whole box (ShardedWorkload.plan_once): its planner pool may use
        # all of the host's cores (up to 16) instead of this rank's 1/LOCAL_WORLD_SIZE share (read
        # when the library's pool starts, i.e. at the first plan); the other ranks only wait for
        # the broadcast plan.  Box host, config 4 / G = 8: 16 threads 1.58-1.61 ms, 8 threads
        # 1.62-1.64 (profiles/r02/planner_side/)
        os.environ.setdefault("MLF_PLAN_THREADS", str(max(1, min(16, os.cpu_count() or 1))))
    if not dist.is_initialized():
        # NCCL when every rank has its own GPU; ranks sharing a device (tests) use gloo only
        use_nccl = torch.cuda.is_available() and torch.cuda.device_count() >= world
        dist.init_process_group(backend="nccl" if use_nccl else "gloo")
    ctrl = dist.new_group(backend="gloo")
    return rank, world, local, ctrl


def agg_slots_needed(cfg: dict, world: int) -> int:
    counts = [0] * world
    for a in cfg["aggs"]:
        counts[cfg["node_rank"][a]] += 1
    return max(counts) if counts else 0


class IpcMapper:
    """Opens every distinct peer allocation once (cudaIpcOpenMemHandle)."""

    def __init__(self, device: int):
        self.device = device
        self.opened = {}

    def open(self, blob: bytes) -> int:
        h = blob[:64]
        off = int.from_bytes(blob[64:72], "little", signed=True)
        if h not in self.opened:
            self.opened[h] = m.ipc_open(self.device, h + bytes(8))
        return self.opened[h] + off

    def close(self):
        for h, p in self.opened.items():
            m.ipc_close(self.device, p, h + bytes(8))
        self.opened = {}


class ShardedWorkload:
    """Rank `rank`'s part of a config sharded over `world` GPUs."""

    def __init__(self, cfg: dict, rank: int, world: int, device: int, ctrl, mode: str = "fold", variant: int = 0,
                 fused_get: bool = False, stage_mib: int = 0, multicast: bool = False):
        """mode: "fold" (SM peer loads inside the commit kernel), "tree" (tree_reduce on the
        aggregator GPU first) or "staged" (fold whose remote operand slices are pulled by the
        copy engines into a local staging buffer of stage_mib MiB; 0 = large enough for every
        remote slice, so each is pulled in one copy)."""
        assert cfg["G"] == world, "config shard count must equal the world size"
        self.cfg, self.rank, self.world, self.ctrl, self.mode = cfg, rank, world, ctrl, mode
        dev = torch.device("cuda", device)
        S, W = cfg["S"], cfg["W"]
        tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
        e = cfg["e"]
        local = [w for w in range(W) if cfg["home"][w] == rank]
        self.row = -(-S // 64) * 64               # 256-byte aligned rows (128-bit loads)
        self.slots_all = torch.empty((max(len(local), 1), self.row), dtype=tdt, device=dev)
        slot_tensors = {w: self.slots_all[i, :S] for i, w in enumerate(local)}
        prev = (rank - 1) % world
        self.mirror = (torch.zeros(cfg["shards"][prev][1], dtype=torch.float32, device=dev)
                       if cfg["replica"] else None)
        self.mirror_h = (torch.zeros(cfg["shards"][prev][1], dtype=torch.float32, device=dev)
                         if (cfg["replica"] and cfg.get("gamma", 0.0)) else None)
        self.replica_mode = cfg.get("replica_mode", 0) if cfg["replica"] else 0
        self.retain = None
        if self.replica_mode == 1:
            # the replica of shard `prev` lives here and starts equal to w0 of that shard
            pb, pn = cfg["shards"][prev]
            m.synth_fill(device, self.mirror.data_ptr(), pn, elem_offset=pb, dtype=m.MLF_F32, seed=cfg["seed"],
                         kind=2, stream=torch.cuda.current_stream(dev).cuda_stream)
            self.n_retain = cfg.get("n_retain", max(len(local), 1) * 2)
            self.retain = torch.empty((self.n_retain, -(-S // 64) * 64), dtype=tdt, device=dev)
        self.n_slots = agg_slots_needed(cfg, world) if mode == "tree" else 0
        if mode == "staged" and not stage_mib:
            # room for every remote operand's slice of this shard (whole-slice staging: one big
            # copy per operand), rows rounded to 4096 elements; at least 64 MiB
            n_sh = cfg["shards"][rank][1]
            stride = -(-max(n_sh, 1) // 4096) * 4096
            stage_mib = max(64, -(-((W - len(local)) * stride * e) // (1 << 20)))
        self.stage = (torch.empty(stage_mib << 18, dtype=torch.float32, device=dev)
                      if mode == "staged" else None)
        # fused get: every GPU holds a full-length view of the model, written by all shards' commits
        self.view = torch.empty(-(-S // 64) * 64, dtype=torch.float32, device=dev) if fused_get else None
        # NVLS: the views are PyTorch symmetric memory bound to one multicast object, so the
        # fused get stores each tile once (multimem.st) and NVSwitch replicates it
        self.mc_ptr = 0
        if fused_get and multicast:
            import torch.distributed._symmetric_memory as symm_mem
            self.view = symm_mem.empty(-(-S // 64) * 64, dtype=torch.float32, device=dev)
            try:
                self._symm = symm_mem.rendezvous(self.view, dist.group.WORLD)
            except RuntimeError:                  # older builds: the group must be enabled first
                symm_mem.enable_symm_mem_for_group(dist.group.WORLD.group_name)
                self._symm = symm_mem.rendezvous(self.view, dist.group.WORLD)
            self.mc_ptr = int(self._symm.multicast_ptr)
            if not self.mc_ptr:
                raise RuntimeError("multicast requested but this box's GPUs offer no NVLS multicast")
        self.scratch = (torch.empty((self.n_slots, self.row), dtype=torch.float32, device=dev)
                        if self.n_slots else None)
        torch.cuda.synchronize(dev)
        mine = {"rank": rank, "workers": local,
                "slots": m.ipc_export(device, self.slots_all.data_ptr()),
                "mirror": m.ipc_export(device, self.mirror.data_ptr()) if self.mirror is not None else None,
                "mirror_h": (m.ipc_export(device, self.mirror_h.data_ptr())
                             if self.mirror_h is not None else None),
                "scratch": m.ipc_export(device, self.scratch.data_ptr()) if self.scratch is not None else None,
                "retain": m.ipc_export(device, self.retain.data_ptr()) if self.retain is not None else None,
                "view": (m.ipc_export(device, self.view.data_ptr())
                         if self.view is not None and not self.mc_ptr else None)}
        allinfo = [None] * world
        dist.all_gather_object(allinfo, mine, group=ctrl)
        allinfo.sort(key=lambda d: d["rank"])
        self.mapper = IpcMapper(device)
        peer_slots = [None] * W
        for info in allinfo:
            r = info["rank"]
            base = self.slots_all.data_ptr() if r == rank else self.mapper.open(info["slots"])
            for i, w in enumerate(info["workers"]):
                peer_slots[w] = base + i * self.row * e
        backup_ptr = backup_h_ptr = None
        if cfg["replica"]:
            nxt = (rank + 1) % world
            backup_ptr = self.mirror.data_ptr() if nxt == rank else self.mapper.open(allinfo[nxt]["mirror"])
            if self.mirror_h is not None:
                backup_h_ptr = (self.mirror_h.data_ptr() if nxt == rank
                                else self.mapper.open(allinfo[nxt]["mirror_h"]))
        scratch_tab = None
        if self.n_slots:
            scratch_tab = []
            for info in allinfo:
                base = self.scratch.data_ptr() if info["rank"] == rank else self.mapper.open(info["scratch"])
                scratch_tab += [base + s * self.row * 4 for s in range(self.n_slots)]
        retain_tab = None
        if self.retain is not None:
            retain_tab = []
            rowb = self.retain.shape[1] * self.retain.element_size()
            for info in allinfo:
                base = self.retain.data_ptr() if info["rank"] == rank else self.mapper.open(info["retain"])
                retain_tab += [base + s * rowb for s in range(self.n_retain)]
        bcast = None
        if self.mc_ptr:
            bcast = [self.mc_ptr]
        elif self.view is not None:
            bcast = [self.view.data_ptr() if info["rank"] == rank else self.mapper.open(info["view"])
                     for info in allinfo]
        self.wl = Workload(cfg, device=device, rank=rank, world=world, variant=variant, peer_slots=peer_slots,
                           backup_ptr=backup_ptr, agg_slots=self.n_slots, agg_scratch=scratch_tab,
                           slot_tensors=slot_tensors, backup_h_ptr=backup_h_ptr, retain_table=retain_tab,
                           bcast=bcast, stage=self.stage, bcast_multicast=bool(self.mc_ptr))
        ev = self.wl.ctx.phase_event()
        evs = [None] * world
        dist.all_gather_object(evs, (rank, ev), group=ctrl)
        self.wl.ctx.open_phase_events([b for (r, b) in sorted(evs) if r != rank])
        self.two_phase = mode == "tree"
        self.barrier()

    def barrier(self):
        dist.barrier(group=self.ctrl)

    def fill(self, iteration: int):
        self.wl.fill_updates(iteration)
        torch.cuda.current_stream().synchronize()
        self.barrier()

    def plan_once(self, iteration: int):
        """The batch's plan: mlf_plan on rank 0 only (with the host's cores to itself), the integer
        plan broadcast over the gloo control group and rebuilt with plan_from_dict elsewhere.
        mlf_plan is deterministic, so this equals every rank planning for itself, and every
        rank's mlf_execute still validates the plan against its own copy of the batch."""
        wl = self.wl
        pd = None
        if self.rank == 0:
            t0 = time.perf_counter()
            try:
                pb = wl.plan(iteration)
                pd = pb.to_dict(self.cfg["W"])
            except m.MlfError as e:            # every rank raises the same error, none hangs
                pd = {"_error": (e.code, str(e).split(": ", 1)[-1])}
            self.last_plan_ms = (time.perf_counter() - t0) * 1e3
        obj = [pd]
        dist.broadcast_object_list(obj, src=0, group=self.ctrl)
        pd = obj[0]
        if "_error" in pd:
            raise m.MlfError(*pd["_error"])
        if self.rank != 0:
            pb = m.plan_from_dict(pd)
            self.last_plan_ms = 0.0
        return pb, pd

    def step(self, iteration: int, flush=None):
        """One batch on every rank.  Returns (plan dict, this rank's device ms)."""
        wl = self.wl
        draws = wl.submit_all(iteration)
        pb, pd = self.plan_once(iteration)
        if flush is not None:
            flush()
        torch.cuda.current_stream().synchronize()
        self.barrier()                          # every rank's slots are final
        if self.two_phase:
            wl.ctx.execute(pb, m.MLF_PHASE_AGGREGATE)
            self.barrier()                      # every phase-1 record enqueued (overlaps GPU work)
            wl.ctx.execute(pb, m.MLF_PHASE_COMMIT)
        else:
            wl.ctx.execute(pb)
        ms = wl.ctx.sync()
        wl.after_commit(pd, draws)
        self.barrier()                          # nobody reads a slot any more
        return pd, ms

    def close(self):
        self.wl.ctx.close()
        self.barrier()
        self.mapper.close()


def max_over_ranks(x: float, ctrl) -> float:
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=ctrl)
    return float(t.item())


class DistributionRun:
    """NEXT-4 (App. B.3) on the box: rank j holds PS shard j of a model of S fp32 elements
    (w0 here) and a full-length model view; pull requests from virtual workers on every GPU
    are served along an mlf_plan_distribution tree by mlf_distribute_phase."""

    def __init__(self, S: int, rank: int, world: int, device: int, ctrl, seed: int = 0x4D4C46):
        from synthgen.configs import shard_bounds
        self.S, self.rank, self.world, self.ctrl = S, rank, world, ctrl
        dev = torch.device("cuda", device)
        self.shards = shard_bounds(S, world)
        b, n = self.shards[rank]
        self.shard = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
        if n:
            m.synth_fill(device, self.shard.data_ptr(), n, elem_offset=b, dtype=m.MLF_F32, seed=seed, kind=2,
                         stream=torch.cuda.current_stream(dev).cuda_stream)
        self.view = torch.empty(-(-S // 64) * 64, dtype=torch.float32, device=dev)
        torch.cuda.synchronize(dev)
        mine = (rank, m.ipc_export(device, self.shard.data_ptr()), m.ipc_export(device, self.view.data_ptr()))
        allinfo = [None] * world
        dist.all_gather_object(allinfo, mine, group=ctrl)
        allinfo.sort()
        self.mapper = IpcMapper(device)
        self.shard_ptrs = [self.shard.data_ptr() if r == rank else self.mapper.open(sb) for (r, sb, _) in allinfo]
        self.view_ptrs = [self.view.data_ptr() if r == rank else self.mapper.open(vb) for (r, _, vb) in allinfo]
        self.ctx = m.Context(device=device, model_shard=self.shard[:n] if n else self.shard, update_slots=[], lr=0.0,
                             model_elems=S, shard_begin=b, rank=rank, world=world, node_rank=list(range(world)),
                             n_nodes=world, stream=torch.cuda.current_stream(dev).cuda_stream)
        ev = self.ctx.phase_event()
        evs = [None] * world
        dist.all_gather_object(evs, (rank, ev), group=ctrl)
        self.ctx.open_phase_events([e for (r, e) in sorted(evs) if r != rank])
        dist.barrier(group=ctrl)

    def plan(self, nic_up, nic_down, request_nodes, distributors) -> dict:
        """Box network: node j = GPU j (site j), PS shard j on GPU j weighted by its length."""
        G = self.world
        return m.plan_distribution(G, nic_up, nic_down, request_nodes, list(range(G)), self.S * 4,
                                   site=list(range(G)), distributors=distributors,
                                   shard_weights=[max(x, 1) for (_, x) in self.shards])

    def run(self, dplan: dict, request_nodes, flush=None):
        """Phase 1, host barrier, phase 2; returns (this rank's source, device ms max over ranks)."""
        if flush is not None:
            flush()
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.ctrl)
        args = (dplan, request_nodes, self.view_ptrs, self.shard_ptrs, [b for (b, _) in self.shards],
                [x for (_, x) in self.shards])
        src = self.ctx.distribute(*args, phase=m.MLF_PHASE_AGGREGATE)
        dist.barrier(group=self.ctrl)
        self.ctx.distribute(*args, phase=m.MLF_PHASE_COMMIT)
        ms = self.ctx.sync()
        ms = max_over_ranks(ms, self.ctrl)
        dist.barrier(group=self.ctrl)
        return src, ms

    def close(self):
        self.ctx.close()
        dist.barrier(group=self.ctrl)
        self.mapper.close()


def w_checksum(w: torch.Tensor) -> int:
    """Exact integer digest of an fp32 tensor's bits (for bitwise comparisons across runs)."""
    return int(w.view(torch.int32).to(torch.int64).sum().item())
