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

import json
import os
import time

import numpy as np
import torch
import torch.distributed as dist

from synthgen import configs as cfgs

from . import mlfabric as m
from .harness import Workload, committed_bytes


NV_GUIDE_GBPS = 770.0     # pool-measured peer copy per direction per GPU (B200_PROFILING.md)


def init_dist():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
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
        copy engines into a local staging buffer of stage_mib MiB, default 4096)."""
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
        self.stage = (torch.empty((stage_mib or 4096) << 18, dtype=torch.float32, device=dev)
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

    def step(self, iteration: int, flush=None):
        """One batch on every rank.  Returns (plan dict, this rank's device ms)."""
        wl = self.wl
        draws = wl.submit_all(iteration)
        t0 = time.perf_counter()
        pb = wl.plan(iteration)
        self.last_plan_ms = (time.perf_counter() - t0) * 1e3
        pd = pb.to_dict(self.cfg["W"])
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


def plan_traffic(cfg: dict, pd: dict, mode: str) -> dict:
    """Algorithmic bytes per device of one executed plan.

    Returns per-rank lists: hbm (bytes read+written in local HBM), nv_in, nv_out.
    """
    G, S, e = cfg["G"], cfg["S"], cfg["e"]
    home, nr = cfg["home"], cfg["node_rank"]
    sl = [n for (_, n) in cfg["shards"]]
    hbm, nin, nout = [0] * G, [0] * G, [0] * G
    order = pd["order"]
    for ci, (f, k) in enumerate(zip(pd["commit_first"], pd["commit_count"])):
        gid = pd["group"][order[f]]
        if mode == "tree" and gid > 0:
            a = nr[pd["group_node"][gid - 1]]
            for p in range(f, f + k):
                h = home[order[p]]
                hbm[h] += S * e
                if h != a:
                    nout[h] += S * e
                    nin[a] += S * e
            hbm[a] += S * 4                       # aggregate written once
            for j in range(G):
                hbm[a] += sl[j] * 4               # each shard's slice read from the aggregator's HBM
                if a != j:
                    nout[a] += sl[j] * 4
                    nin[j] += sl[j] * 4
            continue
        for p in range(f, f + k):
            h = home[order[p]]
            for j in range(G):
                hbm[h] += sl[j] * e
                if h != j:
                    nout[h] += sl[j] * e
                    nin[j] += sl[j] * e
    for j in range(G):
        hbm[j] += 2 * sl[j] * 4                   # w read + write
        if pd["replica_boundary_commit"] >= 0:
            t = (j + 1) % G
            hbm[t] += sl[j] * 4
            if t != j:
                nout[j] += sl[j] * 4
                nin[t] += sl[j] * 4
    return {"hbm": hbm, "nv_in": nin, "nv_out": nout}


def measure_nvlink(device: int, rank: int, world: int, ctrl, nbytes: int = 1 << 30) -> dict:
    """Per-GPU NVLink ingress (GB/s): every rank pulls nbytes from its right neighbour at
    once, (a) with the library's copy kernel (SM peer loads) and (b) on a copy engine;
    timed on the device, max over ranks; best of 4 each."""
    dev = torch.device("cuda", device)
    src = torch.ones(nbytes // 4, dtype=torch.float32, device=dev)
    dst = torch.empty_like(src)
    torch.cuda.synchronize(dev)
    blobs = [None] * world
    dist.all_gather_object(blobs, (rank, m.ipc_export(device, src.data_ptr())), group=ctrl)
    blobs = dict(blobs)
    mp = IpcMapper(device)
    peer = mp.open(blobs[(rank + 1) % world])
    out = {}
    for name, fn in (("sm_peer_loads", m.copy_kernel), ("copy_engine", m.copy_engine),
                     ("tma_bulk", m.copy_bulk)):
        best = 0.0
        for _ in range(4):
            dist.barrier(group=ctrl)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            fn(device, dst.data_ptr(), peer, nbytes, torch.cuda.current_stream().cuda_stream)
            s1.record()
            s1.synchronize()
            ms = max_over_ranks(s0.elapsed_time(s1), ctrl)
            best = max(best, nbytes / (ms / 1e3) / 1e9)
        out[name] = round(best, 1)
    # one-way: only rank 0 pulls (from rank 1), every other link idle
    for name, fn in (("one_way_copy_engine", m.copy_engine), ("one_way_tma_bulk", m.copy_bulk)):
        best = 0.0
        for _ in range(3):
            dist.barrier(group=ctrl)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            if rank == 0:
                fn(device, dst.data_ptr(), peer, nbytes, torch.cuda.current_stream().cuda_stream)
            s1.record()
            s1.synchronize()
            ms = max_over_ranks(s0.elapsed_time(s1), ctrl)
            best = max(best, nbytes / (ms / 1e3) / 1e9)
        out[name] = round(best, 1)
    dist.barrier(group=ctrl)
    mp.close()
    del src, dst
    return out


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


def bench_distribution(S: int, rank: int, world: int, local: int, ctrl, b_nv: float, steps: int = 5,
                       flush=None) -> dict:
    """NEXT-4: every GPU's view receives the whole model (S fp32) along the plan's tree.
    Device time, max over ranks, best of `steps`; roofline = the busiest GPU's NVLink
    ingress/egress of the executed hops at b_nv."""
    G = world
    run = DistributionRun(S, rank, world, local, ctrl)
    reqs = [g for g in range(G) for _ in range(64 // G)]
    B = int(NV_GUIDE_GBPS * 1e9)
    plans = {
        "uniform": run.plan([B] * G, [B] * G, reqs, list(range(G))[::-1]),
        "degraded_gpu0_egress": run.plan([B // 10] + [B] * (G - 1), [B] * G, reqs, [(j + 1) % G for j in range(G)]),
        "all_via_gpu1": {"order": list(range(len(reqs))), "group": [1] * len(reqs), "n_direct": 0, "n_groups": 1,
                         "group_node": [1 % G], "t_total_ns": 0},
    }
    out = {}
    for name, dp in plans.items():
        best = None
        srcs = None
        for _ in range(steps):
            src, ms = run.run(dp, reqs, flush=flush)
            best = ms if best is None else min(best, ms)
            allsrc = [None] * world
            dist.all_gather_object(allsrc, src, group=ctrl)
            srcs = allsrc
        # executed hops: gathers pull every remote shard, copies pull a whole view
        nin, nout = [0] * G, [0] * G
        for r, sr in enumerate(srcs):
            if sr == -1:
                for j, (_, n) in enumerate(run.shards):
                    if j != r:
                        nin[r] += n * 4
                        nout[j] += n * 4
            elif sr >= 0:
                nin[r] += S * 4
                nout[sr] += S * 4
        t_roof = max(max(nin), max(nout)) / (b_nv * 1e9)
        out[name] = {"ms": round(best, 4), "groups": dp["n_groups"], "n_direct": dp["n_direct"],
                     "sources": srcs, "plan_t_total_ms": round(dp["t_total_ns"] / 1e6, 4),
                     "roofline_frac": round(t_roof * 1e3 / best, 4) if best else None}
    run.close()
    out["model_bytes"] = S * 4
    out["what"] = ("mlf_plan_distribution + mlf_distribute_phase: views filled from the servers (gather) or "
                   "from a distributor's view (TMA bulk copy); device ms, max over ranks, best of runs")
    return out


def w_checksum(w: torch.Tensor) -> int:
    """Exact integer digest of an fp32 tensor's bits (for bitwise comparisons across runs)."""
    return int(w.view(torch.int32).to(torch.int64).sum().item())


def nccl_baseline(cfg: dict, rank: int, world: int, local: int, ctrl, steps: int, warmup: int, flush=None):
    """The library-collective baseline the fused path is measured against (SURVEY §8(e),
    "measured alternative"): per batch, the plan's slices of every committed update travel
    by NCCL grouped send/recv into a local staging buffer, then the same commit kernel folds
    them from local HBM (a world = 1 context over this shard).  Timed with CUDA events on the
    current stream around transfer + fold, max over ranks.  Needs the NCCL default group."""
    assert dist.get_backend() == "nccl" and not cfg["replica"] and not cfg.get("gamma")
    sw = ShardedWorkload(cfg, rank, world, local, ctrl, mode="fold")
    sw.fill(0)
    wl = sw.wl
    S, W, e = cfg["S"], cfg["W"], cfg["e"]
    b, n = cfg["shards"][rank]
    tdt = wl.slots[wl.local_workers[0]].dtype if wl.local_workers else torch.float32
    remote = [w for w in range(W) if cfg["home"][w] != rank]
    row = {w: i for i, w in enumerate(remote)}
    stage = torch.empty((max(len(remote), 1), -(-max(n, 1) // 64) * 64), dtype=tdt,
                        device=torch.device("cuda", local))
    # a world = 1 context over the same shard: local slots as they are, remote ones = staging
    # rows shifted so that the kernel's slot + shard_begin lands on the row
    ptrs = [wl.slots[w].data_ptr() if w in wl.slots else stage[row[w]].data_ptr() - b * e for w in range(W)]
    st = torch.cuda.current_stream()
    ctx2 = m.Context(device=local, model_shard=wl.w, update_slots=ptrs, lr=cfg["lr"], model_elems=S,
                     shard_begin=b, dtype=wl.dt, node_rank=[0] * cfg["n_nodes"], n_nodes=cfg["n_nodes"],
                     worker_node=cfg["worker_node"], stream=st.cuda_stream)
    recs = []
    for s in range(warmup + steps):
        draws = cfgs.batch_draws(cfg, s, wl.v_init, wl.v_prev)
        for w, d in enumerate(draws):
            ctx2.submit(w, d["version"], d["t_avail"], d["norm"])
        net, prm, keep = wl.net_params(s)
        pb = ctx2.plan(net, prm)
        pd = pb.to_dict(W)
        if flush is not None:
            flush()
        st.synchronize()
        sw.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ops = []
        for g in pd["order"]:
            h = cfg["home"][g]
            if h == rank:
                for j in range(world):
                    bj, nj = cfg["shards"][j]
                    if j != rank and nj > 0:
                        ops.append(dist.P2POp(dist.isend, wl.slots[g][bj:bj + nj], j))
            elif n > 0:
                ops.append(dist.P2POp(dist.irecv, stage[row[g], :n], h))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        ctx2.execute(pb)
        e1.record(st)
        ctx2.sync()
        e1.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1), ctrl)
        wl.after_commit(pd, draws)
        sw.barrier()
        if s >= warmup:
            recs.append(dict(ms=ms, bytes=committed_bytes(cfg, pd)))
    digest = w_checksum(wl.w)
    ctx2.close()
    sw.close()
    T = sum(r["ms"] for r in recs) / 1e3
    return {"value": round(sum(r["bytes"] for r in recs) / T / 1e9, 2), "unit": "GB/s",
            "ms_per_step": round(T * 1e3 / len(recs), 4), "w_digest": digest,
            "what": "NCCL grouped send/recv of the plan's slices into local staging, then the same fused "
                    "commit kernel from local HBM (not overlapped)"}


def e2e_multi(cfg: dict, rank: int, world: int, local: int, ctrl, steps: int) -> dict:
    """The metric end to end through the public API on every rank: committed updates of the
    workers homed on a rank move from pinned host memory (phase 1, H2D), the sharded commit
    runs (phase 2), and every rank pulls its shard to pinned host memory (D2H).  Wall time
    per batch, max over ranks.  One pinned source buffer per rank is registered for all of
    its workers (host RAM bound; the bytes moved are the same)."""
    import time as _t

    sw = ShardedWorkload(cfg, rank, world, local, ctrl, mode="fold")
    sw.fill(0)
    host = sw.slots_all[0].cpu().pin_memory()
    for w in sw.wl.slots:
        sw.wl.ctx.set_update_host(w, host.data_ptr())
    sw.two_phase = True                      # host staging: peers read after every rank's H2D
    pulled = torch.empty(max(sw.wl.shard_elems, 1), dtype=torch.float32).pin_memory()
    dst = pulled.data_ptr() - sw.wl.shard_begin * 4
    tot_b, tot_s = 0, 0.0
    st0 = None
    for s in range(2 + steps):
        if s == 2:
            st0 = sw.wl.ctx.stats()
        sw.barrier()
        t0 = _t.perf_counter()
        pd, _ = sw.step(s)
        sw.wl.ctx.pull(dst, True)
        dt = max_over_ranks(_t.perf_counter() - t0, ctrl)
        if s >= 2:
            tot_b += committed_bytes(cfg, pd)
            tot_s += dt
    st1 = sw.wl.ctx.stats()
    h2d = torch.tensor([float(st1[1] - st0[1])], dtype=torch.float64)
    d2h = torch.tensor([float(st1[2] - st0[2])], dtype=torch.float64)
    dist.all_reduce(h2d, group=ctrl)
    dist.all_reduce(d2h, group=ctrl)
    sw.close()
    return {"value": round(tot_b / tot_s / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": int(h2d.item() / steps), "d2h_bytes_per_step": int(d2h.item() / steps),
            "includes": "submit + plan (host, every rank) + H2D of committed updates on their home GPU + "
                        "sharded commit over NVLink + D2H pull of every shard; wall time, max over ranks"}


def run_bench_multi(a):
    """bench.py at N > 1: config 3 (64 workers, VGG-19-sized updates) over N PS shards."""
    from bench import METRIC, Clocks, cpu_baseline_oracle, hbm_peak  # noqa: F401  (same process)

    rank, world, local, ctrl = init_dist()
    # one GPU per rank; more ranks than GPUs (a rehearsal of a larger N on a smaller box)
    # share devices round-robin and say so in the line
    shared = world > torch.cuda.device_count()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cid = a.config or 3
    os.environ["MLF_COMMIT_IMPL"] = a.kernel
    peak_hbm, peak_src = hbm_peak()
    nv_meas = measure_nvlink(local, rank, world, ctrl)
    # denominator: the best of this run's two measurements and the pool's measured peer copy
    # (770 GB/s per direction, B200_PROFILING.md) — never the slower of them
    b_nv = max(NV_GUIDE_GBPS, nv_meas["copy_engine"], nv_meas["sm_peer_loads"], nv_meas["tma_bulk"])
    b_nv_one_way = max(b_nv, nv_meas["one_way_copy_engine"], nv_meas["one_way_tma_bulk"])
    flush_w = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_r = torch.ones(64 << 20, dtype=torch.float32, device=dev)

    def l2_flush():
        flush_w.zero_()
        flush_r.sum()

    digests = {}

    def run(mode, steps, warmup, clocks=False):
        cfg = cfgs.config(cid, G=world, tau=a.tau, dtype=a.dtype)
        sw = ShardedWorkload(cfg, rank, world, local, ctrl, mode=mode)
        sw.fill(0)
        ck = Clocks(local)
        recs = []
        kl0 = 0
        for s in range(warmup + steps):
            if s == warmup:
                kl0 = sw.wl.ctx.stats()[0]
                if clocks:
                    ck.__enter__()
            pd, ms = sw.step(s, flush=l2_flush)
            ms_max = max_over_ranks(ms, ctrl)
            if s >= warmup:
                tr = plan_traffic(cfg, pd, mode)
                t_roof = max(max(tr["hbm"][j] / (peak_hbm * 1e9), tr["nv_in"][j] / (b_nv * 1e9),
                                 tr["nv_out"][j] / (b_nv * 1e9)) for j in range(world))
                recs.append(dict(ms=ms_max, bytes=committed_bytes(cfg, pd), t_roof=t_roof, tr=tr,
                                 commits=pd["n_commit"], groups=pd["n_groups"], plan_ms=sw.last_plan_ms))
        if clocks:
            ck.__exit__()
        kl = sw.wl.ctx.stats()[0] - kl0
        digests[mode] = w_checksum(sw.wl.w)
        sw.close()
        return cfg, recs, ck, kl

    torch.cuda.synchronize()
    dist.barrier(group=ctrl)
    modes = [a.mode] + ([x for x in ("fold", "staged", "tree") if x != a.mode] if not a.no_variants else [])
    results = {}
    for i, mode in enumerate(modes):
        results[mode] = run(mode, a.steps if i == 0 else max(3, a.steps // 2), a.warmup if i == 0 else 2,
                            clocks=(i == 0))
    nb = None
    cfg0 = cfgs.config(cid, G=world, tau=a.tau, dtype=a.dtype)
    if not a.no_variants and dist.get_backend() == "nccl" and not cfg0["replica"]:
        nb = nccl_baseline(cfg0, rank, world, local, ctrl, a.steps, a.warmup, flush=l2_flush)
        # same batches from the same w0: the library-collective path must land on the same bits
        same = torch.tensor([1.0 if nb["w_digest"] == digests[modes[0]] else 0.0], dtype=torch.float64)
        dist.all_reduce(same, op=dist.ReduceOp.MIN, group=ctrl)
        nb["bitwise_equal_to_primary"] = bool(same.item() == 1.0)
        del nb["w_digest"]
    ar = None
    if not a.no_variants:
        # NEXT-3: AllReduce via push/get vs NCCL all_reduce, ResNet-50-sized buffer per GPU
        # optional side measurements: a failure here (raised on every rank alike) is reported in
        # the line instead of costing the primary number
        from .allreduce import bench_allreduce
        try:
            ar = bench_allreduce(25_600_000, rank, world, local, ctrl, steps=5, warmup=2, flush=l2_flush)
        except Exception as e:                    # noqa: BLE001
            ar = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
    dv = None
    if not a.no_variants:
        try:
            dv = bench_distribution(cfg0["S"], rank, world, local, ctrl, b_nv, steps=5, flush=l2_flush)
        except Exception as e:                    # noqa: BLE001
            dv = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
    e2e = None
    if not a.no_e2e:
        e2e = e2e_multi(cfgs.config(cid, G=world, tau=a.tau, dtype=a.dtype), rank, world, local, ctrl,
                        max(3, a.steps // 4))
    torch.cuda.synchronize()
    dist.barrier(group=ctrl)
    if rank != 0:
        return
    cfg, recs, ck, kl = results[modes[0]]
    T = sum(r["ms"] for r in recs) / 1e3
    value = sum(r["bytes"] for r in recs) / T / 1e9
    t_roof = sum(r["t_roof"] for r in recs)
    tr0 = recs[0]["tr"]
    jmax = max(range(world), key=lambda j: max(tr0["nv_in"][j], tr0["nv_out"][j]))
    nv_bytes = sum(max(r["tr"]["nv_in"][jmax], r["tr"]["nv_out"][jmax]) for r in recs)
    hbm_bytes = sum(max(r["tr"]["hbm"]) for r in recs)
    nv_bound = nv_bytes / b_nv > hbm_bytes / peak_hbm
    line = {
        "metric": METRIC,
        "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": round(T * 1e3 / len(recs), 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": a.dtype, "data": "synthetic",
        "config": {"workload": f"config{cid}", "workers": cfg["W"], "update_elems": cfg["S"],
                   "tau_max": cfg["tau"], "update_dtype": a.dtype, "shards": world, "mode": modes[0],
                   "committed_per_step": round(sum(r["commits"] for r in recs) / len(recs), 2),
                   "groups_per_step": round(sum(r["groups"] for r in recs) / len(recs), 2),
                   "l2": "flushed before every step (256 MiB write + 256 MiB read); operands >> L2",
                   "parallelism": f"ps-shards{world} (one process per GPU, " + {
                       "fold": "NVLink peer loads in the commit kernel)",
                       "staged": "copy-engine NVLink pulls into local staging + commit kernel)",
                       "tree": "tree_reduce on the aggregator GPU + peer loads)"}[modes[0]],
                   **({"shared_gpus": f"{world} ranks on {torch.cuda.device_count()} GPUs: not a valid bench number"}
                      if shared else {})},
        "roofline": {"bound": "nvlink" if nv_bound else "hbm",
                     "achieved": round((nv_bytes if nv_bound else hbm_bytes) / T / 1e9, 1),
                     "peak": round(b_nv if nv_bound else peak_hbm, 1), "unit": "GB/s",
                     "frac": round(t_roof / T, 4), "traffic": None,
                     "peak_source": ("max(770 GB/s pool peer copy [B200_PROFILING.md], this run's copy-engine "
                                     "and SM peer-load ingress)" if nv_bound else peak_src),
                     "plan_relative_t_roof_ms": round(t_roof * 1e3 / len(recs), 4),
                     "frac_vs_one_way_peak": (round(t_roof / T * b_nv / b_nv_one_way, 4) if nv_bound else None),
                     "one_way_peak": b_nv_one_way,
                     "kernel": f"fused_commit_{a.kernel}"},
        "nvlink_measured_GBps": nv_meas,
        "planner_ms": round(sum(r["plan_ms"] for r in recs) / len(recs), 3),
        "step_ms_p10_p50_p90": [round(float(x), 4) for x in np.percentile([r["ms"] for r in recs], [10, 50, 90])],
        "gpu_launches": int(kl),
        "clocks": ck.summary(),
    }
    for mode2 in modes[1:]:
        cfg2, recs2, _, _ = results[mode2]
        T2 = sum(r["ms"] for r in recs2) / 1e3
        line.setdefault("variants", {})[f"mode_{mode2}"] = {
            "value": round(sum(r["bytes"] for r in recs2) / T2 / 1e9, 2), "unit": "GB/s",
            "ms_per_step": round(T2 * 1e3 / len(recs2), 4),
            "roofline_frac": round(sum(r["t_roof"] for r in recs2) / T2, 4)}
    if nb is not None:
        line.setdefault("variants", {})["nccl_sendrecv_then_fold"] = nb
    if ar is not None:
        line.setdefault("variants", {})["allreduce_push_get_vs_nccl"] = ar
    if dv is not None:
        line.setdefault("variants", {})["model_distribution"] = dv
    if e2e is not None:
        line["e2e"] = e2e
    print(json.dumps(line), flush=True)
