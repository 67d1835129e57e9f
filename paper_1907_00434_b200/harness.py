"""Driving a BASELINE workload through the C ABI on one process/device (plumbing only).

PyTorch allocates the device memory (model shard, backup shard, update slots)
and provides the stream; every compute step goes through libmlfabric
(mlf_synth_fill produces the synthetic updates, mlf_plan plans, mlf_execute
commits).  Nothing here implements any of the method's arithmetic.
"""
from __future__ import annotations

import math

import torch

from synthgen import configs as cfgs
from . import mlfabric as m

KIND_UPDATE, KIND_W0 = 1, 2


class Workload:
    """Config `cfg` (synthgen.configs.config) on this process's device, shard `rank`."""

    def __init__(self, cfg: dict, *, device: int = 0, rank: int = 0, world: int = 1, variant: int = 0,
                 peer_slots=None, backup_ptr=None, agg_slots: int = 0, agg_scratch=None, stream=None,
                 slot_tensors: dict | None = None, backup_h_ptr=None, retain_table=None, bcast=None,
                 stage=None, bcast_multicast: bool = False):
        self.cfg = cfg
        self.device, self.rank, self.world = device, rank, world
        self.variant = variant
        self.S = cfg["S"]
        self.dt = m.MLF_BF16 if cfg["dtype"] == "bf16" else m.MLF_F32
        tdt = torch.bfloat16 if self.dt == m.MLF_BF16 else torch.float32
        dev = torch.device("cuda", device)
        b, n = cfg["shards"][rank]
        self.shard_begin, self.shard_elems = b, n
        self.stream = stream or torch.cuda.current_stream(dev)
        self.w = torch.empty(n, dtype=torch.float32, device=dev)
        self.backup = torch.zeros(n, dtype=torch.float32, device=dev) if (cfg["replica"] and world == 1) else None
        # momentum (NEXT-1): the server-side history h = w_t - w_{t-1}, zero at start
        self.gamma = cfg.get("gamma", 0.0)
        self.h = torch.zeros(n, dtype=torch.float32, device=dev) if self.gamma else None
        self.backup_h = (torch.zeros(n, dtype=torch.float32, device=dev)
                         if (self.gamma and cfg["replica"] and world == 1) else None)
        # update slots of the workers homed here (full-length vectors)
        self.local_workers = [w for w in range(cfg["W"]) if cfg["home"][w] == rank]
        if slot_tensors is not None:
            self.slots = dict(slot_tensors)
        else:
            self.slots = {w: torch.empty(self.S, dtype=tdt, device=dev) for w in self.local_workers}
        slot_ptrs = []
        for w in range(cfg["W"]):
            if w in self.slots:
                slot_ptrs.append(self.slots[w].data_ptr())
            else:
                slot_ptrs.append(peer_slots[w])
        bptr = backup_ptr if backup_ptr is not None else (self.backup.data_ptr() if self.backup is not None else None)
        # replica trees (NEXT-2): the backup is the replica's own model (starts equal to w0) and
        # punted updates are retained in a pool until the replica has them
        self.replica_mode = cfg.get("replica_mode", 0) if cfg["replica"] else 0
        self.retain = None
        if self.replica_mode == 1 and retain_table is None:
            n_ret = cfg.get("n_retain", 2 * cfg["W"])
            self.retain = torch.empty((n_ret, -(-self.S // 64) * 64), dtype=tdt, device=dev)
            retain_table = [self.retain[i].data_ptr() for i in range(n_ret)]
        self.fill_w0()
        if self.replica_mode == 1 and self.backup is not None:
            m.synth_fill(device, self.backup.data_ptr(), n, elem_offset=b, dtype=m.MLF_F32, seed=cfg["seed"],
                         kind=KIND_W0, variant=variant, stream=self.stream.cuda_stream)
        self.ctx = m.Context(device=device, model_shard=self.w, update_slots=slot_ptrs, lr=cfg["lr"],
                             model_elems=self.S, shard_begin=b, rank=rank, world=world, dtype=self.dt,
                             backup_shard=bptr, worker_rank=cfg["home"], node_rank=cfg["node_rank"],
                             n_nodes=cfg["n_nodes"], agg_slots=agg_slots, agg_scratch=agg_scratch,
                             stream=self.stream.cuda_stream, v0=0, worker_node=cfg["worker_node"],
                             gamma=self.gamma, history=self.h,
                             backup_history=(backup_h_ptr if backup_h_ptr is not None else self.backup_h),
                             replica_mode=self.replica_mode, retain_slots=retain_table, bcast=bcast,
                             stage=stage, bcast_multicast=bcast_multicast, tau_max=cfg["tau"])
        self.v_init, self.v_prev = 0, 0
        self.iteration = 0
        self.carried = []
        self._keep = None

    # ---------------------------------------------------------------- data
    def fill_w0(self):
        m.synth_fill(self.device, self.w.data_ptr(), self.shard_elems, elem_offset=self.shard_begin,
                     dtype=m.MLF_F32, seed=self.cfg["seed"], kind=KIND_W0, variant=self.variant,
                     stream=self.stream.cuda_stream)

    def fill_updates(self, iteration: int):
        for w, t in self.slots.items():
            m.synth_fill(self.device, t.data_ptr(), self.S, dtype=self.dt, seed=self.cfg["seed"],
                         kind=KIND_UPDATE, a=w, b=iteration, variant=self.variant, stream=self.stream.cuda_stream)

    # ---------------------------------------------------------------- planning
    def net_params(self, iteration: int):
        c = self.cfg
        up, down, site = cfgs.network(c, iteration)
        net, k1 = m.make_net(c["n_nodes"], up, down, None, site)
        weights = [n for (_, n) in c["shards"]] if c["G"] > 1 else None
        prm, k2 = m.make_params(c["servers"], aggs=c["aggs"], replicas=c["replicas"], raggs=c["raggs"],
                                v_init=self.v_init, tau_max=c["tau"], div_max=c["div_max"],
                                gamma=c.get("gamma", 0.0), hist_norm=0.0, carried=self.carried,
                                shard_weights=weights, replica_mode=self.replica_mode,
                                sync_mode=c.get("sync_mode", 0))
        return net, prm, (k1, k2)

    def submit_all(self, iteration: int):
        draws = cfgs.batch_draws(self.cfg, iteration, self.v_init, self.v_prev)
        self.ctx.submit_batch(range(len(draws)), [d["version"] for d in draws], [d["t_avail"] for d in draws],
                              [d["norm"] for d in draws])
        return draws

    def plan(self, iteration: int):
        net, prm, keep = self.net_params(iteration)
        self._keep = keep
        return self.ctx.plan(net, prm)

    def after_commit(self, plan_dict: dict, draws):
        """Harness bookkeeping: versions, punted replica items for the next batch."""
        self.v_prev = self.v_init
        if plan_dict.get("sync_mode"):
            self.v_init += 1 if plan_dict["n_commit"] else 0     # one version per iteration (R22)
        else:
            self.v_init += plan_dict["n_commit"]
        if self.cfg["replica"]:
            items = list(self.carried) + [dict(node=self.cfg["worker_node"][g], size=self.S * self.cfg["e"],
                                               norm=draws[g]["norm"]) for g in plan_dict["order"]]
            self.carried = [items[i] for i in plan_dict["punted"]]
        self.iteration += 1

    def step(self, iteration: int | None = None, refill: bool = True):
        """One batch: fill updates, submit, plan, execute (async).  Returns (plan buffers, dict, draws)."""
        it = self.iteration if iteration is None else iteration
        if refill:
            self.fill_updates(it)
        draws = self.submit_all(it)
        pb = self.plan(it)
        n = len(draws)
        pd = pb.to_dict(n)
        self.ctx.execute(pb)
        self.after_commit(pd, draws)
        return pb, pd, draws


def committed_bytes(cfg: dict, plan_dict: dict) -> int:
    return plan_dict["n_commit"] * cfg["S"] * cfg["e"]


def isfinite(x):
    return x is not None and math.isfinite(x)
