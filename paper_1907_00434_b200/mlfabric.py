"""Thin ctypes binding over libmlfabric.so (include/mlfabric.h).  Argument marshalling only:
every step of the path (planning, reduce, commit, mirror) runs in the library.

There is no fallback: if the shared library is missing the import fails loudly
(build it with ``python -c "import __graft_entry__ as g; g.build()"``).
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MLF_LIB") or os.path.join(_HERE, "lib", "libmlfabric.so")

MLF_OK, MLF_E_INVALID, MLF_E_STATE, MLF_E_CUDA, MLF_E_UNSCHEDULABLE, MLF_E_CAPACITY = range(6)
MLF_F32, MLF_BF16 = 0, 1
MLF_PHASE_AGGREGATE, MLF_PHASE_COMMIT = 1, 2

# every symbol include/mlfabric.h declares
EXPORTS = (
    "mlf_plan", "mlf_init", "mlf_submit_update", "mlf_submit_batch", "mlf_set_update_host", "mlf_set_pull_host", "mlf_batch_view",
    "mlf_version",
    "mlf_execute", "mlf_execute_phase", "mlf_sync", "mlf_pull_model", "mlf_stats", "mlf_destroy",
    "mlf_last_error", "mlf_ipc_export", "mlf_ipc_open", "mlf_ipc_close", "mlf_phase_event_export",
    "mlf_phase_events_open", "mlf_gather", "mlf_synth_fill", "mlf_copy_kernel", "mlf_copy_engine",
    "mlf_copy_bulk", "mlf_read_probe", "mlf_plan_distribution", "mlf_distribute_phase", "mlf_release",
)


class MlfError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"mlfabric error {code}: {msg}")
        self.code = code


if not os.path.exists(LIB_PATH):
    raise ImportError(f"libmlfabric.so not built ({LIB_PATH}); run __graft_entry__.build()")
_lib = C.CDLL(LIB_PATH)

_p = C.c_void_p
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


class MlfNet(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("nic_up", _i64p), ("nic_down", _i64p), ("bw", _i64p), ("site", _i32p)]


class MlfBatch(C.Structure):
    _fields_ = [("n", C.c_int32), ("node", _i32p), ("bytes", _i64p), ("version", _i64p),
                ("t_avail_ns", _i64p), ("norm", _f64p)]


class MlfPlanParams(C.Structure):
    _fields_ = [("n_servers", C.c_int32), ("server", _i32p), ("shard_weight", _i64p),
                ("k", C.c_int32), ("agg", _i32p),
                ("n_replicas", C.c_int32), ("replica", _i32p), ("k_r", C.c_int32), ("replica_agg", _i32p),
                ("v_init", C.c_int64), ("tau_max", C.c_int32),
                ("div_max", C.c_double), ("gamma", C.c_double), ("hist_norm", C.c_double),
                ("n_carried", C.c_int32), ("carried_node", _i32p), ("carried_bytes", _i64p),
                ("carried_norm", _f64p), ("replica_mode", C.c_int32), ("sync_mode", C.c_int32)]


class MlfPlanOut(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("n_commit", C.c_int32), ("order", _i32p), ("drop_reason", _u8p),
                ("group", _i32p), ("n_direct", C.c_int32), ("n_groups", C.c_int32), ("group_node", _i32p),
                ("n_server_commits", C.c_int32), ("commit_first", _i32p), ("commit_count", _i32p),
                ("commit_t_ns", _i64p), ("replica_frozen", C.c_int32), ("replica_boundary_commit", C.c_int32),
                ("n_punted", C.c_int32), ("punted", _i32p), ("delayed_last", C.c_uint8),
                ("t_total_ns", C.c_int64), ("n_replica_commits", C.c_int32),
                ("replica_commit_first", _i32p), ("replica_commit_count", _i32p),
                ("replica_commit_group", _i32p), ("replica_bytes", C.c_int64), ("sync_mode", C.c_uint8)]


class MlfConfig(C.Structure):
    _fields_ = [("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("model_elems", C.c_int64), ("shard_begin", C.c_int64), ("shard_elems", C.c_int64),
                ("n_workers", C.c_int32), ("update_dtype", C.c_int32), ("lr", C.c_float),
                ("model_shard", _p), ("backup_shard", _p), ("update_slot", C.POINTER(_p)),
                ("worker_rank", _i32p), ("n_nodes", C.c_int32), ("node_rank", _i32p),
                ("worker_node", _i32p), ("agg_slots", C.c_int32), ("agg_scratch", C.POINTER(_p)),
                ("stream", _p), ("gamma", C.c_double), ("history_shard", _p), ("backup_history", _p),
                ("replica_mode", C.c_int32), ("n_retain", C.c_int32), ("retain_slot", C.POINTER(_p)),
                ("n_bcast", C.c_int32), ("bcast", C.POINTER(_p)),
                ("stage_buf", _p), ("stage_bytes", C.c_int64), ("bcast_multicast", C.c_int32),
                ("enforce_tau", C.c_int32), ("tau_max", C.c_int32)]


class MlfIpcHandle(C.Structure):
    _fields_ = [("handle", C.c_uint8 * 64), ("offset", C.c_int64)]


class MlfDistParams(C.Structure):
    _fields_ = [("n_servers", C.c_int32), ("server", _i32p), ("shard_weight", _i64p), ("k", C.c_int32),
                ("distributor", _i32p), ("model_bytes", C.c_int64)]


class MlfDistOut(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("order", _i32p), ("group", _i32p), ("n_direct", C.c_int32),
                ("n_groups", C.c_int32), ("group_node", _i32p), ("t_total_ns", C.c_int64),
                ("t_recv_ns", _i64p), ("t_start_ns", _i64p), ("t_dist_ns", _i64p)]


class MlfIpcEvent(C.Structure):
    _fields_ = [("handle", C.c_uint8 * 64)]


_lib.mlf_last_error.restype = C.c_char_p
_lib.mlf_plan.argtypes = [C.POINTER(MlfNet), C.POINTER(MlfBatch), C.POINTER(MlfPlanParams), C.POINTER(MlfPlanOut)]
_lib.mlf_plan_distribution.argtypes = [C.POINTER(MlfNet), C.c_int32, _i32p, C.POINTER(MlfDistParams),
                                       C.POINTER(MlfDistOut)]
_lib.mlf_distribute_phase.argtypes = [_p, C.POINTER(MlfDistOut), C.c_int32, _i32p, C.POINTER(_p), C.POINTER(_p),
                                      _i64p, _i64p, C.c_int32, _i32p]
_lib.mlf_init.argtypes = [C.POINTER(MlfConfig), C.c_int64, C.POINTER(_p)]
_lib.mlf_submit_update.argtypes = [_p, C.c_int32, C.c_int64, C.c_int64, C.c_double, _i32p]
_lib.mlf_submit_batch.argtypes = [_p, C.c_int32, _i32p, _i64p, _i64p, C.POINTER(C.c_double)]
_lib.mlf_set_update_host.argtypes = [_p, C.c_int32, _p]
_lib.mlf_set_pull_host.argtypes = [_p, _p]
_lib.mlf_batch_view.argtypes = [_p, C.POINTER(MlfBatch)]
_lib.mlf_version.argtypes = [_p, _i64p]
_lib.mlf_execute.argtypes = [_p, C.POINTER(MlfPlanOut)]
_lib.mlf_execute_phase.argtypes = [_p, C.POINTER(MlfPlanOut), C.c_int32]
_lib.mlf_sync.argtypes = [_p, C.POINTER(C.c_float)]
_lib.mlf_release.argtypes = [_p, C.c_int32]
_lib.mlf_pull_model.argtypes = [_p, _p, C.c_int32, _i64p]
_lib.mlf_stats.argtypes = [_p, _i64p, _i64p, _i64p]
_lib.mlf_destroy.argtypes = [_p]
_lib.mlf_destroy.restype = None
_lib.mlf_ipc_export.argtypes = [C.c_int32, _p, C.POINTER(MlfIpcHandle)]
_lib.mlf_ipc_open.argtypes = [C.c_int32, C.POINTER(MlfIpcHandle), C.POINTER(_p)]
_lib.mlf_ipc_close.argtypes = [C.c_int32, _p, C.c_int64]
_lib.mlf_phase_event_export.argtypes = [_p, C.POINTER(MlfIpcEvent)]
_lib.mlf_phase_events_open.argtypes = [_p, C.c_int32, C.POINTER(MlfIpcEvent)]
_lib.mlf_synth_fill.argtypes = [C.c_int32, _p, C.c_int64, C.c_int64, C.c_int32, C.c_uint64, C.c_int32,
                                C.c_int64, C.c_int64, C.c_int32, _p]
_lib.mlf_copy_kernel.argtypes = [C.c_int32, _p, _p, C.c_int64, _p]
_lib.mlf_copy_engine.argtypes = [C.c_int32, _p, _p, C.c_int64, _p]
_lib.mlf_copy_bulk.argtypes = [C.c_int32, _p, _p, C.c_int64, _p]
_lib.mlf_read_probe.argtypes = [C.c_int32, _p, C.c_int64, _p]
_lib.mlf_gather.argtypes = [C.c_int32, _p, C.c_int32, C.POINTER(_p), _i64p, _i64p, C.c_int32, _p]


def lib():
    return _lib


def _check(st: int):
    if st != MLF_OK:
        raise MlfError(st, _lib.mlf_last_error().decode(errors="replace"))


def _arr(x, dt):
    return np.ascontiguousarray(np.asarray(x, dtype=dt))


def _ptr(a: np.ndarray | None, ct):
    if a is None:
        return C.cast(None, C.POINTER(ct))
    return a.ctypes.data_as(C.POINTER(ct))


# ----------------------------------------------------------------- planning
def plan(n_nodes, nic_up, nic_down, batch, servers, *, bw=None, site=None, aggs=(), replicas=(), raggs=(),
         v_init=0, tau_max=1, div_max=math.inf, gamma=0.0, hist_norm=0.0, carried=(), shard_weights=None,
         replica_mode=0, sync_mode=0) -> dict:
    """mlf_plan.  `batch` = list of dicts (node, size, version, t_avail, norm) or a dict of arrays;
    `carried` = list of dicts (node, size, norm).  Returns the plan as a dict of Python lists."""
    keep = []

    def A(x, dt):
        a = _arr(x, dt)
        keep.append(a)
        return a

    up, down = A(nic_up, np.int64), A(nic_down, np.int64)
    bw_a = A(bw, np.int64) if bw is not None else None
    site_a = A(site, np.int32) if site is not None else None
    net = MlfNet(int(n_nodes), _ptr(up, C.c_int64), _ptr(down, C.c_int64), _ptr(bw_a, C.c_int64),
                 _ptr(site_a, C.c_int32))
    if isinstance(batch, dict):
        cols = batch
    else:
        cols = {k: [b[k] for b in batch] for k in ("node", "size", "version", "t_avail", "norm")}
    n = len(cols["node"])
    bn, bs, bv = A(cols["node"], np.int32), A(cols["size"], np.int64), A(cols["version"], np.int64)
    bt, bnorm = A(cols["t_avail"], np.int64), A(cols["norm"], np.float64)
    b = MlfBatch(n, _ptr(bn, C.c_int32), _ptr(bs, C.c_int64), _ptr(bv, C.c_int64), _ptr(bt, C.c_int64),
                 _ptr(bnorm, C.c_double))
    sv, ag = A(servers, np.int32), A(list(aggs), np.int32)
    rp, ra = A(list(replicas), np.int32), A(list(raggs), np.int32)
    sw = A(shard_weights, np.int64) if shard_weights is not None else None
    cn = A([c["node"] for c in carried], np.int32)
    cb = A([c["size"] for c in carried], np.int64)
    cm = A([c["norm"] for c in carried], np.float64)
    prm = MlfPlanParams(len(sv), _ptr(sv, C.c_int32), _ptr(sw, C.c_int64), len(ag), _ptr(ag, C.c_int32),
                        len(rp), _ptr(rp, C.c_int32), len(ra), _ptr(ra, C.c_int32), int(v_init), int(tau_max),
                        float(div_max), float(gamma), float(hist_norm), len(cn), _ptr(cn, C.c_int32),
                        _ptr(cb, C.c_int64), _ptr(cm, C.c_double), int(replica_mode), int(sync_mode))
    return plan_raw(net, b, prm, n + len(cn), keep)


def plan_distribution(n_nodes, nic_up, nic_down, request_nodes, servers, model_bytes: int, *, bw=None, site=None,
                      distributors=(), shard_weights=None) -> dict:
    """mlf_plan_distribution (NEXT-4, App. B.3): distribution tree for a batch of pulls."""
    keep = []

    def A(x, dt):
        a = _arr(x, dt)
        keep.append(a)
        return a

    up, down = A(nic_up, np.int64), A(nic_down, np.int64)
    bw_a = A(bw, np.int64) if bw is not None else None
    site_a = A(site, np.int32) if site is not None else None
    net = MlfNet(int(n_nodes), _ptr(up, C.c_int64), _ptr(down, C.c_int64), _ptr(bw_a, C.c_int64),
                 _ptr(site_a, C.c_int32))
    rq, sv, ds = A(list(request_nodes), np.int32), A(list(servers), np.int32), A(list(distributors), np.int32)
    sw = A(shard_weights, np.int64) if shard_weights is not None else None
    prm = MlfDistParams(len(sv), _ptr(sv, C.c_int32), _ptr(sw, C.c_int64), len(ds), _ptr(ds, C.c_int32),
                        int(model_bytes))
    n, k = len(rq), max(len(ds), 1)
    order, group = np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32)
    t_recv, t_start = np.zeros(max(n, 1), np.int64), np.zeros(max(n, 1), np.int64)
    gnode, t_dist = np.zeros(k, np.int32), np.zeros(k, np.int64)
    out = MlfDistOut(max(n, 1), _ptr(order, C.c_int32), _ptr(group, C.c_int32), 0, 0, _ptr(gnode, C.c_int32), 0,
                     _ptr(t_recv, C.c_int64), _ptr(t_start, C.c_int64), _ptr(t_dist, C.c_int64))
    _check(_lib.mlf_plan_distribution(C.byref(net), n, _ptr(rq, C.c_int32), C.byref(prm), C.byref(out)))
    ng = out.n_groups
    return {"order": order[:n].tolist(), "group": group[:n].tolist(), "n_direct": out.n_direct, "n_groups": ng,
            "group_node": gnode[:ng].tolist(), "t_total_ns": out.t_total_ns, "t_recv_ns": t_recv[:n].tolist(),
            "t_start_ns": t_start[:n].tolist(), "t_dist_ns": t_dist[:ng].tolist()}


class PlanBuffers:
    """Caller-allocated mlf_plan_out arrays (reusable across batches)."""

    def __init__(self, capacity: int):
        cap = max(int(capacity), 1)
        self.capacity = cap
        self.order = np.zeros(cap, np.int32)
        self.drop = np.zeros(cap, np.uint8)
        self.group = np.zeros(cap, np.int32)
        self.group_node = np.zeros(cap, np.int32)
        self.cfirst = np.zeros(cap, np.int32)
        self.ccount = np.zeros(cap, np.int32)
        self.ct = np.zeros(cap, np.int64)
        self.punted = np.zeros(cap, np.int32)
        self.rfirst = np.zeros(cap, np.int32)
        self.rcount = np.zeros(cap, np.int32)
        self.rgroup = np.zeros(cap, np.int32)
        self.out = MlfPlanOut()
        o = self.out
        o.capacity = cap
        o.order, o.drop_reason, o.group = _ptr(self.order, C.c_int32), _ptr(self.drop, C.c_uint8), _ptr(self.group, C.c_int32)
        o.group_node = _ptr(self.group_node, C.c_int32)
        o.commit_first, o.commit_count = _ptr(self.cfirst, C.c_int32), _ptr(self.ccount, C.c_int32)
        o.commit_t_ns, o.punted = _ptr(self.ct, C.c_int64), _ptr(self.punted, C.c_int32)
        o.replica_commit_first, o.replica_commit_count = _ptr(self.rfirst, C.c_int32), _ptr(self.rcount, C.c_int32)
        o.replica_commit_group = _ptr(self.rgroup, C.c_int32)

    def to_dict(self, n: int) -> dict:
        o = self.out
        return {
            "n_commit": o.n_commit, "order": self.order[:o.n_commit].tolist(),
            "drop_reason": self.drop[:n].tolist(), "group": self.group[:n].tolist(),
            "n_direct": o.n_direct, "n_groups": o.n_groups, "group_node": self.group_node[:o.n_groups].tolist(),
            "n_server_commits": o.n_server_commits, "commit_first": self.cfirst[:o.n_server_commits].tolist(),
            "commit_count": self.ccount[:o.n_server_commits].tolist(),
            "commit_t_ns": self.ct[:o.n_server_commits].tolist(),
            "replica_frozen": o.replica_frozen, "replica_boundary_commit": o.replica_boundary_commit,
            "n_punted": o.n_punted, "punted": self.punted[:o.n_punted].tolist(),
            "delayed_last": int(o.delayed_last), "t_total_ns": o.t_total_ns,
            "n_replica_commits": o.n_replica_commits,
            "replica_commit_first": self.rfirst[:o.n_replica_commits].tolist(),
            "replica_commit_count": self.rcount[:o.n_replica_commits].tolist(),
            "replica_commit_group": self.rgroup[:o.n_replica_commits].tolist(),
            "replica_bytes": o.replica_bytes, "sync_mode": int(o.sync_mode),
        }


def plan_raw(net: MlfNet, batch: MlfBatch, prm: MlfPlanParams, capacity: int, keep=None,
             bufs: PlanBuffers | None = None, as_dict: bool = True):
    bufs = bufs or PlanBuffers(capacity)
    _check(_lib.mlf_plan(C.byref(net), C.byref(batch), C.byref(prm), C.byref(bufs.out)))
    return bufs.to_dict(batch.n) if as_dict else bufs


def plan_from_dict(d: dict) -> MlfPlanOut:
    """Build an mlf_plan_out from a plan dict (e.g. to feed a hand-made plan to execute)."""
    n = max(len(d["drop_reason"]), len(d["order"]), 1)
    # replica outputs index carried ++ order: they can be longer than the batch
    b = PlanBuffers(max(n, len(d.get("punted", [])), len(d["commit_first"]), len(d.get("group_node", [])),
                        len(d.get("replica_commit_first", [])),
                        d.get("replica_frozen", 0) + d.get("n_punted", 0)))
    o = b.out
    o.n_commit = d["n_commit"]
    b.order[:len(d["order"])] = d["order"]
    b.drop[:len(d["drop_reason"])] = d["drop_reason"]
    b.group[:len(d["group"])] = d["group"]
    o.n_direct, o.n_groups = d["n_direct"], d["n_groups"]
    b.group_node[:len(d["group_node"])] = d["group_node"]
    o.n_server_commits = d["n_server_commits"]
    b.cfirst[:o.n_server_commits] = d["commit_first"]
    b.ccount[:o.n_server_commits] = d["commit_count"]
    b.ct[:o.n_server_commits] = d.get("commit_t_ns", [0] * o.n_server_commits)
    o.replica_frozen = d.get("replica_frozen", 0)
    o.replica_boundary_commit = d.get("replica_boundary_commit", -1)
    o.n_punted = d.get("n_punted", 0)
    b.punted[:len(d.get("punted", []))] = d.get("punted", [])
    o.delayed_last = d.get("delayed_last", 0)
    o.t_total_ns = d.get("t_total_ns", 0)
    rf = d.get("replica_commit_first", [])
    o.n_replica_commits = len(rf)
    b.rfirst[:len(rf)] = rf
    b.rcount[:len(rf)] = d.get("replica_commit_count", [])
    b.rgroup[:len(rf)] = d.get("replica_commit_group", [0] * len(rf))
    o.replica_bytes = d.get("replica_bytes", 0)
    o.sync_mode = d.get("sync_mode", 0)
    return b


# ----------------------------------------------------------------- execution
class Context:
    """One mlf_ctx (one process, one device, one PS shard)."""

    def __init__(self, *, device: int, model_shard, update_slots, lr: float, model_elems: int,
                 shard_begin: int = 0, rank: int = 0, world: int = 1, dtype: int = MLF_F32,
                 backup_shard=None, worker_rank=None, node_rank=None, n_nodes=None, agg_slots: int = 0,
                 agg_scratch=None, stream=None, v0: int = 0, worker_node=None, gamma: float = 0.0,
                 history=None, backup_history=None, replica_mode: int = 0, retain_slots=None, bcast=None,
                 stage=None, bcast_multicast: bool = False, tau_max: int | None = None):
        """update_slots: list of int device pointers (or torch tensors); model_shard/backup_shard:
        torch tensors or int pointers; stream: int cudaStream_t (None -> default stream);
        tau_max: the server's registered delay bound (Table 1), enforced by mlf_execute on every
        asynchronous plan (None: not enforced)."""
        def ptr(x):
            if x is None:
                return None
            return x if isinstance(x, int) else x.data_ptr()
        self._h = _p()
        # the library borrows every buffer for the context's lifetime (include/mlfabric.h,
        # ownership): hold the tensors passed in, so none is freed while the context uses it
        self._refs = [x for x in (model_shard, backup_shard, history, backup_history, stage, *update_slots,
                                  *(agg_scratch or []), *(retain_slots or []), *(bcast or []))
                      if x is not None and not isinstance(x, int)]
        self.n_workers = len(update_slots)
        self._slots = (_p * max(self.n_workers, 1))(*[ptr(s) for s in update_slots])
        self._wr = _arr(worker_rank if worker_rank is not None else [0] * self.n_workers, np.int32)
        nn = n_nodes if n_nodes is not None else (len(node_rank) if node_rank is not None else self.n_workers)
        self._nr = _arr(node_rank if node_rank is not None else [0] * nn, np.int32)
        self._wn = _arr(worker_node, np.int32) if worker_node is not None else None
        scr = [ptr(s) for s in (agg_scratch or [])]
        self._scr = (_p * max(len(scr), 1))(*scr)
        shard_elems = model_shard.numel() if hasattr(model_shard, "numel") else int(model_elems)
        self.cfg = MlfConfig(device, rank, world, int(model_elems), int(shard_begin), int(shard_elems),
                             self.n_workers, dtype, float(lr), ptr(model_shard), ptr(backup_shard), self._slots,
                             _ptr(self._wr, C.c_int32), int(nn), _ptr(self._nr, C.c_int32),
                             _ptr(self._wn, C.c_int32), int(agg_slots), self._scr, stream, float(gamma),
                             ptr(history), ptr(backup_history), int(replica_mode), 0, None)
        ret = [ptr(s) for s in (retain_slots or [])]
        self._ret = (_p * max(len(ret), 1))(*ret)
        if ret:
            self.cfg.n_retain = len(ret) // int(world)
            self.cfg.retain_slot = self._ret
        bc = [ptr(x) for x in (bcast or [])]
        self._bc = (_p * max(len(bc), 1))(*bc)
        if bc:
            self.cfg.n_bcast = len(bc)
            self.cfg.bcast = self._bc
            self.cfg.bcast_multicast = 1 if bcast_multicast else 0
        if tau_max is not None:
            self.cfg.enforce_tau = 1
            self.cfg.tau_max = int(tau_max)
        if stage is not None:                       # copy-engine staging buffer (torch tensor)
            self.cfg.stage_buf = ptr(stage)
            self.cfg.stage_bytes = stage.numel() * stage.element_size()
        _check(_lib.mlf_init(C.byref(self.cfg), int(v0), C.byref(self._h)))
        self._bufs = None

    def close(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.mlf_destroy(h)
            self._h = _p()
        self._refs = []

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def submit(self, worker: int, version: int, t_avail_ns: int = 0, norm: float = 0.0) -> int:
        idx = C.c_int32()
        _check(_lib.mlf_submit_update(self._h, worker, int(version), int(t_avail_ns), float(norm), C.byref(idx)))
        return idx.value

    def submit_batch(self, workers, versions, t_avail_ns=None, norms=None):
        """mlf_submit_batch: one push per worker, in order, all or nothing (int32 / int64 /
        int64 / float64 arrays; t_avail_ns, norms None -> 0)."""
        w, v = _arr(workers, np.int32), _arr(versions, np.int64)
        t = _arr(t_avail_ns, np.int64) if t_avail_ns is not None else None
        nr = _arr(norms, np.float64) if norms is not None else None
        _check(_lib.mlf_submit_batch(self._h, len(w), _ptr(w, C.c_int32), _ptr(v, C.c_int64), _ptr(t, C.c_int64),
                                     _ptr(nr, C.c_double)))

    def set_update_host(self, worker: int, host_ptr: int | None):
        _check(_lib.mlf_set_update_host(self._h, worker, host_ptr))

    def set_pull_host(self, host_ptr: int | None):
        """Every execute also delivers this rank's new shard to host_ptr + shard_begin (pinned)."""
        _check(_lib.mlf_set_pull_host(self._h, host_ptr))

    def batch_view(self) -> MlfBatch:
        b = MlfBatch()
        _check(_lib.mlf_batch_view(self._h, C.byref(b)))
        return b

    def version(self) -> int:
        v = C.c_int64()
        _check(_lib.mlf_version(self._h, C.byref(v)))
        return v.value

    def plan(self, net: MlfNet, prm: MlfPlanParams, capacity: int | None = None) -> PlanBuffers:
        b = self.batch_view()
        cap = max(capacity or 0, b.n + prm.n_carried, 1)
        if self._bufs is None or self._bufs.capacity < cap:
            self._bufs = PlanBuffers(cap)
        return plan_raw(net, b, prm, cap, bufs=self._bufs, as_dict=False)

    def execute(self, plan, phase: int = MLF_PHASE_AGGREGATE | MLF_PHASE_COMMIT):
        out = plan.out if isinstance(plan, PlanBuffers) else plan
        _check(_lib.mlf_execute_phase(self._h, C.byref(out), phase))

    def sync(self) -> float:
        ms = C.c_float()
        _check(_lib.mlf_sync(self._h, C.byref(ms)))
        return ms.value

    def release(self, max_batches: int):
        """mlf_release: wait until <= max_batches executed batches run; free the others' slots."""
        _check(_lib.mlf_release(self._h, int(max_batches)))

    def pull(self, dst, dst_is_host: bool) -> int:
        v = C.c_int64()
        d = dst if isinstance(dst, int) else dst.data_ptr()
        _check(_lib.mlf_pull_model(self._h, d, int(dst_is_host), C.byref(v)))
        return v.value

    def distribute(self, dplan: dict, request_nodes, views, shards, begins, elems,
                   phase: int = MLF_PHASE_AGGREGATE | MLF_PHASE_COMMIT) -> int:
        """mlf_distribute_phase (NEXT-4): execute a plan_distribution() plan into the per-rank
        model views.  Returns this rank's source (-1 servers, r >= 0 rank r's view, -2 none)."""
        n = len(request_nodes)
        rq = _arr(request_nodes, np.int32)
        order, group = _arr(dplan["order"], np.int32), _arr(dplan["group"], np.int32)
        gnode = _arr(dplan["group_node"] or [0], np.int32)
        out = MlfDistOut(max(n, 1), _ptr(order, C.c_int32), _ptr(group, C.c_int32), int(dplan["n_direct"]),
                         int(dplan["n_groups"]), _ptr(gnode, C.c_int32), int(dplan["t_total_ns"]), None, None, None)
        vw = (_p * len(views))(*[v if isinstance(v, int) else v.data_ptr() for v in views])
        sh = (_p * len(shards))(*[x if isinstance(x, int) else x.data_ptr() for x in shards])
        b, e = _arr(begins, np.int64), _arr(elems, np.int64)
        src = C.c_int32()
        _check(_lib.mlf_distribute_phase(self._h, C.byref(out), n, _ptr(rq, C.c_int32), vw, sh, _ptr(b, C.c_int64),
                                         _ptr(e, C.c_int64), int(phase), C.byref(src)))
        return src.value

    def phase_event(self) -> bytes:
        e = MlfIpcEvent()
        _check(_lib.mlf_phase_event_export(self._h, C.byref(e)))
        return bytes(e.handle)

    def open_phase_events(self, blobs):
        arr = (MlfIpcEvent * max(len(blobs), 1))()
        for i, b in enumerate(blobs):
            C.memmove(arr[i].handle, b, 64)
        _check(_lib.mlf_phase_events_open(self._h, len(blobs), arr))

    def stats(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        _check(_lib.mlf_stats(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value


def make_net(n_nodes, nic_up, nic_down, bw=None, site=None):
    """(MlfNet, keep-alive arrays)."""
    up, down = _arr(nic_up, np.int64), _arr(nic_down, np.int64)
    bw_a = _arr(bw, np.int64) if bw is not None else None
    site_a = _arr(site, np.int32) if site is not None else None
    net = MlfNet(int(n_nodes), _ptr(up, C.c_int64), _ptr(down, C.c_int64), _ptr(bw_a, C.c_int64),
                 _ptr(site_a, C.c_int32))
    return net, (up, down, bw_a, site_a)


def make_params(servers, *, aggs=(), replicas=(), raggs=(), v_init=0, tau_max=1, div_max=math.inf, gamma=0.0,
                hist_norm=0.0, carried=(), shard_weights=None, replica_mode=0, sync_mode=0):
    """(MlfPlanParams, keep-alive arrays)."""
    sv, ag = _arr(servers, np.int32), _arr(list(aggs), np.int32)
    rp, ra = _arr(list(replicas), np.int32), _arr(list(raggs), np.int32)
    sw = _arr(shard_weights, np.int64) if shard_weights is not None else None
    cn = _arr([c["node"] for c in carried], np.int32)
    cb = _arr([c["size"] for c in carried], np.int64)
    cm = _arr([c["norm"] for c in carried], np.float64)
    prm = MlfPlanParams(len(sv), _ptr(sv, C.c_int32), _ptr(sw, C.c_int64), len(ag), _ptr(ag, C.c_int32),
                        len(rp), _ptr(rp, C.c_int32), len(ra), _ptr(ra, C.c_int32), int(v_init), int(tau_max),
                        float(div_max), float(gamma), float(hist_norm), len(cn), _ptr(cn, C.c_int32),
                        _ptr(cb, C.c_int64), _ptr(cm, C.c_double), int(replica_mode), int(sync_mode))
    return prm, (sv, ag, rp, ra, sw, cn, cb, cm)


# ----------------------------------------------------------------- peer memory / test kernels
def ipc_export(device: int, dev_ptr: int) -> bytes:
    h = MlfIpcHandle()
    _check(_lib.mlf_ipc_export(device, dev_ptr, C.byref(h)))
    return bytes(h.handle) + int(h.offset).to_bytes(8, "little", signed=True)


def ipc_open(device: int, blob: bytes) -> int:
    h = MlfIpcHandle()
    C.memmove(h.handle, blob[:64], 64)
    h.offset = int.from_bytes(blob[64:72], "little", signed=True)
    p = _p()
    _check(_lib.mlf_ipc_open(device, C.byref(h), C.byref(p)))
    return p.value


def ipc_close(device: int, dev_ptr: int, blob: bytes):
    _check(_lib.mlf_ipc_close(device, dev_ptr, int.from_bytes(blob[64:72], "little", signed=True)))


def synth_fill(device: int, dst_ptr: int, n: int, *, elem_offset: int = 0, dtype: int = MLF_F32, seed: int,
               kind: int, a: int = 0, b: int = 0, variant: int = 0, stream=None):
    _check(_lib.mlf_synth_fill(device, dst_ptr, int(n), int(elem_offset), dtype, seed, kind, int(a), int(b),
                               variant, stream))


def copy_kernel(device: int, dst_ptr: int, src_ptr: int, nbytes: int, stream=None):
    _check(_lib.mlf_copy_kernel(device, dst_ptr, src_ptr, int(nbytes), stream))


def gather(device: int, dst_ptr: int, shard_ptrs, begins, elems, copy_engine: int = 0, stream=None):
    """mlf_gather: the whole model from its shards (local or mapped peer pointers).
    copy_engine: 0 TMA bulk copies, 1 copy engine, 2 SM 128-bit peer loads."""
    n = len(shard_ptrs)
    sp = (_p * max(n, 1))(*shard_ptrs)
    b, e = _arr(begins, np.int64), _arr(elems, np.int64)
    _check(_lib.mlf_gather(device, dst_ptr, n, sp, _ptr(b, C.c_int64), _ptr(e, C.c_int64), int(copy_engine), stream))


def copy_bulk(device: int, dst_ptr: int, src_ptr: int, nbytes: int, stream=None):
    _check(_lib.mlf_copy_bulk(device, dst_ptr, src_ptr, int(nbytes), stream))


def read_probe(device: int, src_ptr: int, nbytes: int, stream=None):
    _check(_lib.mlf_read_probe(device, src_ptr, int(nbytes), stream))


def copy_engine(device: int, dst_ptr: int, src_ptr: int, nbytes: int, stream=None):
    _check(_lib.mlf_copy_engine(device, dst_ptr, src_ptr, int(nbytes), stream))
