"""bench.py's multi-GPU legs (N > 1): bench harness, NOT product code.

Moved out of the product package (paper_1907_00434_b200/) so that the package holds only the
hot path and its plumbing.  Everything here drives the package's public classes
(ShardedWorkload, DistributionRun, MlfAllReduce) and times them; none of it touches
oracle/ (the CPU baseline is bench.py's own leg).

* run_bench_multi — config 3 (or --config) sharded over N GPUs: fold / staged / tree modes,
  the NCCL send/recv baseline, AllReduce vs NCCL, model distribution, e2e with host buffers;
* plan_traffic — SURVEY §8(d) algorithmic bytes per device of one executed plan;
* measure_nvlink — the NVLink denominators (every rank pulling at once, and one-way).
"""
from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist

from paper_1907_00434_b200 import mlfabric as m
from paper_1907_00434_b200.allreduce import MlfAllReduce, allreduce_config
from paper_1907_00434_b200.harness import Workload, committed_bytes
from paper_1907_00434_b200.multigpu import (NV_GUIDE_GBPS, DistributionRun, IpcMapper, ShardedWorkload,
                                            init_dist, max_over_ranks, w_checksum)
from synthgen import configs as cfgs

from .common import METRIC, Clocks, hbm_peak


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


def same_workload_one_gpu(cid: int, a, device: int, steps: int = 5, warmup: int = 2, flush=None) -> dict:
    """Config `cid` with every worker and the whole model on one GPU (G = 1: one shard, every
    transfer local): committed update-GB/s and ms per batch, device-timed like the main line."""
    cfg = cfgs.config(cid, G=1, tau=a.tau, dtype=a.dtype)
    torch.cuda.empty_cache()
    wl = Workload(cfg, device=device)
    wl.fill_updates(0)
    torch.cuda.synchronize()
    tot_b, tot_ms = 0, 0.0
    for s in range(warmup + steps):
        draws = wl.submit_all(s)
        pb = wl.plan(s)
        pd = pb.to_dict(cfg["W"])
        if flush is not None:
            flush()
        wl.ctx.execute(pb)
        ms = wl.ctx.sync()
        wl.after_commit(pd, draws)
        if s >= warmup:
            tot_b += committed_bytes(cfg, pd)
            tot_ms += ms
    wl.ctx.close()
    del wl
    torch.cuda.empty_cache()
    return {"value": round(tot_b / (tot_ms / 1e3) / 1e9, 2), "unit": "GB/s", "ms_per_step": round(tot_ms / steps, 4),
            "what": f"config{cid} with all {cfg['W']} workers and the whole model on GPU 0 (HBM-bound, no NVLink)"}


def run_bench_multi(a):
    """bench.py at N > 1: config 3 (64 workers, VGG-19-sized updates) over N PS shards.
    Returns the JSON line on rank 0 (bench.py adds the CPU baseline and prints it), None elsewhere."""
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
        if clocks:
            ck.start()
        recs = []
        kl0 = 0
        for s in range(warmup + steps):
            if s == warmup:
                kl0 = sw.wl.ctx.stats()[0]
                if clocks:
                    ck.mark()
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
    if not a.no_variants:
        # the mixed transport: the copy engines pull 3 of every 4 remote operands in 3 chunks, the
        # kernel reads the rest over the peer mappings, the first chunk straight from the peers
        # (config 3 at 2 GPUs: 90.2% of the NVLink roofline vs 89.7% with every second operand in
        # 4 chunks and 87.9% for fold; profiles/r02/hybrid/skip/)
        mixed = {"MLF_STAGE_SKIP": "4", "MLF_STAGE_CHUNKS": "3", "MLF_STAGE_FIRST_DIRECT": "1"}
        saved = {k: os.environ.get(k) for k in mixed}
        os.environ.update(mixed)
        try:
            results["staged_mixed"] = run("staged", max(3, a.steps // 2), 2)
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        modes.append("staged_mixed")
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
    # the same workload on ONE GPU (rank 0 alone, the others wait): sharding moves (N-1)/N of
    # every update over NVLink, so the 1-GPU HBM time is the figure to read the N-GPU line against
    one = None
    if not a.no_variants:
        torch.cuda.synchronize()
        dist.barrier(group=ctrl)
        if rank == 0:
            try:
                one = same_workload_one_gpu(cid, a, local, flush=l2_flush)
            except Exception as e:                # noqa: BLE001  (e.g. the slots do not fit)
                one = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
    torch.cuda.synchronize()
    dist.barrier(group=ctrl)
    if rank != 0:
        return None
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
    if one is not None:
        line["same_workload_1gpu"] = one
    if e2e is not None:
        line["e2e"] = e2e
    return line


def bench_allreduce(S: int, rank: int, world: int, device: int, ctrl, steps: int = 5, warmup: int = 2,
                    flush=None) -> dict:
    """MLfabric AllReduce vs NCCL all_reduce on the same per-GPU buffer of S fp32 values."""
    cfg = allreduce_config(S, world)
    res = {}
    variants = [(True, False), (False, False)]
    if dist.get_backend() == "nccl":
        variants.append((True, True))             # NVLS multicast get (one GPU per rank)
    for fused, mc in variants:
        try:
            ar = MlfAllReduce(cfg, rank, world, device, ctrl, fused=fused, multicast=mc)
        except Exception:                         # no multicast on this box (fails on every rank alike)
            if not mc:
                raise
            continue
        ar.sw.fill(0)
        push = get = wall = 0.0
        for s in range(warmup + steps):
            _, mp, mg, mw = ar.run(s, flush=flush)
            if s >= warmup:
                push, get, wall = push + mp, get + mg, wall + mw
        ar.close()
        res[(fused, mc)] = (push / steps, get / steps, wall / steps)
    # NCCL on the default (NCCL) process group, same bytes per GPU
    t = torch.ones(S, dtype=torch.float32, device=torch.device("cuda", device))
    nccl_ms = None
    if dist.get_backend() == "nccl":
        for _ in range(warmup):
            dist.all_reduce(t)
        torch.cuda.synchronize()
        acc = 0.0
        for _ in range(steps):
            if flush is not None:
                flush()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dist.all_reduce(t)
            e1.record()
            e1.synchronize()
            acc += max_over_ranks(e0.elapsed_time(e1), ctrl)
        nccl_ms = acc / steps
    nbytes = S * 4

    def busbw(ms):
        return round(2 * (world - 1) / world * nbytes / (ms / 1e3) / 1e9, 1) if ms else None

    fp, _, fw = res[(True, False)]
    gp, gg, gw = res[(False, False)]
    mcp = res[(True, True)][0] if (True, True) in res else None
    return {"bytes_per_gpu": nbytes,
            "mlfabric_fused_ms": round(fp, 4), "mlfabric_fused_busbw_GBps": busbw(fp),
            "mlfabric_fused_wall_ms": round(fw, 3),
            "mlfabric_fused_multicast_ms": round(mcp, 4) if mcp else None,
            "mlfabric_fused_multicast_busbw_GBps": busbw(mcp) if mcp else None,
            "mlfabric_push_then_gather_ms": round(gp + gg, 4), "push_ms": round(gp, 4), "gather_ms": round(gg, 4),
            "mlfabric_push_then_gather_busbw_GBps": busbw(gp + gg),
            "nccl_ms": round(nccl_ms, 4) if nccl_ms else None, "nccl_busbw_GBps": busbw(nccl_ms),
            "timing": "device time (CUDA events), max over ranks; busbw = 2(N-1)/N * bytes / time"}
