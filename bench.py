#!/usr/bin/env python
"""bench.py — committed update-GB/s of the MLfabric plan-execution hot path on B200.

Metric (BASELINE.json): aggregated update GB/s committed (device-timed, max over
ranks), with the roofline fraction of the dominant kernel (fused_commit).

Step = one batch through the whole hot path: every virtual worker pushes
(mlf_submit_update), mlf_plan orders / aggregates / replicates (host C++),
mlf_execute runs the fused reduce + scale + apply (+ mirror) pass on the GPU.
value = committed update bytes of K steps / sum of the K device-timed executes
(CUDA events on the launching stream, L2 flushed before every step, inputs
resident in HBM).  Planning is host-side, pipelined in a deployment, and
reported separately as planner_ms.

N = 1: BASELINE config 2 (32 virtual workers, 25.6M-element fp32 updates,
tau_max = 4 as written).  N > 1 (torchrun): config 3 (64 workers, VGG-19
143.67M-element updates) sharded over N PS shards, one process per GPU.
`--impl reference` times the CPU oracle on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from benchkit.common import METRIC, Clocks, hbm_peak  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=None)
    ap.add_argument("--tau", type=int, default=None)
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--gamma", type=float, default=0.0, help="momentum (NEXT-1); 0 = the north-star form")
    ap.add_argument("--mode", default="fold", choices=["fold", "staged", "tree"],
                    help="N > 1 transport: fold (SM peer loads), staged (copy-engine staging), tree")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--kernel", default=os.environ.get("MLF_COMMIT_IMPL"), choices=["ldg", "bulk"],
                    help="fused commit kernel (default bulk: TMA bulk copies; ldg: 128-bit load streaming)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------- reference arm (CPU oracle)
def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np

    import synthgen as sg
    from oracle.numerics import execute_plan
    from oracle.plan import Item, Params, make_net, plan as oracle_plan
    from synthgen import configs

    cid = a.config or (2 if a.gpus == 1 else 3)
    cfg = configs.config(cid, G=None if cid < 3 else a.gpus, tau=a.tau, dtype=a.dtype)
    S_sample = min(cfg["S"], 1 << 20)
    idx = np.arange(S_sample)
    dt = sg.DTYPE_BF16 if a.dtype == "bf16" else sg.DTYPE_F32
    w = sg.w0_values(cfg["seed"], idx)
    v_init = v_prev = 0
    tot_bytes, tot_s = 0, 0.0
    # the Python planner is O(#U^2 * G): on sharded configs each step plans a 16-update sample
    # of the batch so that a whole --steps/--warmup run stays within minutes
    W_s = cfg["W"] if cfg["G"] == 1 else min(cfg["W"], 16)
    for it in range(a.warmup + a.steps):
        up, down, site = configs.network(cfg, it)
        draws = configs.batch_draws(cfg, it, v_init, v_prev)[:W_s]
        ops = {g: sg.update_values(cfg["seed"], g, it, idx, dt) for g in range(W_s)}
        t0 = time.perf_counter()
        batch = [Item(cfg["worker_node"][g], cfg["S"] * cfg["e"], d["version"], d["t_avail"], d["norm"])
                 for g, d in enumerate(draws)]
        weights = [n for (_, n) in cfg["shards"]] if cfg["G"] > 1 else None
        p = oracle_plan(make_net(cfg["n_nodes"], up, down, None, site), batch,
                        Params(servers=cfg["servers"], aggs=cfg["aggs"], v_init=v_init, tau_max=cfg["tau"],
                               shard_weights=weights))
        w, _, _ = execute_plan(w, p, lambda g: ops[g], cfg["lr"])
        dt_s = time.perf_counter() - t0
        v_prev, v_init = v_init, v_init + p["n_commit"]
        if it >= a.warmup:
            tot_bytes += p["n_commit"] * S_sample * cfg["e"]
            tot_s += dt_s
    val = tot_bytes / tot_s / 1e9
    sample = (f"oracle plan of {W_s} of {cfg['W']} updates per batch + numpy numerics on the first {S_sample} of "
              f"{cfg['S']} elements per update")
    line = {"impl": "reference", "metric": METRIC,
            "value": round(val, 4),
            "unit": "GB/s", "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": round(tot_s / a.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "weak" if a.gpus == 1 else "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"config{cid}", "workers": cfg["W"], "update_elems": cfg["S"],
                       "tau_max": cfg["tau"], "update_dtype": a.dtype},
            "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def cpu_baseline_oracle(cfg, dt, budget_s=15.0):
    """The oracle as it stands on this host: plan + numerics of config batches on a sample."""
    import numpy as np

    import synthgen as sg
    from oracle.numerics import execute_plan
    from oracle.plan import Item, Params, make_net, plan as oracle_plan
    from synthgen import configs

    S_sample = min(cfg["S"], 4 << 20)
    idx = np.arange(S_sample)
    w = sg.w0_values(cfg["seed"], idx)
    v_init = v_prev = 0
    tot_b, tot_s, it = 0, 0.0, 0
    # sharded configs: the Python planner is O(#U^2 * G), so each batch plans a 16-update sample
    W_s = cfg["W"] if cfg["G"] == 1 else min(cfg["W"], 16)
    weights = [n for (_, n) in cfg["shards"]] if cfg["G"] > 1 else None
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < budget_s and it < 50:
        up, down, site = configs.network(cfg, it)
        draws = configs.batch_draws(cfg, it, v_init, v_prev)[:W_s]
        ops = {g: sg.update_values(cfg["seed"], g, it, idx, dt) for g in range(W_s)}
        t0 = time.perf_counter()
        batch = [Item(cfg["worker_node"][g], cfg["S"] * cfg["e"], d["version"], d["t_avail"], d["norm"])
                 for g, d in enumerate(draws)]
        p = oracle_plan(make_net(cfg["n_nodes"], up, down, None, site), batch,
                        Params(servers=cfg["servers"], aggs=cfg["aggs"], v_init=v_init, tau_max=cfg["tau"],
                               shard_weights=weights))
        w, _, _ = execute_plan(w, p, lambda g: ops[g], cfg["lr"])
        tot_s += time.perf_counter() - t0
        tot_b += p["n_commit"] * S_sample * cfg["e"]
        v_prev, v_init = v_init, v_init + p["n_commit"]
        it += 1
    out = {"value": round(tot_b / tot_s / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
           "cpu": cpu_model(), "host_cores": os.cpu_count(),
           "sample": f"{it} batches of config{cfg['cid']}: oracle plan of {W_s} of {cfg['W']} updates + numpy "
                     f"numerics on the first {S_sample} of {cfg['S']} elements of every update (single-threaded numpy)"}
    try:
        out["all_cores"] = cpu_oracle_all_cores(cfg, dt, p)
    except Exception as e:  # the single-core figure above is the reported baseline
        out["all_cores"] = {"error": str(e)[:200]}
    return out


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _oracle_slice(args):
    """One host core: the oracle's numerics for one batch on a slice of the model."""
    import numpy as np

    import synthgen as sg
    from oracle.numerics import execute_plan
    seed, lo, hi, plan, lr, dt = args
    idx = np.arange(lo, hi)
    w = sg.w0_values(seed, idx)
    ops = {g: sg.update_values(seed, g, 0, idx, dt) for g in plan["order"]}
    t0 = time.perf_counter()
    execute_plan(w, plan, lambda g: ops[g], lr)
    return time.perf_counter() - t0


def cpu_oracle_all_cores(cfg, dt, plan):
    """'Best plain CPU': the oracle numerics of one batch split over every host core (one
    process per slice), wall time = the slowest slice."""
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    per = min(cfg["S"] // cores, 4 << 20)
    args = [(cfg["seed"], i * per, (i + 1) * per, plan, cfg["lr"], dt) for i in range(cores)]
    with mp.get_context("spawn").Pool(cores) as pool:
        times = pool.map(_oracle_slice, args)
    nbytes = plan["n_commit"] * per * cores * cfg["e"]
    return {"value": round(nbytes / max(times) / 1e9, 4), "unit": "GB/s", "cores": cores,
            "sample": f"one batch, {cores} slices of {per} elements, numpy numerics only (plan excluded)"}


_READ_PEAK = {}


def read_peak_gbps():
    """Read-only HBM rate: the best of torch.sum (a library reduction) and mlf_read_probe (TMA bulk
    reads into shared memory, nothing written) over 4 GiB, best of 6 each, CUDA events — the read
    end of a mixed read/write ceiling."""
    import torch

    from paper_1907_00434_b200 import mlfabric as m
    if "v" not in _READ_PEAK:
        x = torch.ones(1 << 30, dtype=torch.float32, device="cuda")
        nbytes = x.numel() * 4
        st = torch.cuda.current_stream().cuda_stream
        res = {}
        for name, fn in (("torch_sum", lambda: x.sum()), ("tma_read_probe", lambda: m.read_probe(0, x.data_ptr(), nbytes, st))):
            best = 0.0
            for _ in range(6):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                e1.synchronize()
                best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
            res[name] = round(best, 1)
        del x
        torch.cuda.empty_cache()
        _READ_PEAK["v"] = max(res.values())
        _READ_PEAK["probes"] = res
    return _READ_PEAK["v"]


def roofline_extras(alg_bytes, write_bytes, ms, copy_peak, traffic):
    """frac_dram: ncu DRAM bytes of one launch (profiles/traffic.json) over the kernel time, against
    the copy peak.  frac_mixed: a ceiling for THIS read/write mix from two measured points — reads at
    the library read rate B_r, and the copy (1:1) peak B_c, which fixes the write cost
    1/B_w = 2/B_c - 1/B_r; t_roof = R/B_r + W/B_w."""
    out = {}
    if traffic:
        out["frac_dram"] = round(traffic / (ms / 1e3) / 1e9 / copy_peak, 4)
    try:
        br = read_peak_gbps()
    except Exception:                       # noqa: BLE001  (reported, not fatal)
        return out
    reads = alg_bytes - write_bytes
    inv_w = max(2.0 / copy_peak - 1.0 / br, 0.0)
    t_roof = reads / (br * 1e9) + write_bytes * inv_w / 1e9
    out.update({"read_peak_GBps": round(br, 1), "mixed_peak_GBps": round(alg_bytes / t_roof / 1e9, 1),
                "frac_mixed": round(t_roof / (ms / 1e3), 4),
                "read_peak_probes_GBps": _READ_PEAK.get("probes"),
                "read_peak_source": "max(torch.sum, mlf_read_probe TMA bulk reads) over 4 GiB, best of 6, this run"})
    return out


def run_single(a):
    import numpy as np
    import torch

    from paper_1907_00434_b200 import mlfabric as m  # noqa: F401  (loads libmlfabric.so: fails loudly if absent)
    from paper_1907_00434_b200.harness import Workload, committed_bytes
    from synthgen import configs

    cid = a.config or 2
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    peak, peak_src = hbm_peak()
    flush_w = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_r = torch.ones(64 << 20, dtype=torch.float32, device=dev)

    def l2_flush():
        # evict L2 with a 256 MiB write, then leave it holding clean unrelated lines (256 MiB read)
        # so the timed kernel neither hits stale operands nor pays for write-backs of dirty flush data
        flush_w.zero_()
        flush_r.sum()

    def measure(tau, dtype, steps, warmup, kernel, clocks=False, gamma=0.0):
        os.environ["MLF_COMMIT_IMPL"] = kernel
        cfg = configs.config(cid, G=1 if cid >= 3 else None, tau=tau, dtype=dtype, gamma=gamma)
        wl = Workload(cfg, device=0)
        wl.fill_updates(0)
        torch.cuda.synchronize()
        recs = []
        ck = Clocks(0)
        if clocks:
            ck.start()
        kl0 = 0
        for s in range(warmup + steps):
            timed = s >= warmup
            if timed and s == warmup:
                kl0 = wl.ctx.stats()[0]
                if clocks:
                    ck.mark()
            draws = wl.submit_all(s)
            t0 = time.perf_counter()
            pb = wl.plan(s)
            plan_ms = (time.perf_counter() - t0) * 1e3
            pd = pb.to_dict(cfg["W"])
            l2_flush()
            wl.ctx.execute(pb)
            ms = wl.ctx.sync()
            wl.after_commit(pd, draws)
            if timed:
                n_ops = sum(pd["commit_count"])
                hist = 2 if gamma else 1                  # momentum adds the history stream
                alg = n_ops * wl.shard_elems * cfg["e"] + 2 * hist * wl.shard_elems * 4
                if pd["replica_boundary_commit"] >= 0:
                    alg += hist * wl.shard_elems * 4
                recs.append(dict(ms=ms, bytes=committed_bytes(cfg, pd), alg=alg, plan_ms=plan_ms,
                                 commits=pd["n_commit"], groups=pd["n_groups"],
                                 wbytes=hist * wl.shard_elems * 4 * (2 if pd["replica_boundary_commit"] >= 0 else 1)))
        if clocks:
            ck.__exit__()
        kl = wl.ctx.stats()[0] - kl0
        wl.ctx.close()
        T = sum(r["ms"] for r in recs)
        return cfg, recs, T, ck, kl

    def writeback_inclusive(tau, dtype, kernel, gamma, steps=20):
        """The headline kernel's time with the write-backs it leaves in L2 charged to it.  Odd
        steps time [execute] alone, even steps [execute; a 256 MiB read] (the read evicts every
        line the kernel left dirty); every step also times [1-element memset; the same read] and
        the memset alone after a flush, so the read's own time and the launch gap before it
        cancel: penalty = T[exec; read] - T[exec] - (T[memset; read] - T[memset]).  Reported as
        the kernel's device time (ctx.sync, first to last kernel) plus that penalty."""
        os.environ["MLF_COMMIT_IMPL"] = kernel
        cfg = configs.config(cid, G=1 if cid >= 3 else None, tau=tau, dtype=dtype, gamma=gamma)
        wl = Workload(cfg, device=0)
        wl.fill_updates(0)
        st = torch.cuda.current_stream(dev)
        x, e, y, z, k_ms, alg = [], [], [], [], [], []
        tiny = flush_w[:1]

        def ev():
            return torch.cuda.Event(enable_timing=True)
        for s in range(4 + steps):
            draws = wl.submit_all(s)
            pb = wl.plan(s)
            pd = pb.to_dict(cfg["W"])
            l2_flush()
            e0, e1 = ev(), ev()
            e0.record(st)
            wl.ctx.execute(pb)
            if s % 2 == 0:
                flush_r.sum()
            e1.record(st)
            kms = wl.ctx.sync()
            wl.after_commit(pd, draws)
            l2_flush()
            e2, e3, e4, e5 = ev(), ev(), ev(), ev()
            e2.record(st)
            tiny.zero_()
            flush_r.sum()
            e3.record(st)
            e4.record(st)
            tiny.zero_()
            e5.record(st)
            torch.cuda.synchronize()
            if s >= 4:
                (x if s % 2 == 0 else e).append(e0.elapsed_time(e1))
                y.append(e2.elapsed_time(e3))
                z.append(e4.elapsed_time(e5))
                k_ms.append(kms)
                hist = 2 if gamma else 1
                alg.append(sum(pd["commit_count"]) * wl.shard_elems * cfg["e"] + 2 * hist * wl.shard_elems * 4)
        wl.ctx.close()

        def mean(v):
            return sum(v) / len(v)
        penalty = mean(x) - mean(e) - (mean(y) - mean(z))
        ms = mean(k_ms) + penalty
        return {"ms_incl_writeback": round(ms, 4), "writeback_penalty_ms": round(penalty, 4),
                "frac_incl_writeback": round(mean(alg) / (ms / 1e3) / 1e9 / peak, 4),
                "writeback_how": "kernel device time + (T[exec; 256 MiB read] - T[exec]) - (T[memset; read] - "
                                 "T[memset]), 10 + 10 steps"}

    def summarize(recs, T):
        v = sum(r["bytes"] for r in recs) / (T / 1e3) / 1e9
        ach = sum(r["alg"] for r in recs) / (T / 1e3) / 1e9
        return {"value": round(v, 2), "unit": "GB/s", "ms_per_step": round(T / len(recs), 4),
                "roofline_frac": round(ach / peak, 4), "achieved_GBps": round(ach, 1)}

    # warm-up + timed region (barrier + synchronize on both sides: single process)
    torch.cuda.synchronize()
    cfg, recs, T, ck, kl = measure(a.tau, a.dtype, a.steps, a.warmup, a.kernel, clocks=True, gamma=a.gamma)
    torch.cuda.synchronize()
    tot_bytes = sum(r["bytes"] for r in recs)
    value = tot_bytes / (T / 1e3) / 1e9
    alg = sum(r["alg"] for r in recs)
    wbytes = sum(r["wbytes"] for r in recs)
    achieved = alg / (T / 1e3) / 1e9
    wb = writeback_inclusive(a.tau, a.dtype, a.kernel, a.gamma)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        key = f"config{cid}_tau{cfg['tau']}_{a.dtype}_{a.kernel}"
        traffic = tj.get(key)
    line = {
        "metric": METRIC,
        "value": round(value, 2), "unit": "GB/s", "n_gpus": 1, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": round(T / a.steps, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": a.dtype, "data": "synthetic",
        "config": {"workload": f"config{cid}", "workers": cfg["W"], "update_elems": cfg["S"],
                   "tau_max": cfg["tau"], "update_dtype": a.dtype, "shards": 1,
                   "committed_per_step": round(sum(r["commits"] for r in recs) / len(recs), 2),
                   "groups_per_step": round(sum(r["groups"] for r in recs) / len(recs), 2),
                   "l2": "flushed before every step (256 MiB write + 256 MiB read); operands >> L2"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                     "frac_of_8TBps_spec": round(achieved / 8000.0, 4),
                     "kernel": "fused_commit_momentum" if a.gamma else f"fused_commit_{a.kernel}",
                     "algorithmic_bytes_per_step": int(alg / len(recs)),
                     # the copy peak is a 1:1 read/write ceiling and this pass is read-dominated; and
                     # ~4% of w's writes are still dirty in L2 when the kernel ends (drained by the
                     # untimed flush): the two figures below are the ones to read as a fraction
                     **roofline_extras(alg / len(recs), wbytes / len(recs), T / len(recs), peak, traffic),
                     # the same kernel with the write-backs it leaves in L2 charged to it
                     **wb},
        "planner_ms": round(sum(r["plan_ms"] for r in recs) / len(recs), 3),
        "step_ms_p10_p50_p90": [round(float(x), 4) for x in np.percentile([r["ms"] for r in recs], [10, 50, 90])],
        "gpu_launches": int(kl),
        "clocks": ck.summary(),
    }
    if not a.no_variants:
        var = {}
        other = "bulk" if a.kernel == "ldg" else "ldg"
        nv = max(5, a.steps // 2)
        _, r2, T2, _, _ = measure(a.tau, a.dtype, nv, 3, other)
        var[f"kernel_{other}"] = summarize(r2, T2)
        if cid == 2 and (a.tau is None or a.tau != 32):
            for k in (a.kernel, other):
                _, r3, T3, _, _ = measure(32, a.dtype, nv, 3, k)
                var[f"tau32_{k}"] = summarize(r3, T3)
            # NEXT-1: momentum gamma = 0.9 (Eq. 2 with history), bulk kernel
            _, r4, T4, _, _ = measure(a.tau, a.dtype, nv, 3, "bulk", gamma=0.9)
            var["momentum0.9_bulk"] = summarize(r4, T4)
            _, r5, T5, _, _ = measure(32, a.dtype, nv, 3, "bulk", gamma=0.9)
            var["momentum0.9_tau32_bulk"] = summarize(r5, T5)
            if a.dtype == "f32":
                # NEXT-1 with bf16 updates: the consumer-bound case (16-warp momentum kernel)
                for t in (4, 8, 32):
                    _, r7, T7, _, _ = measure(t, "bf16", nv, 3, "bulk", gamma=0.9)
                    var[f"momentum0.9_bf16_tau{t}_bulk"] = summarize(r7, T7)
            if a.dtype == "f32":
                # SURVEY §8(d) config 2's bf16 variant: 2-byte updates widened exactly in the kernel
                for t in (4, 32):
                    _, r6, T6, _, _ = measure(t, "bf16", nv, 3, "bulk")
                    var[f"bf16_tau{t}_bulk"] = summarize(r6, T6)
        line["variants"] = var
        os.environ["MLF_COMMIT_IMPL"] = a.kernel
    # e2e through the public API with host buffers
    if not a.no_e2e:
        line["e2e"] = e2e_single(cid, a)
        # device-resident updates, the host planner pipelined with the device: the steady-state
        # rate a deployment sees when the producers write their updates straight into HBM
        line["e2e_device_resident"] = {f"tau{t}": e2e_device_resident(cid, a, t, steps=200 if t < 32 else 40)
                                       for t in sorted({configs.config(cid).get("tau") if a.tau is None else a.tau,
                                                        32})}
    if not a.no_cpu_baseline:
        import synthgen as sg
        line["cpu_baseline"] = cpu_baseline_oracle(configs.config(cid, G=1 if cid >= 3 else None, tau=a.tau, dtype=a.dtype),
                                                   sg.DTYPE_BF16 if a.dtype == "bf16" else sg.DTYPE_F32)
    print(json.dumps(line), flush=True)


def e2e_device_resident(cid, a, tau, steps=40):
    """Committed update-GB/s by WALL time over `steps` batches through the public API with the
    updates resident in HBM: two slot sets (the producers of batch b+1 write while batch b
    commits; here both sets alias the same device buffers, so no extra HBM), and per batch
    mlf_release(1) + mlf_submit_batch + mlf_plan (host C++) + mlf_execute, so the host planning
    of batch b+1 overlaps the device commit of batch b.  The synthetic descriptors and networks
    (the input generator's draws) are made before the timed region, like the resident updates;
    the versions follow the committed counts as the batches run.  No L2 flush (operands >> L2)."""
    import numpy as np
    import torch

    from paper_1907_00434_b200 import mlfabric as m
    from synthgen import configs

    cfg = configs.config(cid, G=1 if cid >= 3 else None, tau=tau, dtype=a.dtype)
    W, S, nn = cfg["W"], cfg["S"], cfg["n_nodes"]
    tdt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
    dt = m.MLF_BF16 if a.dtype == "bf16" else m.MLF_F32
    slots = torch.empty((W, -(-S // 64) * 64), dtype=tdt, device="cuda")
    for i in range(W):
        m.synth_fill(0, slots[i].data_ptr(), S, dtype=dt, seed=cfg["seed"], kind=1, a=i, b=0)
    w = torch.empty(S, dtype=torch.float32, device="cuda")
    m.synth_fill(0, w.data_ptr(), S, dtype=m.MLF_F32, seed=cfg["seed"], kind=2)
    ctx = m.Context(device=0, model_shard=w, update_slots=[slots[i % W, :S] for i in range(2 * W)], lr=cfg["lr"],
                    model_elems=S, dtype=dt, worker_node=[cfg["worker_node"][i % W] for i in range(2 * W)],
                    n_nodes=nn, node_rank=[0] * nn, stream=torch.cuda.current_stream().cuda_stream,
                    tau_max=cfg["tau"])
    # input generation (not timed): per batch the stragglers, arrival times, norms and network
    n_b = 3 + steps
    late, tav, norms, nets = [], [], [], []
    for s in range(n_b):
        d = configs.batch_draws(cfg, s, 0, 1)            # version 1 marks a straggler (built on v_prev)
        late.append(np.array([x["version"] == 1 for x in d]))
        tav.append(np.array([x["t_avail"] for x in d], np.int64))
        norms.append(np.array([x["norm"] for x in d], np.float64))
        up, down, site = configs.network(cfg, s)
        nets.append(m.make_net(nn, up, down, None, site))
    workers = [np.arange(W, dtype=np.int32), np.arange(W, 2 * W, dtype=np.int32)]
    prm, keep2 = m.make_params(cfg["servers"], aggs=cfg["aggs"], v_init=0, tau_max=cfg["tau"])
    bytes_per = S * cfg["e"]
    torch.cuda.synchronize()
    v_init = v_prev = 0
    tot_b, plan_s, host_s, t0, kl0 = 0, 0.0, 0.0, None, 0
    for s in range(n_b):
        if s == 3:
            ctx.sync()
            kl0 = ctx.stats()[0]
            t0 = time.perf_counter()
        ctx.release(1)
        th = time.perf_counter()
        ctx.submit_batch(workers[s % 2], np.where(late[s], v_prev, v_init), tav[s], norms[s])
        prm.v_init = v_init
        tp = time.perf_counter()
        pb = ctx.plan(nets[s][0], prm)
        te = time.perf_counter()
        ctx.execute(pb)
        n_commit = pb.out.n_commit
        v_prev, v_init = v_init, v_init + n_commit
        if s >= 3:
            plan_s += te - tp
            host_s += time.perf_counter() - th
            tot_b += n_commit * bytes_per
    ctx.sync()
    wall = time.perf_counter() - t0
    launches = ctx.stats()[0] - kl0
    ctx.close()
    return {"value": round(tot_b / wall / 1e9, 2), "unit": "GB/s", "ms_per_step": round(wall / steps * 1e3, 4),
            "planner_ms": round(plan_s / steps * 1e3, 4), "host_ms": round(host_s / steps * 1e3, 4),
            "gpu_launches": int(launches), "steps": steps,
            "includes": "wall time; per batch: mlf_release + mlf_submit_batch + mlf_plan + mlf_execute "
                        "(device-resident updates, host work of batch b+1 overlapped with the commit of batch b); "
                        "host_ms = submit + plan + execute calls per batch"}


def e2e_single(cid, a):
    """Same metric end to end: pinned host updates -> (H2D of committed ones) -> commit -> D2H pull."""
    import torch

    from paper_1907_00434_b200 import mlfabric as m  # noqa: F401  (loads libmlfabric.so: fails loudly if absent)
    from paper_1907_00434_b200.harness import Workload, committed_bytes
    from synthgen import configs

    cfg = configs.config(cid, G=1 if cid >= 3 else None, tau=a.tau, dtype=a.dtype)
    wl = Workload(cfg, device=0)
    wl.fill_updates(0)
    hosts = {}
    for w, t in wl.slots.items():
        hosts[w] = t.cpu().pin_memory()
        wl.ctx.set_update_host(w, hosts[w].data_ptr())
    pulled = torch.empty(cfg["S"], dtype=torch.float32).pin_memory()
    torch.cuda.synchronize()
    steps = max(3, a.steps // 4)

    def run(pipelined: bool, s0: int):
        # pipelined: mlf_set_pull_host makes mlf_execute overlap H2D / commit / D2H chunk by chunk;
        # serial: execute (H2D then commit), then mlf_pull_model
        wl.ctx.set_pull_host(pulled.data_ptr() if pipelined else None)
        tot_b, tot_s, st0 = 0, 0.0, None
        for s in range(s0, s0 + 2 + steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            draws = wl.submit_all(s)
            pb = wl.plan(s)
            pd = pb.to_dict(cfg["W"])
            wl.ctx.execute(pb)
            wl.ctx.sync()
            if not pipelined:
                wl.ctx.pull(pulled.data_ptr(), True)
            dt_s = time.perf_counter() - t0
            wl.after_commit(pd, draws)
            if s == s0 + 1:
                st0 = wl.ctx.stats()
            if s >= s0 + 2:
                tot_b += committed_bytes(cfg, pd)
                tot_s += dt_s
        st1 = wl.ctx.stats()
        return tot_b / tot_s / 1e9, (st1[1] - st0[1]) // steps, (st1[2] - st0[2]) // steps

    def run_double(s0: int):
        # two slot sets: batch s uses set s % 2 (mlf_release(ctx, 1) frees it once batch s - 2
        # is done), so batch s + 1 is submitted, planned and its H2D started while batch s
        # still commits and pulls
        W, S, nn = cfg["W"], cfg["S"], cfg["n_nodes"]
        slots2 = torch.empty((2 * W, -(-S // 64) * 64), dtype=wl.slots[0].dtype, device="cuda")
        w2 = torch.empty(S, dtype=torch.float32, device="cuda")
        m.synth_fill(0, w2.data_ptr(), S, dtype=m.MLF_F32, seed=cfg["seed"], kind=2)
        ctx2 = m.Context(device=0, model_shard=w2, update_slots=[slots2[i, :S] for i in range(2 * W)], lr=cfg["lr"],
                         model_elems=S, dtype=wl.dt, worker_node=[cfg["worker_node"][i % W] for i in range(2 * W)],
                         n_nodes=nn, node_rank=[0] * nn, stream=torch.cuda.current_stream().cuda_stream)
        for i in range(2 * W):
            ctx2.set_update_host(i, hosts[i % W].data_ptr())
        ctx2.set_pull_host(pulled.data_ptr())
        v_init = v_prev = 0
        tot_b, t0 = 0, None
        for s in range(s0, s0 + 2 + steps):
            if s == s0 + 2:
                ctx2.sync()
                t0 = time.perf_counter()
            ctx2.release(1)
            base = (s % 2) * W
            draws = configs.batch_draws(cfg, s, v_init, v_prev)
            for k, d in enumerate(draws):
                ctx2.submit(base + k, d["version"], d["t_avail"], d["norm"])
            up, down, site = configs.network(cfg, s)
            net, keep1 = m.make_net(nn, up, down, None, site)
            prm, keep2 = m.make_params(cfg["servers"], aggs=cfg["aggs"], v_init=v_init, tau_max=cfg["tau"])
            pb = ctx2.plan(net, prm)
            pd = pb.to_dict(W)
            ctx2.execute(pb)
            v_prev, v_init = v_init, v_init + pd["n_commit"]
            if s >= s0 + 2:
                tot_b += committed_bytes(cfg, pd)
        ctx2.sync()
        dt = time.perf_counter() - t0
        ctx2.close()
        return tot_b / dt / 1e9

    v_pipe, h2d, d2h = run(True, 0)
    v_serial, _, _ = run(False, 100)
    wl.ctx.close()
    v_double = run_double(200) if cfg["G"] == 1 and not cfg["replica"] else None
    # the host link alone: one pinned H2D copy of a step's committed bytes, best of 3
    dev_buf = torch.empty(max(int(h2d) // 4, 1), dtype=torch.float32, device="cuda")
    host_buf = torch.empty_like(dev_buf, device="cpu").pin_memory()
    best = None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev_buf.copy_(host_buf, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best or 0.0, dev_buf.numel() * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9)
    v = v_double if v_double else v_pipe
    return {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h),
            "includes": "every step: submit + plan (host) + H2D of the committed updates only + fused commit + D2H "
                        "of the new model, pipelined over 16 MB chunks inside mlf_execute (copy engines both ways); "
                        "two slot sets, so step s+1's submit/plan/H2D overlap step s's commit and D2H "
                        "(mlf_release); wall time over the steps",
            "single_buffer_value": round(v_pipe, 3),
            "serial_value": round(v_serial, 3),
            "pcie_h2d_GBps": round(best, 1),
            "frac_of_h2d_link": round(v / best, 4) if best else None}


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    rank, world, local = dist_env()
    multi = world > 1 or a.gpus > 1
    if a.kernel is None:
        a.kernel = "bulk"
    if multi:
        from benchkit.multi import run_bench_multi
        line = run_bench_multi(a)
        if line is None:                      # ranks > 0: rank 0 prints the line
            return
        if not a.no_cpu_baseline:
            # the oracle on rank 0 after every rank's GPU work (same sharded config, bounded sample)
            import synthgen as sg
            from synthgen import configs
            cid = a.config or 3
            line["cpu_baseline"] = cpu_baseline_oracle(configs.config(cid, G=world, tau=a.tau, dtype=a.dtype),
                                                       sg.DTYPE_BF16 if a.dtype == "bf16" else sg.DTYPE_F32)
        print(json.dumps(line), flush=True)
        return
    run_single(a)


if __name__ == "__main__":
    main()
