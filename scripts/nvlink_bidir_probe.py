"""One process, two GPUs: is the multi-GPU fold bound by the fabric under traffic in BOTH directions?

(1) one-way: the fused commit on cuda:0 with its 16 operands in cuda:1's HBM;
(2) two-way: the same commit on cuda:0 (operands on cuda:1) and, at the same time, on cuda:1
    (operands on cuda:0) — every byte a GPU reads crosses NVLink, in both directions at once;
(3) the same two-way pattern with TMA bulk copies and with copy engines (no commit arithmetic),
    pulled by the reader or pushed by the owner (remote writes instead of remote reads).
Per case: device time (CUDA events, max over the two GPUs), per-direction GB/s, and the NVLink
data counters of both GPUs from `nvidia-smi nvlink -gt d` (KiB transmitted / received over all
links) read before and after the timed repetitions.  Prints one JSON line.  Needs >= 2 GPUs."""
import json
import os
import re
import subprocess
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from cuda.bindings import runtime as cudart  # noqa: E402

from paper_1907_00434_b200 import mlfabric as m  # noqa: E402

S, W, REPS = 25_600_000, 16, 5


def nvlink_kib(dev):
    """(tx, rx) KiB summed over the links of `dev` (nvidia-smi throughput counters), or None."""
    try:
        out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(dev)], capture_output=True, text=True,
                             timeout=20).stdout
    except Exception:                         # noqa: BLE001
        return None
    tx = sum(int(x) for x in re.findall(r"Tx:\s*(\d+)\s*KiB", out))
    rx = sum(int(x) for x in re.findall(r"Rx:\s*(\d+)\s*KiB", out))
    return (tx, rx) if (tx or rx) else None


def plan_all_direct():
    return m.plan_from_dict({"n_commit": W, "order": list(range(W)), "drop_reason": [0] * W, "group": [0] * W,
                             "n_direct": W, "n_groups": 0, "group_node": [], "n_server_commits": W,
                             "commit_first": list(range(W)), "commit_count": [1] * W, "commit_t_ns": [0] * W,
                             "replica_frozen": 0, "replica_boundary_commit": -1, "n_punted": 0, "punted": [],
                             "delayed_last": 0, "t_total_ns": 0, "n_replica_commits": 0,
                             "replica_commit_first": [], "replica_commit_count": [], "replica_commit_group": [],
                             "replica_bytes": 0, "sync_mode": 0})


def timed(devs, launch):
    """launch(dev) enqueues on dev's current stream; returns the max over devs of the best-of-REPS ms."""
    best = None
    for _ in range(REPS):
        ev = {}
        for d in devs:
            torch.cuda.synchronize(d)
        for d in devs:
            with torch.cuda.device(d):
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record()
                launch(d)
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record()
                ev[d] = (e0, e1)
        ms = 0.0
        for d in devs:
            ev[d][1].synchronize()
            ms = max(ms, ev[d][0].elapsed_time(ev[d][1]))
        best = ms if best is None else min(best, ms)
    return best


def main():
    assert torch.cuda.device_count() >= 2
    for a, b in ((0, 1), (1, 0)):
        torch.cuda.set_device(a)
        err, = cudart.cudaDeviceEnablePeerAccess(b, 0)
        assert err in (cudart.cudaError_t.cudaSuccess, cudart.cudaError_t.cudaErrorPeerAccessAlreadyEnabled), err
    slots, w, ctx, dst = {}, {}, {}, {}
    for d in (0, 1):
        slots[d] = torch.empty((W, S), dtype=torch.float32, device=torch.device("cuda", d))
        for i in range(W):
            m.synth_fill(d, slots[d][i].data_ptr(), S, dtype=m.MLF_F32, seed=7, kind=1, a=i, b=d)
        w[d] = torch.zeros(S, dtype=torch.float32, device=torch.device("cuda", d))
        dst[d] = torch.empty(W * S, dtype=torch.float32, device=torch.device("cuda", d))
    for d in (0, 1):
        o = 1 - d                                          # operands live on the other GPU
        ctx[d] = m.Context(device=d, model_shard=w[d], update_slots=[slots[o][i] for i in range(W)], lr=0.01,
                           model_elems=S, stream=torch.cuda.current_stream(torch.device("cuda", d)).cuda_stream)
    plan = plan_all_direct()
    nbytes = W * S * 4

    def commit(d):
        for i in range(W):
            ctx[d].submit(i, 0)
        ctx[d].execute(plan)

    def copy_with(fn):
        return lambda d: fn(d, dst[d].data_ptr(), slots[1 - d].data_ptr(), nbytes,
                            torch.cuda.current_stream(torch.device("cuda", d)).cuda_stream)

    def push_with(fn):
        # the same bytes moved by the SOURCE GPU: it reads its own HBM and writes into the peer
        return lambda d: fn(d, dst[1 - d].data_ptr(), slots[d].data_ptr(), nbytes,
                            torch.cuda.current_stream(torch.device("cuda", d)).cuda_stream)

    res = {"bytes_per_direction": nbytes, "operands": W}
    cases = (("commit_one_way", (0,), commit), ("commit_two_way", (0, 1), commit),
             ("tma_bulk_two_way", (0, 1), copy_with(m.copy_bulk)), ("copy_engine_two_way", (0, 1), copy_with(m.copy_engine)),
             ("tma_bulk_one_way", (0,), copy_with(m.copy_bulk)),
             ("tma_bulk_push_two_way", (0, 1), push_with(m.copy_bulk)),
             ("sm_store_push_two_way", (0, 1), push_with(m.copy_kernel)),
             ("copy_engine_push_two_way", (0, 1), push_with(m.copy_engine)),
             ("tma_bulk_push_one_way", (0,), push_with(m.copy_bulk)))
    for name, devs, fn in cases:
        timed(devs, fn)                                     # warm-up
        for d in (0, 1):
            ctx[d].sync()
        c0 = [nvlink_kib(d) for d in (0, 1)]
        ms = timed(devs, fn)
        for d in (0, 1):
            ctx[d].sync()
        c1 = [nvlink_kib(d) for d in (0, 1)]
        r = {"ms": round(ms, 4), "GBps_per_direction": round(nbytes / ms / 1e6, 1)}
        if all(c0) and all(c1):
            # counters cover REPS timed runs (+ nothing else between the reads)
            r["nvlink_GB_per_run"] = {f"gpu{d}": {"tx": round((c1[d][0] - c0[d][0]) * 1024 / REPS / 1e9, 3),
                                                  "rx": round((c1[d][1] - c0[d][1]) * 1024 / REPS / 1e9, 3)}
                                      for d in (0, 1)}
        res[name] = r
    for d in (0, 1):
        ctx[d].close()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
