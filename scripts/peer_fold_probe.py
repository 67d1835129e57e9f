"""One process, two GPUs: the fused commit on cuda:0 with every operand in cuda:1's HBM
(peer access, no IPC), i.e. one-directional NVLink traffic.  Compares the kernel's ingress
with one-directional copy probes, so the bidirectional-contention share of the multi-GPU
gap can be read off.  Prints one JSON line.  Needs >= 2 GPUs."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from cuda.bindings import runtime as cudart  # noqa: E402

from paper_1907_00434_b200 import mlfabric as m  # noqa: E402


def ms_of(fn, reps=5):
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


def main():
    assert torch.cuda.device_count() >= 2
    torch.cuda.set_device(0)
    err, = cudart.cudaDeviceEnablePeerAccess(1, 0)
    assert err in (cudart.cudaError_t.cudaSuccess, cudart.cudaError_t.cudaErrorPeerAccessAlreadyEnabled), err
    S, W = 25_600_000, 16
    d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
    slots = torch.empty((W, S), dtype=torch.float32, device=d1)
    for w in range(W):
        m.synth_fill(1, slots[w].data_ptr(), S, dtype=m.MLF_F32, seed=7, kind=1, a=w, b=0)
    torch.cuda.synchronize(d1)
    wt = torch.zeros(S, dtype=torch.float32, device=d0)
    st = torch.cuda.current_stream(d0).cuda_stream
    ctx = m.Context(device=0, model_shard=wt, update_slots=[slots[w] for w in range(W)], lr=0.01, model_elems=S,
                    stream=st)
    plan = {"n_commit": W, "order": list(range(W)), "drop_reason": [0] * W, "group": [0] * W, "n_direct": W,
            "n_groups": 0, "group_node": [], "n_server_commits": W, "commit_first": list(range(W)),
            "commit_count": [1] * W, "commit_t_ns": [0] * W, "replica_frozen": 0, "replica_boundary_commit": -1,
            "n_punted": 0, "punted": [], "delayed_last": 0, "t_total_ns": 0, "n_replica_commits": 0,
            "replica_commit_first": [], "replica_commit_count": [], "replica_commit_group": [], "replica_bytes": 0,
            "sync_mode": 0}
    out = m.plan_from_dict(plan)

    def commit():
        for w in range(W):
            ctx.submit(w, 0)
        ctx.execute(out)
        ctx.sync()

    commit()
    t_commit = ms_of(commit)
    nbytes = W * S * 4
    src = slots.view(-1)
    dst = torch.empty(nbytes // 4, dtype=torch.float32, device=d0)
    res = {"fused_commit_peer_ingress_GBps": round(nbytes / t_commit / 1e6, 1)}
    for name, fn in (("tma_bulk", m.copy_bulk), ("sm_peer_loads", m.copy_kernel), ("copy_engine", m.copy_engine)):
        t = ms_of(lambda: fn(0, dst.data_ptr(), src.data_ptr(), nbytes, st))
        res[f"{name}_one_way_GBps"] = round(nbytes / t / 1e6, 1)
    res["operands"] = W
    res["bytes"] = nbytes
    ctx.close()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
