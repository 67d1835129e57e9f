"""NVLink transport probe (torchrun, N ranks): every rank pulls from its right neighbour at
once; device time, max over ranks.  Copy-engine pulls by copy size and stream count, SM
peer loads, TMA bulk, and an SM + copy-engine split running concurrently.  Prints one JSON
line per case on rank 0.  Used to choose the staged-mode transport."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1907_00434_b200 import mlfabric as m  # noqa: E402
from paper_1907_00434_b200.multigpu import IpcMapper, init_dist, max_over_ranks  # noqa: E402

TOTAL = 1 << 30


def main():
    rank, world, local, ctrl = init_dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    src = torch.ones(TOTAL // 4, dtype=torch.float32, device=dev)
    dst = torch.empty_like(src)
    torch.cuda.synchronize(dev)
    blobs = [None] * world
    dist.all_gather_object(blobs, (rank, m.ipc_export(local, src.data_ptr())), group=ctrl)
    peer = IpcMapper(local).open(dict(blobs)[(rank + 1) % world])
    streams = [torch.cuda.Stream(dev) for _ in range(8)]
    main_s = torch.cuda.current_stream(dev)

    def timed(fn, reps=3):
        best = 0.0
        for _ in range(reps):
            dist.barrier(group=ctrl)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main_s)
            fn()
            e1.record(main_s)
            e1.synchronize()
            ms = max_over_ranks(e0.elapsed_time(e1), ctrl)
            best = max(best, TOTAL / (ms / 1e3) / 1e9)
        return round(best, 1)

    def join(ns):
        for s in streams[:ns]:
            e = torch.cuda.Event()
            e.record(s)
            main_s.wait_event(e)

    def ce(chunk, ns, frac=1.0, base=0, do_join=True):
        """copy-engine pull of frac*TOTAL bytes in `chunk`-byte copies round-robin on ns streams"""
        ev = torch.cuda.Event()
        ev.record(main_s)
        nbytes = int(TOTAL * frac) // chunk * chunk
        for s in streams[:ns]:
            s.wait_event(ev)
        for i, off in enumerate(range(0, nbytes, chunk)):
            s = streams[i % ns]
            m.copy_engine(local, dst.data_ptr() + base + off, peer + base + off, chunk, s.cuda_stream)
        if do_join:
            join(ns)
        return nbytes

    res = {}
    for chunk in (4 << 20, 16 << 20, 64 << 20, 256 << 20, 1 << 30):
        for ns in (1, 2, 4, 8):
            if chunk == 1 << 30 and ns > 1:
                continue
            res[f"ce_chunk{chunk >> 20}M_streams{ns}"] = timed(lambda: ce(chunk, ns))
    res["sm_peer_loads"] = timed(lambda: m.copy_kernel(local, dst.data_ptr(), peer, TOTAL, main_s.cuda_stream))
    res["tma_bulk"] = timed(lambda: m.copy_bulk(local, dst.data_ptr(), peer, TOTAL, main_s.cuda_stream))
    # concurrent split: fraction f on the copy engines (64 MiB copies, 2 streams), the rest SM / TMA
    for f in (0.25, 0.4, 0.5, 0.6):
        nce = int(TOTAL * f) // (64 << 20) * (64 << 20)

        def split(kern=m.copy_bulk):
            ce_b = ce(64 << 20, 2, f, do_join=False)
            kern(local, dst.data_ptr() + ce_b, peer + ce_b, TOTAL - ce_b, main_s.cuda_stream)
            join(2)

        assert nce > 0
        res[f"split_ce{f}_tma"] = timed(split)
        res[f"split_ce{f}_sm"] = timed(lambda: split(m.copy_kernel))
    if rank == 0:
        for k, v in res.items():
            print(json.dumps({"case": k, "GBps": v, "world": world}), flush=True)
    dist.barrier(group=ctrl)


if __name__ == "__main__":
    main()
