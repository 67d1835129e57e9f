"""Debug: the fused commit (bulk / ldg, each tile) with and without concurrent work on a
side stream (copy-engine memcpy, or the library's TMA copy kernel), compared bitwise."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1907_00434_b200 import mlfabric as m  # noqa: E402


def run(S, W, impl, tile, side):
    os.environ["MLF_COMMIT_IMPL"] = impl
    if tile:
        os.environ["MLF_BULK_TILE"] = str(tile)
    else:
        os.environ.pop("MLF_BULK_TILE", None)
    dev = torch.device("cuda", 0)
    slots = torch.empty((W, S), dtype=torch.float32, device=dev)
    for w in range(W):
        m.synth_fill(0, slots[w].data_ptr(), S, dtype=m.MLF_F32, seed=7, kind=1, a=w, b=0)
    wt = torch.empty(S, dtype=torch.float32, device=dev)
    m.synth_fill(0, wt.data_ptr(), S, dtype=m.MLF_F32, seed=7, kind=2)
    big_src = torch.ones(1 << 28, dtype=torch.float32, device=dev)
    big_dst = torch.empty_like(big_src)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    side_s = torch.cuda.Stream()
    ctx = m.Context(device=0, model_shard=wt, update_slots=[slots[w] for w in range(W)], lr=0.01, model_elems=S,
                    stream=st.cuda_stream)
    plan = {"n_commit": W, "order": list(range(W)), "drop_reason": [0] * W, "group": [0] * W, "n_direct": W,
            "n_groups": 0, "group_node": [], "n_server_commits": W, "commit_first": list(range(W)),
            "commit_count": [1] * W, "replica_boundary_commit": -1, "n_punted": 0, "punted": []}
    pb = m.plan_from_dict(plan)
    for w in range(W):
        ctx.submit(w, 0)
    if side == "ce":
        for _ in range(8):
            m.copy_engine(0, big_dst.data_ptr(), big_src.data_ptr(), big_src.numel() * 4, side_s.cuda_stream)
    elif side == "tma":
        for _ in range(8):
            m.copy_bulk(0, big_dst.data_ptr(), big_src.data_ptr(), big_src.numel() * 4, side_s.cuda_stream)
    ctx.execute(pb)
    ctx.sync()
    torch.cuda.synchronize()
    ctx.close()
    return wt


def main():
    S, W = 16_777_216, 32
    ref = run(S, W, "ldg", 0, "none")
    for impl, tile in (("bulk", 1024), ("bulk", 2048), ("bulk", 4096), ("ldg", 0)):
        for side in ("none", "ce", "tma"):
            got = run(S, W, impl, tile, side)
            bad = int((got.view(torch.int32) != ref.view(torch.int32)).sum())
            print(f"impl={impl} tile={tile} side={side} mismatches={bad}", flush=True)


if __name__ == "__main__":
    main()
