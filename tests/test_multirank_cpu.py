"""World-size-2 gloo tests of the N > 1 host logic (no GPU): every rank plans the same
batch identically (no broadcast needed), the shard split, aggregator slots and the
plan-relative traffic accounting used for the multi-GPU roofline."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from synthgen import configs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cid, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1907_00434_b200 import mlfabric as m
    from benchkit.multi import plan_traffic
    from paper_1907_00434_b200.multigpu import agg_slots_needed

    cfg = configs.config(cid, G=world, scale_S=1_000_003)
    plans = []
    v_init = v_prev = 0
    for it in range(3):
        up, down, site = configs.network(cfg, it)
        draws = configs.batch_draws(cfg, it, v_init, v_prev)
        batch = [dict(node=cfg["worker_node"][g], size=cfg["S"] * cfg["e"], **d) for g, d in enumerate(draws)]
        p = m.plan(cfg["n_nodes"], up, down, batch, cfg["servers"], site=site, aggs=cfg["aggs"],
                   replicas=cfg["replicas"], raggs=cfg["raggs"], v_init=v_init, tau_max=cfg["tau"],
                   div_max=cfg["div_max"], shard_weights=[n for (_, n) in cfg["shards"]])
        plans.append(p)
        v_prev, v_init = v_init, v_init + p["n_commit"]
    allp = [None] * world
    dist.all_gather_object(allp, plans)
    ok = all(x == allp[0] for x in allp)
    tr = {mode: plan_traffic(cfg, plans[0], mode) for mode in ("fold", "tree")}
    q.put((rank, ok, tr, agg_slots_needed(cfg, world), plans[0]))
    dist.destroy_process_group()


@pytest.mark.parametrize("cid", [3, 4, 5])
def test_two_ranks_plan_identically(cid):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cid, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(r[1] for r in res)
    cfg = configs.config(cid, G=world, scale_S=1_000_003)
    tr = res[0][2]
    for mode in ("fold", "tree"):
        # every NVLink byte leaves one GPU and enters another
        assert sum(tr[mode]["nv_in"]) == sum(tr[mode]["nv_out"])
    pd = res[0][4]
    committed = pd["n_commit"]
    # fold mode: each committed update crosses NVLink except the slice its home shard keeps
    e, S = cfg["e"], cfg["S"]
    home = cfg["home"]
    sl = [n for (_, n) in cfg["shards"]]
    expect = sum(S * e - sl[home[g]] * e for g in pd["order"])
    if pd["replica_boundary_commit"] >= 0:
        expect += sum(sl) * 4
    assert sum(tr["fold"]["nv_in"]) == expect
    assert res[0][3] >= 1 and committed > 0


def test_shard_bounds_aligned_and_cover():
    for S in (1, 63, 64, 1000, 143_667_240, 100_000_000, 25_600_000):
        for G in (1, 2, 4, 8):
            b = configs.shard_bounds(S, G)
            assert sum(n for _, n in b) == S
            assert all(x % 64 == 0 for x, _ in b)
            ne = [x for x in b if x[1] > 0]
            assert ne[0][0] == 0 and all(ne[i][0] + ne[i][1] == ne[i + 1][0] for i in range(len(ne) - 1))
