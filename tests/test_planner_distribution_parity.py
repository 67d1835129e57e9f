"""mlf_plan_distribution (C++, NEXT-4) vs oracle/distribution.py: every output equal.

Host logic only (no GPU)."""
import pytest

from oracle.distribution import plan_distribution as oracle_dist
from oracle.netmodel import Unschedulable
from paper_1907_00434_b200 import mlfabric as m
from tests.instances import random_instance, to_oracle

E_UNSCHEDULABLE = 4


def both(inst, model_bytes):
    net, batch, prm = to_oracle(inst)
    nodes = [b.node for b in batch]
    try:
        o = oracle_dist(net, nodes, model_bytes, prm.servers, prm.shard_weights, prm.aggs)
        oerr = None
    except Unschedulable:
        o, oerr = None, E_UNSCHEDULABLE
    try:
        c = m.plan_distribution(inst.n_nodes, inst.nic_up, inst.nic_down, nodes, inst.servers, model_bytes,
                                bw=inst.bw, site=inst.site, distributors=inst.aggs,
                                shard_weights=inst.shard_weights)
        cerr = None
    except m.MlfError as e:
        c, cerr = None, int(str(e).split()[2].rstrip(":"))
    return o, oerr, c, cerr


def same(o, c):
    return (o.order == c["order"] and o.group == c["group"] and o.n_direct == c["n_direct"]
            and len(o.group_node) == c["n_groups"] and o.group_node == c["group_node"]
            and o.t_total == c["t_total_ns"] and o.t_recv == c["t_recv_ns"] and o.t_start == c["t_start_ns"]
            and o.t_dist == c["t_dist_ns"])


@pytest.mark.parametrize("seed", [11, 12])
def test_random_distribution_plans_bit_exact(seed):
    n_ok = 0
    for i in range(500):
        inst = random_instance(seed * 1000 + 3, i, max_n=8, replica=False, allow_down=(i % 7 == 0))
        sizes = [b["size"] for b in inst.batch]
        model_bytes = max(sizes) if sizes else 1_000_000
        o, oerr, c, cerr = both(inst, model_bytes)
        assert oerr == cerr, (i, oerr, cerr)
        if o is not None:
            assert same(o, c), (i, o, c)
            n_ok += 1
    assert n_ok > 350


def test_larger_distribution_plans_bit_exact():
    for i in range(10):
        inst = random_instance(777, i, max_n=40, max_servers=3, replica=False)
        inst.batch = (inst.batch * 8)[:40]
        o, oerr, c, cerr = both(inst, 5_000_000)
        assert oerr == cerr
        if o is not None:
            assert same(o, c), i


def test_box_model_prefers_direct_pulls():
    # one B200 box (nodes = GPUs, NVLink NICs both ways, PS shards on every GPU): every
    # distributor would add a second hop over the same NICs, so Alg. 3 picks n* = |U|
    G, B = 4, 770_000_000_000
    reqs = [g for g in range(G) for _ in range(16)]
    c = m.plan_distribution(G, [B] * G, [B] * G, reqs, list(range(G)), 574_668_960, site=list(range(G)),
                            distributors=[2, 0, 3, 1])
    assert c["n_direct"] == len(reqs) and c["n_groups"] == 0


def test_degraded_server_uses_a_distributor():
    # node 0's egress degraded to a tenth: the model reaches node 0's requesters faster
    # through a distributor, and the plan says so
    G, B = 4, 770_000_000_000
    up = [B // 10, B, B, B]
    reqs = [0, 1, 2, 3]
    c = m.plan_distribution(G, up, [B] * G, reqs, [0], 1_000_000_000, site=list(range(G)),
                            distributors=[1])
    o = oracle_dist(to_net(G, up, [B] * G, list(range(G))), reqs, 1_000_000_000, [0], None, [1])
    assert same(o, c)
    assert c["n_groups"] == 1


def to_net(n, up, down, site):
    from oracle.netmodel import Net
    return Net(n, list(up), list(down), None, site)
