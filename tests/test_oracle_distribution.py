"""Oracle NEXT-4 (App. B.3 model distribution trees) pinned: closed forms, transposition,
symmetry with Alg. 3, and feasibility of the real-time schedule on the real network."""
from oracle.aggregation import plan_aggregation
from oracle.distribution import plan_distribution, transpose
from oracle.netmodel import NS_PER_S, Net
from oracle.ordering import Item, order_sjf
from tests.instances import random_instance, to_oracle

B = 1_000_000_000          # 1 GB/s
M = 1_000_000_000          # 1 GB model -> 1 s at B


def star():
    # node 0 server, node 1 distributor (4B both ways), nodes 2..5 workers (B both ways)
    up = [B, 4 * B, B, B, B, B]
    down = [B, 4 * B, B, B, B, B]
    return Net(6, up, down)


def test_star_one_distributor_closed_form():
    # server -> D in 1 s (server up B), then D -> 4 workers in parallel in 1 s (D up 4B):
    # T = 2 s against 4 s for four direct pulls through the server's up-link
    p = plan_distribution(star(), [2, 3, 4, 5], M, [0], None, [1])
    assert p.n_direct == 0 and p.group == [1, 1, 1, 1] and p.group_node == [1]
    assert p.t_total == 2 * NS_PER_S
    assert p.t_dist == [1 * NS_PER_S]
    assert p.t_recv == [2 * NS_PER_S] * 4


def test_no_distributors_is_sequential_server_uplink():
    # k° = 0: every request direct; the server's up-link serves them one after another
    p = plan_distribution(star(), [2, 3, 4, 5], M, [0], None, [])
    assert p.n_direct == 4 and p.group == [0, 0, 0, 0]
    assert p.t_total == 4 * NS_PER_S
    assert sorted(p.t_recv) == [1 * NS_PER_S, 2 * NS_PER_S, 3 * NS_PER_S, 4 * NS_PER_S]
    # "we first transfer ... and then proceed backwards": the first request in O is
    # served last
    assert p.t_recv[p.order[0]] == 4 * NS_PER_S and p.t_recv[p.order[-1]] == 1 * NS_PER_S


def test_pull_uses_the_server_uplink_not_its_downlink():
    # a transposition error would route pulls over the server's 1 B/s down-link
    up = [B, B, B]
    down = [1, B, B]
    p = plan_distribution(Net(3, up, down), [1, 2], M, [0], None, [])
    assert p.t_total == 2 * NS_PER_S
    # and the workers' down-links (not their up-links) bound their reception
    up2 = [4 * B, 1, 1]
    down2 = [B, B // 2, B // 2]
    p2 = plan_distribution(Net(3, up2, down2), [1, 2], M, [0], None, [])
    assert p2.t_total == 2 * NS_PER_S            # two parallel pulls at B/2 each


def test_transpose_is_an_involution_and_swaps_pairs():
    n = 3
    net = Net(n, [1, 2, 3], [4, 5, 6], [i * 10 + j for i in range(n) for j in range(n)], [0, 1, 1])
    t = transpose(net)
    assert t.nic_up == [4, 5, 6] and t.nic_down == [1, 2, 3]
    assert t.bw[0 * n + 2] == net.bw[2 * n + 0]
    tt = transpose(t)
    assert (tt.nic_up, tt.nic_down, tt.bw, tt.site) == (net.nic_up, net.nic_down, net.bw, net.site)


def test_symmetric_network_equals_alg3_aggregation():
    # up = down caps and symmetric pair caps: the transposed network is the network itself,
    # so the distribution plan is Alg. 3's aggregation plan of the same requests
    checked = 0
    for i in range(120):
        inst = random_instance(4242, i, max_n=6, replica=False, allow_pair=False)
        net, batch, prm = to_oracle(inst)
        sym = Net(net.n_nodes, list(net.nic_up), list(net.nic_up), None, net.site)
        if not batch:
            continue
        nodes = [b.node for b in batch]
        size = max(b.size for b in batch) or 1
        w = prm.shard_weights or [1] * len(prm.servers)
        p = plan_distribution(sym, nodes, size, prm.servers, prm.shard_weights, prm.aggs)
        items = [Item(x, size) for x in nodes]
        order = order_sjf(sym, items, prm.servers, w).order
        case = plan_aggregation([items[g] for g in order], sym, prm.servers, w, prm.aggs)
        assert p.order == order and p.n_direct == case.n and p.t_total == case.total
        groups = [-1] * len(nodes)
        for c in case.commits:
            for q in c.members:
                groups[order[q]] = c.group
        assert p.group == groups
        checked += 1
    assert checked > 80


def _link_keys(net: Net, src: int, dst: int):
    return net.path(src, dst) or ()


def test_real_time_schedule_is_feasible_random():
    # the returned real-time schedule respects every real link's capacity at all times,
    # delivers every byte, serves each distributor before its members, and ends by T
    checked = 0
    for i in range(200):
        inst = random_instance(9090, i, max_n=6, replica=False)
        net, batch, prm = to_oracle(inst)
        if not batch:
            continue
        nodes = [b.node for b in batch]
        size = max(b.size for b in batch)
        p = plan_distribution(net, nodes, size, prm.servers, prm.shard_weights, prm.aggs)
        T = p.t_total
        usage = {}
        for (src, dst, sz, t_st, t_en, segs) in p.schedule:
            assert 0 <= t_st <= t_en <= T
            if segs:
                # conservation: every byte delivered; the last segment is the ceil'd one
                assert sum(r * (b - a) for (a, b, r) in segs) >= sz * NS_PER_S
                assert sum(r * (b - a) for (a, b, r) in segs[1:]) < sz * NS_PER_S
                for key in _link_keys(net, src, dst):
                    usage.setdefault(key, []).extend(segs)
        for key, segs in usage.items():
            cap = net.capacity(key)
            pts = sorted({a for (a, _, _) in segs} | {b for (_, b, _) in segs})
            for t in pts:
                assert sum(r for (a, b, r) in segs if a <= t < b) <= cap, (i, key, t)
        # distributor before members, and every request no later than T
        for q, g in enumerate(p.group):
            assert g >= 0 and 0 <= p.t_start[q] <= p.t_recv[q] <= T
            if g > 0:
                assert p.t_dist[g - 1] <= p.t_start[q]
        checked += 1
    assert checked > 150
