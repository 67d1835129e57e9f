"""Oracle O3 pinned: Fig. 6 drop, Fig. 1 delay arithmetic, SJF/SPT optimality, delay invariant."""
import json
import os

import synthgen as sg
from oracle.bruteforce import best_order_sum, best_order_sum_recursive, order_t_ens
from oracle.checks import check_plan
from oracle.netmodel import Net
from oracle.ordering import DROP_EXPIRED, DROP_LOOKAHEAD, Item, deadline, order_final, order_sjf, t_en_server
from oracle.plan import plan
from tests.instances import random_instance, to_oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
S = 10**9
MB = 10**6


def test_fig6_lookahead_drops_g1():
    g = json.load(open(os.path.join(GOLD, "fig6_lookahead_drop.json")))
    net = Net(3, g["nic_up_Bps"], g["nic_down_Bps"])
    batch = [Item(0, g["sizes_bytes"][0], g["versions"][0]), Item(1, g["sizes_bytes"][1], g["versions"][1])]
    e = g["expected"]
    # the two transfer times the paper quotes
    t1 = net.transfer(batch[0].size, 0, 2, 0)
    assert t1.t_en == e["t_en_g1_alone_ns"]
    nw = net.fork()
    nw.reserve(t1)
    assert nw.transfer(batch[1].size, 1, 2, 0).t_en == e["t_en_g2_after_g1_ns"]
    assert [deadline(it.version, g["tau_max"], g["v_init"]) for it in batch] == [1, 5]
    res = order_final(net, batch, [2], [1], g["tau_max"], g["v_init"])
    assert res.order == e["order"]
    assert res.drop_reason == e["drop_reason"]
    assert res.sends[1].t_en == e["t_en_g2_final_ns"]


def test_fig1_delay_arithmetic():
    g = json.load(open(os.path.join(GOLD, "fig1_delay.json")))
    v_g = g["v_st"] - g["tau_max"] + g["u"]
    delay = (g["v_st"] + g["N_prime"]) - v_g            # R1: (v_init + p) - v(g)
    assert delay == g["expected_delay"] == g["tau_max"] + (g["N_prime"] - g["u"])
    assert deadline(v_g, g["tau_max"], g["v_st"]) == g["expected_deadline"] == g["u"]


def test_sjf_spec_example():
    # sizes {30, 10, 20} MB on one 10 MB/s bottleneck -> (10, 20, 30), t_en = 1, 3, 6 s
    net = Net(4, [0, 0, 0, 0], [0, 0, 0, 10 * MB])
    batch = [Item(0, 30 * MB), Item(1, 10 * MB), Item(2, 20 * MB)]
    r = order_sjf(net, batch, [3], [1])
    assert r.order == [1, 2, 0]
    assert [r.sends[g].t_en for g in r.order] == [1 * S, 3 * S, 6 * S]
    r2 = order_final(net, [Item(i.node, i.size, 100) for i in batch], [3], [1], 10, 100)
    assert r2.order == [1, 2, 0]                       # deadlines never bind -> Alg. 1


def test_spt_is_optimal_on_one_bottleneck_bruteforce():
    # 1||sum C_j: shortest processing time first minimises the sum of completion times;
    # with one shared server bottleneck, equal availability and non-binding deadlines
    # Alg. 2 must reach the exhaustive optimum.
    key = sg.stream_key(5, sg.KIND_MISC, 2, 0)
    c = 0
    for trial in range(60):
        n = 1 + sg.word(key, c) % 5
        c += 1
        rate = (1 + sg.word(key, c) % 9) * MB
        c += 1
        ups = []
        batch = []
        for i in range(n):
            ups.append(0 if sg.word(key, c) % 2 else rate + (sg.word(key, c + 1) % 5) * MB)
            batch.append(Item(i, (1 + sg.word(key, c + 2) % 30) * MB + sg.word(key, c + 3) % 1000, 50))
            c += 4
        net = Net(n + 1, ups + [0], [0] * n + [rate])
        res = order_final(net, batch, [n], [1], 100, 50)
        got = sum(res.sends[g].t_en for g in res.order)
        best, _ = best_order_sum(net, batch, [n], [1])
        assert got == best
        assert best_order_sum_recursive(net, batch, [n], [1]) == best
        assert order_t_ens(net, batch, [n], [1], res.order) == [res.sends[g].t_en for g in res.order]


def test_tau4_six_fresh_updates_four_commit():
    net = Net(7, [0] * 7, [0] * 6 + [10 * MB])
    batch = [Item(i, (i + 1) * MB, 20) for i in range(6)]
    res = order_final(net, batch, [6], [1], 4, 20)
    assert res.order == [0, 1, 2, 3]
    assert res.drop_reason == [0, 0, 0, 0, DROP_EXPIRED, DROP_EXPIRED]


def test_expired_at_batch_start_and_due_set_argmin():
    net = Net(4, [0, 0, 0, 0], [0, 0, 0, 10 * MB])
    # dl = v + tau - v_init: versions 10, 13, 13 with tau 3, v_init 13 -> dl = 0, 3, 3
    batch = [Item(0, MB, 10), Item(1, 5 * MB, 13), Item(2, 2 * MB, 13)]
    res = order_final(net, batch, [3], [1], 3, 13)
    assert res.drop_reason[0] == DROP_EXPIRED
    assert res.order == [2, 1]
    # two updates due at position 1: the faster one is picked, the other expires at p = 2
    batch2 = [Item(0, 5 * MB, 11), Item(1, 2 * MB, 11), Item(2, 1 * MB, 20)]
    res2 = order_final(net, batch2, [3], [1], 3, 13)   # dl = 1, 1, 10
    assert res2.order[0] == 1 and res2.drop_reason[0] == DROP_EXPIRED


def test_lookahead_can_fire_on_an_sjf_pick_with_shard_components():
    # R5's no-op argument needs t_en to be monotone in the residual.  A single transfer is;
    # an App. B.2 send whose components are reserved one after another is not.  Worked by
    # hand (units of 1e9 bytes and 1e9 B/s): W0 up 2, pair W0->B 1, A down 2; W1 up 1.
    # g0 (4, from W0): c->A at 2 on [0,1], then c->B at 1 on [1,3] -> t_en 3.
    # g1 (2.8, from W1): c->A at 1 on [0,1.4], c->B on [1.4,2.8]      -> t_en 2.8 (SJF pick).
    # After g1's reservation A's residual is 1 on [0,1.4], so g0's first component no
    # longer takes all of W0's up-link: c->A ends at 1.7, c->B runs at 1 from 0 and ends at
    # 2.3 < 2.8 -> Alg. 2's look-ahead drops the SJF pick g1 (listing line 10).
    G = 10**9
    n = 4
    bw = [0] * (n * n)
    bw[0 * n + 3] = 1 * G
    net = Net(n, [2 * G, 1 * G, 0, 0], [0, 0, 2 * G, 0], bw)
    batch = [Item(0, 4 * G, 0), Item(1, 28 * G // 10, 0)]
    s0, nw0 = t_en_server(net, batch[0], [2, 3], [1, 1])
    s1, nw1 = t_en_server(net, batch[1], [2, 3], [1, 1])
    assert (s0.t_en, s1.t_en) == (3 * S, 28 * S // 10)
    s0_after, _ = t_en_server(nw1, batch[0], [2, 3], [1, 1])
    assert s0_after.t_en == 23 * S // 10
    res = order_final(net, batch, [2, 3], [1, 1], 100, 0)
    assert res.drop_reason == [0, DROP_LOOKAHEAD] and res.order == [0]


def test_lookahead_never_fires_on_sjf_picks_single_server():
    # R5: with one server a send is one transfer, and reservations only delay it, so for an
    # SJF pick t_en(g*) <= t_en(g°, NW'): the look-ahead never fires.
    for i in range(200):
        inst = random_instance(21, i, max_n=7, max_servers=1, replica=False)
        for b in inst.batch:
            b["version"] = inst.v_init                    # dl = tau for all
        inst.tau_max = 100                                # never due before the end
        net, batch, prm = to_oracle(inst)
        if not batch:
            continue
        res = order_final(net, batch, prm.servers, prm.shard_weights or [1] * len(prm.servers), 100, inst.v_init)
        assert DROP_LOOKAHEAD not in res.drop_reason
        assert sorted(res.order) == list(range(len(batch)))


def test_sync_mode_keeps_the_list():
    # MLfabric-S: no ordering, no drops; Alg. 3 still groups the list
    for i in range(200):
        inst = random_instance(4321, i, max_n=8, replica=False)
        inst.sync_mode = 1
        net, batch, prm = to_oracle(inst)
        p = plan(net, batch, prm)
        assert p["order"] == list(range(len(batch))) and set(p["drop_reason"]) <= {0}
        assert sum(p["commit_count"]) == len(batch)


def test_delay_bound_invariant_1000_batches():
    for i in range(1000):
        inst = random_instance(1234, i, max_n=8, replica=(i % 3 == 0))
        inst.sync_mode = 0                     # the delay bound is an asynchronous-SGD notion
        net, batch, prm = to_oracle(inst)
        p = plan(net, batch, prm)
        check_plan(p, [b.version for b in batch], inst.tau_max, inst.v_init, len(inst.aggs))
