"""Oracle O4 pinned: the Fig. 7 caption instance, the n = |U| degeneracy, brute-force bounds."""
import json
import os

from oracle.aggregation import det_agg, plan_aggregation
from oracle.bruteforce import best_partition, compositions, eval_partition
from oracle.netmodel import Net
from oracle.ordering import Item, order_final
from tests.instances import random_instance, to_oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def fig7():
    g = json.load(open(os.path.join(GOLD, "fig7_partition.json")))
    net = Net(len(g["nic_up_Bps"]), g["nic_up_Bps"], g["nic_down_Bps"])
    items = [Item(i, g["size_bytes"]) for i in range(g["workers"])]
    return g, net, items


def test_fig7_totals_per_case():
    g, net, items = fig7()
    totals = [det_agg(n, items, net, [g["server"]], [1], g["aggs"]).total for n in range(7)]
    assert totals == g["expected"]["totals_ns"]


def test_fig7_chosen_partition():
    g, net, items = fig7()
    case = plan_aggregation(items, net, [g["server"]], [1], g["aggs"])
    assert case.n == g["expected"]["n_star"]
    assert [c.members for c in case.commits] == g["expected"]["groups"]
    assert [c.group for c in case.commits] == g["expected"]["group_ids"]
    # "u6 is not added to G2": u6 would reach A1 at 3.75 s > t_max = 3 s
    assert case.member_arrivals[3] == 1_250_000_000 and case.member_arrivals[4] == 2_500_000_000


def test_all_direct_case_reproduces_alg2_schedules():
    # n = |U|: DetAgg on the batch-start network (R10) reproduces Alg. 2's schedules
    for i in range(150):
        inst = random_instance(77, i, max_n=7, replica=False)
        net, batch, prm = to_oracle(inst)
        w = prm.shard_weights or [1] * len(prm.servers)
        ores = order_final(net, batch, prm.servers, w, prm.tau_max, prm.v_init)
        items = [batch[g] for g in ores.order]
        case = det_agg(len(items), items, net, prm.servers, w, prm.aggs)
        assert [c.send.t_en for c in case.commits] == [ores.sends[g].t_en for g in ores.order]


def test_heuristic_bounded_below_by_bruteforce():
    ratios = []
    for i in range(120):
        inst = random_instance(99, i, max_n=5, replica=False)
        net, batch, prm = to_oracle(inst)
        w = prm.shard_weights or [1] * len(prm.servers)
        items = list(batch)
        if not items:
            continue
        case = plan_aggregation(items, net, prm.servers, w, prm.aggs)
        # the chosen case's own partition, re-evaluated without the greedy rule, gives its total
        sizes = tuple(len(c.members) for c in case.commits if c.group > 0)
        assert eval_partition(items, net, prm.servers, w, prm.aggs, case.n, sizes)[0] == case.total
        best = best_partition(items, net, prm.servers, w, prm.aggs)
        assert best[0] <= case.total
        ratios.append(case.total / best[0] if best[0] else 1.0)
    assert min(ratios) >= 1.0


def test_compositions_enumerator():
    assert sorted(compositions(3, 2)) == [(1, 2), (2, 1), (3,)]
    assert list(compositions(0, 2)) == [()]
    assert len(list(compositions(5, 5))) == 16
