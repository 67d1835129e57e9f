"""C++ planner (mlf_plan through the C ABI) vs the oracle: every integer output equal.

Host logic only (no GPU): mlf_plan is pure host C++.
"""
import json
import math
import os

import pytest

from oracle.plan import PlanError, plan as oracle_plan
from paper_1907_00434_b200 import mlfabric as m
from tests.instances import random_instance, to_oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def cpp_plan(inst):
    return m.plan(inst.n_nodes, inst.nic_up, inst.nic_down, inst.batch, inst.servers, bw=inst.bw, site=inst.site,
                  aggs=inst.aggs, replicas=inst.replicas, raggs=inst.raggs, v_init=inst.v_init,
                  tau_max=inst.tau_max, div_max=inst.div_max, gamma=inst.gamma, hist_norm=inst.hist_norm,
                  carried=inst.carried, shard_weights=inst.shard_weights, replica_mode=inst.replica_mode,
                  sync_mode=inst.sync_mode)


def both(inst):
    try:
        o = oracle_plan(*to_oracle(inst))
        oerr = None
    except PlanError as e:
        o, oerr = None, e.code
    try:
        c = cpp_plan(inst)
        cerr = None
    except m.MlfError as e:
        c, cerr = None, e.code
    return o, oerr, c, cerr


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_random_instances_bit_exact(seed):
    n_err = 0
    for i in range(750):
        inst = random_instance(seed * 1000 + 7, i, max_n=8, allow_down=(i % 5 == 0))
        o, oerr, c, cerr = both(inst)
        assert oerr == cerr, (i, oerr, cerr)
        n_err += oerr is not None
        if o is not None:
            assert o == c, i
    assert n_err < 750 * 0.3


def test_larger_instances_bit_exact():
    for i in range(12):
        inst = random_instance(555, i, max_n=48, max_servers=3)
        o, oerr, c, cerr = both(inst)
        assert oerr == cerr
        if o is not None:
            assert o == c


@pytest.mark.slow
def test_instances_64_128():
    for i, n in enumerate((64, 64, 128)):
        inst = random_instance(909, i, max_n=n, max_servers=2)
        inst.batch = (inst.batch * 40)[:n]
        o, oerr, c, cerr = both(inst)
        assert oerr == cerr
        if o is not None:
            assert o == c


def test_paper_examples_through_cpp():
    g = json.load(open(os.path.join(GOLD, "fig6_lookahead_drop.json")))
    batch = [dict(node=i, size=g["sizes_bytes"][i], version=g["versions"][i], t_avail=0, norm=0.0) for i in range(2)]
    p = m.plan(3, g["nic_up_Bps"], g["nic_down_Bps"], batch, [2], tau_max=g["tau_max"], v_init=g["v_init"])
    assert p["order"] == g["expected"]["order"] and p["drop_reason"] == g["expected"]["drop_reason"]
    assert p["commit_t_ns"] == [g["expected"]["t_en_g2_final_ns"]]
    f = json.load(open(os.path.join(GOLD, "fig7_partition.json")))
    batch = [dict(node=i, size=f["size_bytes"], version=0, t_avail=0, norm=0.0) for i in range(6)]
    p = m.plan(9, f["nic_up_Bps"], f["nic_down_Bps"], batch, [f["server"]], aggs=f["aggs"], tau_max=10)
    assert p["n_direct"] == f["expected"]["n_star"]
    per_update = [gid for gid, grp in zip(f["expected"]["group_ids"], f["expected"]["groups"]) for _ in grp]
    assert p["group"] == per_update == [0, 0, 0, 1, 1, 2]
    assert p["commit_count"] == [len(x) for x in f["expected"]["groups"]]
    assert p["t_total_ns"] == 5_000_000_000


def test_errors():
    with pytest.raises(m.MlfError) as e:
        m.plan(2, [0, 0], [0, 5], [dict(node=5, size=1, version=0, t_avail=0, norm=0.0)], [1])
    assert e.value.code == m.MLF_E_INVALID
    with pytest.raises(m.MlfError) as e:
        m.plan(2, [-1, 0], [0, 5], [dict(node=0, size=1, version=0, t_avail=0, norm=0.0)], [1])
    assert e.value.code == m.MLF_E_UNSCHEDULABLE
    with pytest.raises(m.MlfError) as e:
        m.plan(2, [0, 0], [0, 5], [], [1], gamma=1.5)
    assert e.value.code == m.MLF_E_INVALID
    p = m.plan(2, [0, 0], [0, 5], [], [1], div_max=math.inf)
    assert p["n_commit"] == 0 and p["t_total_ns"] == 0


def test_library_exports_every_declared_symbol():
    import re
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "mlfabric.h")).read()
    declared = set(re.findall(r"\b(mlf_[a-z_0-9]+)\s*\(", hdr))
    assert declared == set(m.EXPORTS)
    for s in declared:
        assert hasattr(m.lib(), s)


def test_lookahead_fires_on_sjf_pick_through_cpp():
    # the multi-component instance of tests/test_oracle_ordering.py, through mlf_plan
    G = 10**9
    n = 4
    bw = [0] * (n * n)
    bw[0 * n + 3] = 1 * G
    batch = [dict(node=0, size=4 * G, version=0, t_avail=0, norm=0.0),
             dict(node=1, size=28 * G // 10, version=0, t_avail=0, norm=0.0)]
    p = m.plan(n, [2 * G, 1 * G, 0, 0], [0, 0, 2 * G, 0], batch, [2, 3], bw=bw, tau_max=100)
    assert p["drop_reason"] == [0, 2] and p["order"] == [0]
