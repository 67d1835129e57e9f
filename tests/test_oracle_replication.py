"""Oracle O5 pinned: Eq. 9 coefficients and example, soundness on true momentum vectors,
Eq. 6-8 reordering, Div_max limits, mirror-boundary consistency."""
import json
import math
import os

import numpy as np

from oracle.plan import plan
from oracle.replication import divergence_bound
from tests.instances import random_instance, to_oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def momentum_run(w_prev, w0, updates, gamma):
    """Eq. 2: w_{t+1} = w_t + u + gamma (w_t - w_{t-1}), applied in order."""
    a, b = w_prev.copy(), w0.copy()
    for u in updates:
        a, b = b, b + u + gamma * (b - a)
    return b


def test_eq9_golden():
    g = json.load(open(os.path.join(GOLD, "eq9_divergence.json")))
    d = divergence_bound(g["lead_norms"], g["gamma"], g["hist_norm"])
    assert math.isclose(d, g["expected_bound"], rel_tol=1e-12)
    c = g["expected_coefficients"]
    # coefficients recovered by probing with unit norms in one slot at a time
    assert math.isclose(divergence_bound([0.0, 0.0], g["gamma"], 1.0), c["h0"], rel_tol=1e-12)
    assert math.isclose(divergence_bound([1.0, 0.0], g["gamma"], 0.0), c["u1"], rel_tol=1e-12)
    assert math.isclose(divergence_bound([0.0, 1.0], g["gamma"], 0.0), c["u2"], rel_tol=1e-12)
    assert divergence_bound([3.0, 4.0], 0.0, 9.0) == 7.0       # gamma = 0: sum of lead norms
    assert divergence_bound([], 0.9, 5.0) == 0.0


def test_coefficients_match_momentum_recurrence_and_bound_is_sound():
    rng = np.random.default_rng(0)
    for trial in range(200):
        gamma = float(rng.choice([0.0, 0.3, 0.9, 0.99]))
        m = int(rng.integers(1, 7))
        d = 16
        w_prev = rng.normal(size=d)
        h0 = rng.normal(size=d) * rng.uniform(0, 2)
        w0 = w_prev + h0
        us = [rng.normal(size=d) * rng.uniform(0, 3) for _ in range(m)]
        ws = momentum_run(w_prev, w0, us, gamma)
        # exact expansion: (sum_{j=1..m} g^j) h0 + sum_i (sum_{j=0..m-i} g^j) u_i
        exp = sum(gamma**j for j in range(1, m + 1)) * h0
        for i, u in enumerate(us, start=1):
            exp = exp + sum(gamma**j for j in range(0, m - i + 1)) * u
        assert np.allclose(ws - w0, exp, atol=1e-9)
        bound = divergence_bound([float(np.linalg.norm(u)) for u in us], gamma, float(np.linalg.norm(h0)))
        assert np.linalg.norm(ws - w0) <= bound * (1 + 1e-12) + 1e-12


def test_eq6_8_reordering_divergence():
    rng = np.random.default_rng(1)
    gamma = 0.9
    w_prev, w0 = rng.normal(size=8), rng.normal(size=8)
    u1, u2 = rng.normal(size=8), rng.normal(size=8)
    ws = momentum_run(w_prev, w0, [u1, u2], gamma)
    wr = momentum_run(w_prev, w0, [u2, u1], gamma)
    assert np.allclose(ws - wr, gamma * (u1 - u2), atol=1e-12)


def _replica_instances(n, seed):
    out = []
    i = 0
    while len(out) < n:
        inst = random_instance(seed, i, max_n=7, replica=True)
        i += 1
        if inst.replicas:
            out.append(inst)
    return out


def test_replica_trees_mode_freezes_exactly_the_replica_commits():
    for inst in _replica_instances(150, 777):
        inst.replica_mode = 1
        net, batch, prm = to_oracle(inst)
        p = plan(net, batch, prm)
        total = len(inst.carried) + p["n_commit"]
        assert p["replica_boundary_commit"] == -1
        assert p["replica_frozen"] == sum(p["replica_commit_count"])
        assert p["replica_commit_first"] == [sum(p["replica_commit_count"][:i])
                                             for i in range(p["n_replica_commits"])]
        assert p["punted"] == list(range(p["replica_frozen"], total))
        # the same plan in mirror mode freezes a superset (rounded up to a server commit)
        inst.replica_mode = 0
        pm = plan(*to_oracle(inst))
        assert pm["replica_frozen"] >= p["replica_frozen"]
        assert pm["order"] == p["order"] and pm["replica_bytes"] == p["replica_bytes"]


def test_divmax_limits_and_mirror_consistency():
    for inst in _replica_instances(150, 4242):
        inst.replica_mode = 0
        # Div_max = inf: the bound never binds, so no server delay
        inst.div_max = math.inf
        net, batch, prm = to_oracle(inst)
        p = plan(net, batch, prm)
        assert p["delayed_last"] == 0
        total = len(inst.carried) + p["n_commit"]
        assert p["replica_frozen"] + p["n_punted"] == total
        assert p["punted"] == list(range(p["replica_frozen"], total))
        # Div_max = 0, gamma = 0: lead must be empty at T_last unless all lead norms are 0
        inst.div_max, inst.gamma = 0.0, 0.0
        net, batch, prm = to_oracle(inst)
        p = plan(net, batch, prm)
        items = list(prm.carried) + [batch[g] for g in p["order"]]
        lead = [it.norm for it in items[p["replica_frozen"]:]]
        assert divergence_bound(lead, 0.0, 0.0) == 0.0
        # the mirror boundary covers exactly replica_frozen items
        b = p["replica_boundary_commit"]
        nc = len(inst.carried)
        if b == -1:
            assert p["replica_frozen"] == 0
        elif b == 0:
            assert p["replica_frozen"] == nc
        else:
            assert p["replica_frozen"] == nc + sum(p["commit_count"][:b])
            assert b <= p["n_server_commits"]


def test_delayed_last_commit_hand_worked():
    # §5.3's delay of the last server commit (reading R15b), worked by hand.
    # Nodes: W0, W1 (up 10 MB/s), server S (down 10 MB/s), replica R (down 5 MB/s); two
    # fresh 10 MB updates, no aggregators, gamma 0, unit norms (count-style Div_max).
    # Server plan: g0 on [0,1] s, g1 on [1,2] s -> T_last = 2 s.  Replica plan on the network
    # after the server's reservations: g0 -> R waits for W0's up-link, runs at 5 MB/s on
    # [1,3]; g1 -> R gets 5 MB by 1 s, is blocked by g0 on R's down-link until 3, then
    # finishes on [3,4] -> replica commit times 3 s, 4 s; nothing is frozen by T_last.
    from oracle.plan import Item, Params, make_net
    from paper_1907_00434_b200 import mlfabric as m
    MB, S = 10**6, 10**9
    up, down = [10 * MB, 10 * MB, 0, 0], [0, 0, 10 * MB, 5 * MB]
    batch = [Item(0, 10 * MB, 7, 0, 1.0), Item(1, 10 * MB, 7, 0, 1.0)]
    cases = {
        # Div_max: (replica_frozen, boundary, punted, delayed_last, commit_t_ns)
        0.0: (2, 2, [], 1, [1 * S, 5 * S]),   # a_e = replica commit 2 (at 4 s): g1 starts at 4, ends 5
        1.0: (1, 1, [1], 1, [1 * S, 4 * S]),  # a_e = replica commit 1 (at 3 s): g1 starts at 3, ends 4
        2.0: (0, -1, [0, 1], 0, [1 * S, 2 * S]),  # the lead of 2 is within Div_max: no delay
    }
    for div_max, (frozen, boundary, punted, delayed, times) in cases.items():
        prm = Params(servers=[2], replicas=[3], v_init=7, tau_max=10, div_max=div_max)
        p = plan(make_net(4, up, down), batch, prm)
        assert p["order"] == [0, 1] and p["commit_t_ns"] == times, (div_max, p["commit_t_ns"])
        assert (p["replica_frozen"], p["replica_boundary_commit"], p["punted"], p["delayed_last"]) == \
            (frozen, boundary, punted, delayed), div_max
        assert p["t_total_ns"] == times[-1]
        c = m.plan(4, up, down, [dict(node=it.node, size=it.size, version=7, t_avail=0, norm=1.0) for it in batch],
                   [2], replicas=[3], v_init=7, tau_max=10, div_max=div_max)
        assert {k: c[k] for k in p} == p
