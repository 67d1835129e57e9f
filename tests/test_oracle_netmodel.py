"""Oracle O1/O2 pinned: Fig. 5(b), closed forms, exact piecewise integration, NetUp invariants."""
import json
import os

import pytest

import synthgen as sg
from oracle.netmodel import Net, Unschedulable, component_bytes, send

GOLD = os.path.join(os.path.dirname(__file__), "golden")
S = 10**9
MB = 10**6


def one_link_net(profile):
    # node 0 -> node 1, only node 1's ingress is capped
    net = Net(2, [0, 0], [0, 1])
    net.links[("down", 1)] = tuple(tuple(x) for x in profile)
    return net


def test_fig5b_t_en_is_7s():
    g = json.load(open(os.path.join(GOLD, "fig5b_t_en.json")))
    tr = one_link_net(g["profile_ns_Bps"]).transfer(g["size_bytes"], 0, 1, g["t_avail_ns"])
    assert tr.t_en == g["expected_t_en_ns"]
    assert tr.t_st == 0


def test_closed_forms():
    net = Net(2, [0, 0], [0, 100 * MB])
    assert net.transfer(100 * MB, 0, 1, 0).t_en == 1 * S                 # size / rate
    assert net.transfer(100 * MB, 0, 1, 5 * S).t_en == 6 * S             # shifted start
    tr = one_link_net([(0, 0), (5 * S, 5 * MB)]).transfer(10 * MB, 0, 1, 0)
    assert (tr.t_st, tr.t_en) == (5 * S, 7 * S)                            # forced idle start
    assert net.transfer(1, 0, 1, 0).t_en == 10                             # ceil to the next ns
    assert net.transfer(0, 0, 1, 3).t_en == 3                              # zero bytes: no time


def test_path_is_pointwise_min():
    # SPEC.md:61 example: links (0,6),(3,3) and (0,5),(5,1) -> (0,5),(3,3),(5,1) (MB/s, s)
    net = Net(2, [1, 0], [0, 1])
    net.links[("up", 0)] = ((0, 6 * MB), (3 * S, 3 * MB))
    net.links[("down", 1)] = ((0, 5 * MB), (5 * S, 1 * MB))
    keys = net.path(0, 1)
    assert [net.path_rate(keys, t) for t in (0, 3 * S, 5 * S, 9 * S)] == [5 * MB, 3 * MB, 1 * MB, 1 * MB]
    # 15 MB + 6 MB by t=5 s, then 1 MB/s: 25 MB -> 9 s
    assert net.transfer(25 * MB, 0, 1, 0).t_en == 9 * S


def _integral(net, keys, a, b):
    """Exact integral of the path residual over [a, b) in 1e-9 byte units (independent code)."""
    pts = sorted({a, b} | {t for k in keys for (t, _) in net.profile(k) if a < t < b})
    tot = 0
    for x, y in zip(pts, pts[1:]):
        r = min(dict_rate(net.profile(k), x) for k in keys)
        tot += r * (y - x)
    return tot


def dict_rate(profile, t):
    best = None
    for (ts, r) in profile:
        if ts <= t and (best is None or ts >= best[0]):
            best = (ts, r)
    return best[1]


def test_t_en_is_earliest_finish_on_random_profiles():
    key = sg.stream_key(11, sg.KIND_MISC, 1, 0)
    c = 0
    for trial in range(300):
        net = Net(2, [1, 0], [0, 1])
        for link in (("up", 0), ("down", 1)):
            segs, t = [], 0
            for j in range(sg.randint(key, c, 1, 5)):
                c += 1
                segs.append((t, sg.randint(key, c, 0, 9) * MB + sg.randint(key, c + 7, 0, 999)))
                c += 1
                t += sg.randint(key, c, 1, 4000) * 10**6 + sg.randint(key, c + 3, 0, 999)
            c += 1
            segs[-1] = (segs[-1][0], sg.randint(key, c, 1, 9) * MB)  # last segment positive
            net.links[link] = tuple(segs)
        size = sg.randint(key, c + 1, 1, 40) * MB + sg.randint(key, c + 2, 0, 12345)
        t_avail = sg.randint(key, c + 3, 0, 3000) * 10**6
        c += 4
        tr = net.transfer(size, 0, 1, t_avail)
        keys = net.path(0, 1)
        assert _integral(net, keys, t_avail, tr.t_en) >= size * S
        assert _integral(net, keys, t_avail, tr.t_en - 1) < size * S
        # conservation of the reserved profile, exact in integers
        used = sum(r * (b - a) for a, b, r in tr.segs)
        assert size * S <= used < size * S + tr.segs[-1][2]
        # reserving leaves residual >= 0 and drains the bottleneck during the transfer
        nw = net.fork()
        nw.reserve(tr)
        assert nw.min_residual() >= 0
        for a, b, r in tr.segs:
            assert nw.path_rate(keys, a) == 0


def test_netup_sequencing_and_identity():
    net = Net(3, [0, 0, 0], [0, 0, 10 * MB])
    t1 = net.transfer(20 * MB, 0, 2, 0)
    nw = net.fork()
    nw.reserve(t1)
    t2 = nw.transfer(20 * MB, 1, 2, 0)           # shares the server bottleneck
    assert t2.t_st >= t1.t_en and t2.t_en == 4 * S
    nw0 = net.fork()
    nw0.reserve(net.transfer(0, 0, 2, 0))       # zero-byte reservation = identity
    assert nw0.links == net.links
    assert net.links == {}                      # fork is copy-on-write: original untouched


def test_same_site_zero_time_and_down_links():
    net = Net(3, [5 * MB, 5 * MB, 0], [0, 0, 5 * MB], site=[0, 1, 0])
    assert net.transfer(50 * MB, 0, 2, 7).t_en == 7
    assert net.transfer(50 * MB, 1, 2, 0).t_en == 10 * S
    dead = Net(2, [-1, 0], [0, 5 * MB])
    assert dead.dead(0, 1)
    with pytest.raises(Unschedulable):
        dead.transfer(1, 0, 1, 0)


def test_multiserver_components():
    # App. B.2: comp bytes proportional to shard weights; t_en = max; disjoint bottlenecks
    assert component_bytes(100, [1, 1]) == [50, 50]
    assert component_bytes(4 * 10, [3, 7]) == [12, 28]
    assert sum(component_bytes(12345, [2, 3, 5])) == 12345
    net = Net(3, [0, 0, 0], [0, 10 * MB, 5 * MB])
    s, nw = send(net, 0, [1, 2], [10 * MB, 10 * MB], 0)
    assert s.t_en == 2 * S                      # max(1 s, 2 s): independent bottlenecks
    s1, _ = send(net, 0, [1], [10 * MB], 0)
    assert s1.t_en == net.transfer(10 * MB, 0, 1, 0).t_en   # G = 1 degenerates
