"""O1/O2 — network model, t_en water-filling and NetUp reservation.  TEST INFRASTRUCTURE.

Paper passages:
* The network is G = (V, E) with link capacities B(e) and fixed paths P(v1, v2)
  that may share links (App. B.1).
* t_en: "compute each single update's transfer completion time, t_en, by
  factoring in the bottleneck bandwidth the transfer has available over time,
  and determining how the bytes in the update are transferred by maximally
  using bottleneck capacity at any time" (§5.1.1; Fig. 5(b)
  P:863-866: 30 MB on the residual profile -> t_en = 7).
* NetUp: "reserve capacity on its path over time; the amount of reservation
  equals the time-varying bottleneck bandwidth, and reservation duration equals
  the transfer completion time" (Fig. 5(c)).

Readings:
* R8  integer time: ns, bytes, bytes/s; delivered bytes over dt ns at r B/s are
      r*dt in units of 1e-9 byte; t_en = t_k + ceil(remaining / r).  Python ints
      are exact, so there is no tolerance anywhere.
* R9  links = per-node NIC up / NIC down plus optional per-pair caps; path i->j is
      [up(i), pair(i,j), down(j)] minus uncapped (0) entries; a negative capacity
      is a link that is down (rate 0 forever); same node or same site id -> the
      transfer takes zero time and reserves nothing.
* A transfer is contiguous: it starts at the first instant >= t_avail where the
  path residual is positive and uses the full path residual R(t) =
  min over path links until the bytes are sent (S:108 no pre-emption).
* App. B.2 multi-server: an update to |S| shards has one component per shard;
  components are reserved sequentially in shard order and t_en(g) is the max
  (reading R11).

Parity: pinned by Fig. 5(b) (t_en = 7 s), closed forms (size/rate, forced-idle
start), brute-force numeric integration on random profiles and conservation
(tests/test_oracle_netmodel.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

NS_PER_S = 10**9


class Unschedulable(Exception):
    """The path's residual is zero forever after t_avail."""


def ceil_div(a: int, b: int) -> int:
    return -((-a) // b)


@dataclass
class Transfer:
    src: int
    dst: int
    size: int
    t_avail: int
    t_st: int
    t_en: int
    path: tuple = ()
    segs: tuple = ()          # ((a, b, r), ...) with r > 0: the rate used on [a, b)


@dataclass
class Net:
    """Residual bandwidth of every link as a piecewise-constant profile.

    A profile is a tuple of (t_start_ns, rate_Bps) with t_start strictly
    increasing and the first at 0; the last segment extends to +infinity.
    Profiles are immutable tuples, so fork() (a shallow dict copy) is a
    copy-on-write snapshot.
    """
    n_nodes: int
    nic_up: list
    nic_down: list
    bw: list | None = None         # n*n pair caps, 0 = uncapped
    site: list | None = None       # co-location ids
    links: dict = field(default_factory=dict)

    # ------------------------------------------------------------ topology
    def capacity(self, key) -> int:
        if key[0] == "up":
            return self.nic_up[key[1]]
        if key[0] == "down":
            return self.nic_down[key[1]]
        return self.bw[key[1] * self.n_nodes + key[2]]

    def profile(self, key) -> tuple:
        p = self.links.get(key)
        if p is None:
            p = ((0, max(self.capacity(key), 0)),)   # capacity < 0: link down (rate 0)
        return p

    def same_site(self, src: int, dst: int) -> bool:
        if src == dst:
            return True
        return self.site is not None and self.site[src] == self.site[dst]

    def path(self, src: int, dst: int):
        """Link keys of the fixed path src->dst; None = zero-time transfer."""
        if self.same_site(src, dst):
            return None
        keys = []                                  # capacity 0 = uncapped (not on the path)
        if self.nic_up[src] != 0:
            keys.append(("up", src))
        if self.bw is not None and self.bw[src * self.n_nodes + dst] != 0:
            keys.append(("pair", src, dst))
        if self.nic_down[dst] != 0:
            keys.append(("down", dst))
        return tuple(keys) if keys else None

    def fork(self) -> "Net":
        return Net(self.n_nodes, self.nic_up, self.nic_down, self.bw, self.site, dict(self.links))

    # ------------------------------------------------------------ profiles
    @staticmethod
    def rate_at(profile: tuple, t: int) -> int:
        r = profile[0][1]
        for (ts, rs) in profile:
            if ts <= t:
                r = rs
            else:
                break
        return r

    def path_rate(self, keys, t: int) -> int:
        return min(self.rate_at(self.profile(k), t) for k in keys)

    def breakpoints_after(self, keys, t: int) -> list:
        pts = set()
        for k in keys:
            for (ts, _) in self.profile(k):
                if ts > t:
                    pts.add(ts)
        return sorted(pts)

    # ------------------------------------------------------------ O1: t_en
    def transfer(self, size: int, src: int, dst: int, t_avail: int) -> Transfer:
        """Water-fill `size` bytes along the path from t_avail (Fig. 5(b))."""
        keys = self.path(src, dst)
        if size == 0 or keys is None:
            return Transfer(src, dst, size, t_avail, t_avail, t_avail, (), ())
        need = size * NS_PER_S                      # in units of 1e-9 byte
        times = [t_avail] + self.breakpoints_after(keys, t_avail)
        segs = []
        t_st = None
        for i, a in enumerate(times):
            b = times[i + 1] if i + 1 < len(times) else None
            r = self.path_rate(keys, a)
            if r == 0:
                continue
            if t_st is None:
                t_st = a
            if b is None or r * (b - a) >= need:
                t_en = a + ceil_div(need, r)
                segs.append((a, t_en, r))
                return Transfer(src, dst, size, t_avail, t_st, t_en, keys, tuple(segs))
            need -= r * (b - a)
            segs.append((a, b, r))
        raise Unschedulable(f"path {src}->{dst} has zero residual forever after t={t_avail}")

    # ------------------------------------------------------------ O2: NetUp
    @staticmethod
    def _subtract(profile: tuple, a: int, b: int, r: int) -> tuple:
        """profile - r on [a, b); asserts the residual stays >= 0."""
        pts = sorted({ts for ts, _ in profile} | {a, b})
        out = []
        for t in pts:
            rate = Net.rate_at(profile, t)
            if a <= t < b:
                rate -= r
                assert rate >= 0, "reservation drove a residual negative"
            out.append((t, rate))
        return tuple(out)

    def reserve(self, tr: Transfer) -> None:
        """Subtract the transfer's rate profile from every link of its path (in place)."""
        for k in tr.path:
            p = self.profile(k)
            for (a, b, r) in tr.segs:
                p = self._subtract(p, a, b, r)
            self.links[k] = p

    def dead(self, src: int, dst: int) -> bool:
        """True if the path has zero rate forever (some link is down)."""
        keys = self.path(src, dst)
        return keys is not None and any(self.capacity(k) < 0 for k in keys)

    def min_residual(self) -> int:
        return min((r for p in self.links.values() for (_, r) in p), default=0)


# ---------------------------------------------------------------- App. B.2
def component_bytes(size: int, weights) -> list:
    """Split `size` bytes into |S| components proportional to shard element counts.

    comp_j = floor(size*cum_{j+1}/W) - floor(size*cum_j/W), W = sum(weights).
    With size = e * W (a dense update of e-byte elements) comp_j = e * weights[j].
    """
    W = sum(weights)
    out, cum = [], 0
    for w in weights:
        lo = size * cum // W
        cum += w
        out.append(size * cum // W - lo)
    return out


@dataclass
class Send:
    """A (possibly multi-component) transfer of one update/aggregate."""
    t_st: int
    t_en: int
    parts: list


def send(net: Net, src: int, dsts, sizes, t_avail: int) -> tuple:
    """t_en of a multi-component transfer and the network after NetUp.

    Components reserved sequentially in destination order on a fork of `net`;
    t_en = max over components (R11).  Returns (Send, new_net).
    """
    scratch = net.fork()
    parts = []
    for d, s in zip(dsts, sizes):
        tr = scratch.transfer(s, src, d, t_avail)
        scratch.reserve(tr)
        parts.append(tr)
    t_st = min(p.t_st for p in parts)
    t_en = max(p.t_en for p in parts)
    return Send(t_st, t_en, parts), scratch
