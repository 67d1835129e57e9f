// planner.cpp — mlf_plan: MLfabric's per-batch scheduler in host C++.
//
// PAPER.md (cited P:line): §5 decomposition; Alg. 1 ShrtUp and
// t_en water-filling / NetUp (Fig. 5); deadlines;
// Alg. 2 look-ahead drop; Alg. 3 DetAgg + enumeration over n
// (P:1050-1159); App. B.2 multi-server components; §5.3
// replication with the Eq. 9/12 divergence bound.
// Readings R1-R20 are in DESIGN.md §3; the integer-time model is R8: times in
// ns (int64), sizes in bytes, rates in bytes/s, byte*ns products in __int128.
// Compiled with -ffp-contract=off so the only floating point (the divergence
// bound) is evaluated exactly in the documented order.
//
// Performance (planning is O(#U^2 * G) transfer evaluations).  Every item
// below is exact — the plan equals the plain sequential one bit for bit (scripts/planbench
// replays 3074 instances; tests/ compares plans with the CPU oracle):
//  * a candidate's tentative reservation is never materialised: evaluations read the residual
//    as the link's step profile minus the pending reservations (step profiles too), walked
//    with cursors; a saturated link makes the walk jump to that link's next change;
//  * NetUp merges all of a link's reserved segments in one canonical pass (a canonical
//    profile is unique, so the application order never changes a later t_en);
//  * Alg. 2 caches each class's send with its walk and per-link slacks: after a reservation,
//    unchanged leading components are kept and only the rest re-evaluated, and g*'s own
//    reservation is replayed from its record; when g* is dropped, the records the look-ahead
//    overwrote are put back instead of recomputed;
//  * Alg. 3 starts each case n from Alg. 2's network after its n-th kept update (snapshots
//    every 8 kept updates plus at most 7 replayed reservations, R10), skips the cases whose
//    first tail item already fails (checked during Alg. 2), prunes cases whose running t_max
//    exceeds the best total, and runs the rest as independent tasks;
//  * each ShrtUp/ShrtDline scan's classes and the #U+1 DetAgg cases ("can be parallelized",
//    P:1664-1668) run on a thread pool, reduced in index order (ties -> lowest index, R6/R14).
#include "planner.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <utility>
#include <vector>

namespace mlf {

using i64 = int64_t;
using i128 = __int128;
static constexpr i64 NS_PER_S = 1000000000LL;
static constexpr i64 T_INF = std::numeric_limits<i64>::max();
static constexpr i64 T_LIMIT = std::numeric_limits<i64>::max() / 4;   // time overflow guard

struct PlanFail {
  mlf_status code;
  std::string msg;
};

// ---------------------------------------------------------------- thread pool
// Persistent workers; run(n, f) calls f(i) for i in [0, n) and returns when all
// are done.  Concurrent callers (mlf_plan is reentrant) fall back to serial.
// Items are claimed from one atomic word (job generation << 32 | next item), so a job ends
// when its items are done, not when every worker has checked in: a worker that is asleep or
// late simply finds nothing left (the caller takes every item itself if need be), and a late
// claim can never hit the next job (its generation differs, the CAS fails).
class Pool {
 public:
  static Pool &get() {
    static Pool p;
    return p;
  }
  int threads() const { return (int)th_.size() + 1; }
  void run(int n, const std::function<void(int)> &f, int min_parallel) {
    if (n < min_parallel || th_.empty() || !busy_.try_lock()) {
      for (int i = 0; i < n; ++i) f(i);
      return;
    }
    // the job's generations are even; first the state takes the odd one before it, so that no
    // claim still in flight for the previous job can succeed (its CAS compares against a state
    // word read before this store) while job_ and n_ are rewritten
    gen_ += 2;
    const uint64_t g = gen_;
    state_.store((g - 1) << 32, std::memory_order_seq_cst);
    job_ = &f;
    n_.store(n, std::memory_order_relaxed);
    // items per claim: few enough claims that the claim word does not bounce between cores for
    // every ~50 ns item, enough chunks to balance uneven items
    chunk_.store(std::max(1, n / (4 * threads())), std::memory_order_relaxed);
    done_.store(0, std::memory_order_relaxed);
    state_.store(g << 32, std::memory_order_seq_cst);     // publishes job_ and n_
    if (sleepers_.load(std::memory_order_seq_cst) > 0) {
      std::lock_guard<std::mutex> lk(m_);
      cv_.notify_all();
    }
    work(g);
    // items other workers claimed are still running: they take microseconds
    while (done_.load(std::memory_order_acquire) < n) relax();
    job_ = nullptr;
    busy_.unlock();
  }

 private:
  Pool() {
    // one process per GPU plans on every rank at once: share the host's cores between the
    // local ranks (torchrun's LOCAL_WORLD_SIZE), or take MLF_PLAN_THREADS as given
    unsigned hw = std::thread::hardware_concurrency();
    int total = (int)std::min<unsigned>(hw ? hw : 1, 32);
    if (const char *lw = getenv("LOCAL_WORLD_SIZE")) total = std::max(1, total / std::max(1, atoi(lw)));
    if (const char *pt = getenv("MLF_PLAN_THREADS")) total = std::max(1, std::min(32, atoi(pt)));
    int t = total - 1;
    for (int i = 0; i < t; ++i) th_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    stop_flag_.store(true, std::memory_order_seq_cst);
    {
      std::lock_guard<std::mutex> lk(m_);
      cv_.notify_all();
    }
    for (auto &t : th_) t.join();
  }
  // claim the next items [i, e) of job generation g (false: none left, or that job is over)
  bool claim(uint64_t g, int &i, int &e) {
    uint64_t s = state_.load(std::memory_order_acquire);
    for (;;) {
      const int n = n_.load(std::memory_order_relaxed), at = (int)(uint32_t)s;
      if ((s >> 32) != g || at >= n) return false;
      const int k = std::min(chunk_.load(std::memory_order_relaxed), n - at);
      if (state_.compare_exchange_weak(s, s + (uint64_t)k, std::memory_order_acq_rel, std::memory_order_acquire)) {
        i = at;
        e = at + k;
        return true;
      }
    }
  }
  void work(uint64_t g) {
    int i, e;
    while (claim(g, i, e)) {
      for (int q = i; q < e; ++q) (*job_)(q);   // valid: the job cannot end before these are done
      done_.fetch_add(e - i, std::memory_order_release);
    }
  }
  static void relax() {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      // spin for the next job (a plan's scans come back to back), then sleep
      uint64_t g = seen;
      for (int spin = 0;; ++spin) {
        if (stop_flag_.load(std::memory_order_acquire)) return;
        g = state_.load(std::memory_order_acquire) >> 32;
        if (g != seen && !(g & 1)) break;                // odd: a job is being set up
        if (spin < kSpin) {
          relax();
          continue;
        }
        std::unique_lock<std::mutex> lk(m_);
        sleepers_.fetch_add(1, std::memory_order_seq_cst);
        cv_.wait(lk, [&] {
          const uint64_t now = state_.load(std::memory_order_seq_cst) >> 32;
          return stop_flag_.load(std::memory_order_seq_cst) || (now != seen && !(now & 1));
        });
        sleepers_.fetch_sub(1, std::memory_order_seq_cst);
        spin = 0;
      }
      seen = g;
      work(g);
    }
  }
  static constexpr int kSpin = 4000;               // tens of microseconds of pause instructions
  std::vector<std::thread> th_;
  std::mutex m_, busy_;
  std::condition_variable cv_;
  const std::function<void(int)> *job_ = nullptr;
  uint64_t gen_ = 0;                               // written by the caller holding busy_ only
  alignas(64) std::atomic<uint64_t> state_{0};
  std::atomic<int> n_{0}, chunk_{1};
  alignas(64) std::atomic<int> done_{0};
  alignas(64) std::atomic<int> sleepers_{0};
  std::atomic<bool> stop_flag_{false};
};

// ---------------------------------------------------------------- network
struct Seg {
  i64 t, r;
};
using Profile = std::vector<Seg>;

struct NetDef {
  int n = 0;
  const int64_t *up = nullptr, *down = nullptr, *bw = nullptr;
  const int32_t *site = nullptr;
};

// link keys: up(i) = i, down(j) = n + j, pair(i, j) = 2n + i*n + j
struct Net {
  const NetDef *def = nullptr;
  std::vector<Profile> ud;                         // 2n up/down residual profiles
  std::unordered_map<i64, Profile> pair;           // pair links touched so far

  explicit Net(const NetDef *d) : def(d), ud(2 * d->n) {
    for (int i = 0; i < d->n; ++i) {
      ud[i] = Profile{{0, std::max<i64>(d->up[i], 0)}};
      ud[d->n + i] = Profile{{0, std::max<i64>(d->down[i], 0)}};
    }
  }
  i64 capacity(i64 key) const {
    const i64 n = def->n;
    if (key < n) return def->up[key];
    if (key < 2 * n) return def->down[key - n];
    return def->bw[key - 2 * n];
  }
  const Profile *get(i64 key) const {
    if (key < 2 * (i64)def->n) return &ud[key];
    auto it = pair.find(key);
    return it == pair.end() ? nullptr : &it->second;
  }
  Profile &mut(i64 key) {
    if (key < 2 * (i64)def->n) return ud[key];
    auto it = pair.find(key);
    if (it == pair.end()) it = pair.emplace(key, Profile{{0, std::max<i64>(capacity(key), 0)}}).first;
    return it->second;
  }
};

struct Path {
  int nk = 0;       // 0 = zero-time transfer
  i64 key[3];
};

static bool same_site(const NetDef &d, int a, int b) {
  if (a == b) return true;
  return d.site && d.site[a] == d.site[b];
}

static Path path_of(const NetDef &d, int src, int dst) {
  Path p;
  if (same_site(d, src, dst)) return p;
  const i64 n = d.n;
  if (d.up[src] != 0) p.key[p.nk++] = src;
  if (d.bw && d.bw[(i64)src * n + dst] != 0) p.key[p.nk++] = 2 * n + (i64)src * n + dst;
  if (d.down[dst] != 0) p.key[p.nk++] = n + dst;
  return p;
}

static bool path_dead(const NetDef &d, int src, int dst) {
  if (same_site(d, src, dst)) return false;
  const i64 n = d.n;
  if (d.up[src] < 0) return true;
  if (d.bw && d.bw[(i64)src * n + dst] < 0) return true;
  if (d.down[dst] < 0) return true;
  return false;
}

struct TSeg {
  i64 a, b, r;        // rate r used on [a, b)
};

// A piecewise-constant function as a canonical step profile: segment i holds value p[i].r on
// [p[i].t, p[i+1].t), p[0].t == 0, no two adjacent segments with equal values (a fully
// reserved stretch of a link is ONE zero segment, so a t_en walk skips it in one step).
// combine() adds sign * (the sum of the segments s) to p in one merge pass over the affected
// range.  The function is exactly the one of adding the segments one by one, and a canonical
// profile is unique, so the representation (hence every later t_en) does not depend on the
// order in which reservations were applied.
struct Transfer {
  i64 t_st = 0, t_en = 0;
  Path path;
  std::vector<TSeg> segs;
};

struct Ev {
  i64 t, d;
};
// Per-thread scratch buffers of the hot functions.  Reached through a constant-initialised
// thread_local pointer, so an access is one TLS load (a thread_local std::vector would go
// through the TLS init wrapper on every call); created on a thread's first use, freed at its exit.
struct Scratch {
  std::vector<Ev> ev;
  Profile tmp;
  std::vector<TSeg> segs_apply, segs_send;
  std::vector<i64> comp, take;
  Transfer tr_send;
};
static thread_local Scratch *t_scratch = nullptr;
static Scratch *make_scratch() {
  static thread_local std::unique_ptr<Scratch> owner;
  owner.reset(new Scratch());
  return t_scratch = owner.get();
}
static inline Scratch &scratch() {
  Scratch *s = t_scratch;
  return __builtin_expect(s != nullptr, 1) ? *s : *make_scratch();
}

static void combine(Profile &p, const TSeg *s, int m, int sign) {
  Scratch &S = scratch();
  std::vector<Ev> &ev = S.ev;
  Profile &tmp = S.tmp;
  ev.clear();
  for (int i = 0; i < m; ++i)
    if (s[i].r != 0 && s[i].a < s[i].b) {
      ev.push_back({s[i].a, sign * s[i].r});
      ev.push_back({s[i].b, -sign * s[i].r});
    }
  if (ev.empty()) return;
  // one transfer's segments, or a reserved-rate profile, arrive in time order already
  if (!std::is_sorted(ev.begin(), ev.end(), [](const Ev &x, const Ev &y) { return x.t < y.t; }))
    std::sort(ev.begin(), ev.end(), [](const Ev &x, const Ev &y) { return x.t < y.t; });
  const i64 A = ev.front().t, B = ev.back().t;
  // ia = last segment starting at or before A (p[0].t == 0 <= A)
  size_t ia = (size_t)(std::upper_bound(p.begin(), p.end(), A, [](i64 v, const Seg &x) { return v < x.t; }) -
                       p.begin()) - 1;
  const size_t keep = p[ia].t < A ? ia + 1 : ia;       // p[0, keep) stays as it is
  i64 base = p[ia].r, delta = 0;
  size_t pi = ia + 1, ei = 0;
  tmp.clear();
  for (i64 t = A;;) {
    while (pi < p.size() && p[pi].t <= t) base = p[pi++].r;
    while (ei < ev.size() && ev[ei].t <= t) delta += ev[ei++].d;
    const i64 r = base + delta;
    if (r < 0) throw PlanFail{MLF_E_INVALID, "internal: residual went negative"};
    const i64 prev = tmp.empty() ? (keep > 0 ? p[keep - 1].r : -1) : tmp.back().r;
    if (r != prev) tmp.push_back({t, r});
    if (t >= B) break;
    i64 nt = ev[ei].t;                                 // ei < ev.size() while t < B
    if (pi < p.size()) nt = std::min(nt, p[pi].t);
    t = nt;
  }
  // p[keep, pi) is replaced by tmp (pi = first segment starting after B)
  const size_t old_n = pi - keep, new_n = tmp.size();
  if (new_n > old_n)
    p.insert(p.begin() + (std::ptrdiff_t)pi, new_n - old_n, Seg{0, 0});
  else if (new_n < old_n)
    p.erase(p.begin() + (std::ptrdiff_t)(keep + new_n), p.begin() + (std::ptrdiff_t)pi);
  std::copy(tmp.begin(), tmp.end(), p.begin() + (std::ptrdiff_t)keep);
}

// Reservations evaluated but not applied to a Net: per link, the reserved rate as a step
// profile (0 outside the reservations), so a transfer walks it with a cursor like the
// link's own residual profile.  clear() keeps every buffer's capacity.
struct Pending {
  int nkeys = 0;
  std::vector<i64> keys;
  std::vector<Profile> used;
  void clear() { nkeys = 0; }
  const Profile *find(i64 key) const {
    for (int i = 0; i < nkeys; ++i)
      if (keys[i] == key) return &used[i];
    return nullptr;
  }
  Profile &slot(i64 key, bool *fresh = nullptr) {
    for (int i = 0; i < nkeys; ++i)
      if (keys[i] == key) {
        if (fresh) *fresh = false;
        return used[i];
      }
    if (nkeys == (int)keys.size()) {
      keys.push_back(key);
      used.emplace_back();
    }
    keys[nkeys] = key;
    used[nkeys].assign(1, Seg{0, 0});
    if (fresh) *fresh = true;
    return used[nkeys++];
  }
  // add segments s[0, m) — in time order, disjoint — to the link's reserved rate: into a fresh
  // slot (the zero profile) they are written out directly as the canonical profile combine()
  // would build; otherwise merged by combine()
  void add(i64 key, const TSeg *s, int m) {
    bool fresh;
    Profile &p = slot(key, &fresh);
    if (!fresh) {
      combine(p, s, m, +1);
      return;
    }
    for (int i = 0; i < m; ++i) {
      if (s[i].r == 0 || s[i].a >= s[i].b) continue;
      if (p.back().t == s[i].a) {                 // a breakpoint (value 0) where this segment starts
        if (p.size() > 1 && p[p.size() - 2].r == s[i].r) p.pop_back();
        else p.back().r = s[i].r;
      } else {                                    // p.back().t < s[i].a, value 0 up to s[i].a
        p.push_back({s[i].a, s[i].r});
      }
      p.push_back({s[i].b, 0});
    }
  }
};

// cursor over a step profile: i = the segment holding the current time
struct Cur {
  const Seg *p = nullptr;
  int n = 0, i = 0;
  void seek(const Profile *pr, i64 t) {
    if (!pr) {
      n = 0;
      return;
    }
    p = pr->data();
    n = (int)pr->size();
    const Seg *it = std::upper_bound(p, p + n, t, [](i64 v, const Seg &s) { return v < s.t; });
    i = it == p ? 0 : (int)(it - p) - 1;
  }
  i64 at(i64 t) {                                  // value at t (t never decreases)
    if (!n) return 0;
    while (i + 1 < n && p[i + 1].t <= t) ++i;
    return p[i].r;
  }
  i64 next() const { return (n && i + 1 < n) ? p[i + 1].t : T_INF; }
};

// O1: water-fill `size` bytes from t_avail along the path residual (Fig. 5(b)),
// on `net` minus the pending reservations of L0 and L1.  Returns false if the
// path residual is zero forever after t_avail.
// A walk step of a transfer: on [t0, t1) every path link k had `slack[k]` more residual than
// the path minimum the transfer used.  Reserving at most slack[k] more on link k inside the
// window leaves the path minimum, hence the whole transfer, unchanged (used by the
// ordering's per-class cache, order_final).
struct WalkRec {
  i64 t0, t1, r, slack[3];   // r: the rate the transfer used on [t0, t1)
};

static bool transfer(const Net &net, const Pending *L0, const Pending *L1, i64 size, int src, int dst, i64 t_avail,
                     Transfer &out, std::vector<WalkRec> *rec = nullptr) {
  const NetDef &d = *net.def;
  out.segs.clear();
  out.path = path_of(d, src, dst);
  if (size == 0 || out.path.nk == 0) {
    out.path.nk = 0;
    out.t_st = out.t_en = t_avail;
    return true;
  }
  // one cursor per (link, profile): the link's residual, then the reserved rates of L0 and L1
  // on it (only those that exist); sign = +1 for a residual, -1 for a reservation.  The walk
  // keeps each link's residual rks[k] at `cur` and each cursor's next breakpoint nt, and only
  // advances the cursors whose breakpoint is reached.
  struct C {
    const Seg *p;
    int n, i, link;
    i64 sign, nt;
  };
  C cs[9];
  Seg own[3];                 // pair links not reserved yet: their capacity
  int nc = 0;
  const int nk = out.path.nk;
  i64 rks[3] = {0, 0, 0};
  auto add = [&](const Seg *p, int n, int k, i64 sign) {
    C &c = cs[nc++];
    c.p = p;
    c.n = n;
    const Seg *it = std::upper_bound(p, p + n, t_avail, [](i64 v, const Seg &x) { return v < x.t; });
    c.i = it == p ? 0 : (int)(it - p) - 1;
    c.link = k;
    c.sign = sign;
    c.nt = c.i + 1 < n ? p[c.i + 1].t : T_INF;
    rks[k] += sign * p[c.i].r;
  };
  for (int k = 0; k < nk; ++k) {
    const i64 key = out.path.key[k];
    if (const Profile *pr = net.get(key)) {
      add(pr->data(), (int)pr->size(), k, +1);
    } else {
      own[k] = Seg{0, std::max<i64>(net.capacity(key), 0)};
      add(&own[k], 1, k, +1);
    }
    if (L0)
      if (const Profile *u = L0->find(key)) add(u->data(), (int)u->size(), k, -1);
    if (L1)
      if (const Profile *u = L1->find(key)) add(u->data(), (int)u->size(), k, -1);
  }
  // move every cursor to time t (t never decreases; cursors already there stay)
  auto reach = [&](i64 t) {
    for (int q = 0; q < nc; ++q) {
      C &c = cs[q];
      if (c.nt > t) continue;
      rks[c.link] -= c.sign * c.p[c.i].r;
      do ++c.i;
      while (c.i + 1 < c.n && c.p[c.i + 1].t <= t);
      rks[c.link] += c.sign * c.p[c.i].r;
      c.nt = c.i + 1 < c.n ? c.p[c.i + 1].t : T_INF;
    }
  };
  i128 need = (i128)size * NS_PER_S;
  i64 cur = t_avail;
  bool started = false;
  for (;;) {
    // r = the path minimum at cur, nb = its next possible change; while some link is saturated
    // the path stays at 0 at least until every saturated link's own next change (zjump), so
    // the walk jumps there instead of stepping through the other links' breakpoints
    i64 nbk[3] = {T_INF, T_INF, T_INF};
    for (int q = 0; q < nc; ++q) nbk[cs[q].link] = std::min(nbk[cs[q].link], cs[q].nt);
    i64 r = T_INF, nb = T_INF, zjump = t_avail;
    for (int k = 0; k < nk; ++k) {
      if (rks[k] == 0) zjump = std::max(zjump, nbk[k]);
      r = std::min(r, rks[k]);
      nb = std::min(nb, nbk[k]);
    }
    if (r < 0) throw PlanFail{MLF_E_INVALID, "internal: negative residual"};
    if (r == 0) {
      if (zjump == T_INF) return false;          // a link on the path is saturated forever
      cur = zjump;
      reach(cur);
      continue;
    }
    if (!started) {
      out.t_st = cur;
      started = true;
    }
    if (nb == T_INF || (i128)r * (nb - cur) >= need) {
      i128 dt = (need + r - 1) / r;
      if ((i128)cur + dt > (i128)T_LIMIT) throw PlanFail{MLF_E_INVALID, "model time overflow"};
      out.t_en = cur + (i64)dt;
      out.segs.push_back({cur, out.t_en, r});
      if (rec) rec->push_back({cur, out.t_en, r, {rks[0] - r, nk > 1 ? rks[1] - r : 0, nk > 2 ? rks[2] - r : 0}});
      return true;
    }
    need -= (i128)r * (nb - cur);
    out.segs.push_back({cur, nb, r});
    if (rec) rec->push_back({cur, nb, r, {rks[0] - r, nk > 1 ? rks[1] - r : 0, nk > 2 ? rks[2] - r : 0}});
    cur = nb;
    reach(cur);
  }
}

// O2: NetUp — subtract reservations from the residual profiles.
static void apply_pending(Net &net, const Pending &P, int sign = -1) {
  std::vector<TSeg> &segs = scratch().segs_apply;
  for (int i = 0; i < P.nkeys; ++i) {
    const Profile &u = P.used[i];
    segs.clear();
    for (size_t q = 0; q + 1 < u.size(); ++q)
      if (u[q].r) segs.push_back({u[q].t, u[q + 1].t, u[q].r});
    combine(net.mut(P.keys[i]), segs.data(), (int)segs.size(), sign);
  }
}
static void copy_pending(Pending &dst, const Pending &src) {
  dst.nkeys = src.nkeys;
  dst.keys.assign(src.keys.begin(), src.keys.begin() + src.nkeys);
  dst.used.assign(src.used.begin(), src.used.begin() + src.nkeys);
}
static void apply_transfer(Net &net, const Transfer &tr) {
  for (int k = 0; k < tr.path.nk; ++k) combine(net.mut(tr.path.key[k]), tr.segs.data(), (int)tr.segs.size(), -1);
}

// App. B.2: component sizes proportional to the shard weights.
static void component_bytes(i64 size, const std::vector<i64> &w, i64 wsum, std::vector<i64> &out) {
  out.resize(w.size());
  i64 cum = 0;
  for (size_t j = 0; j < w.size(); ++j) {
    i64 lo = (i64)((i128)size * cum / wsum);
    cum += w[j];
    out[j] = (i64)((i128)size * cum / wsum) - lo;
  }
}

struct Send {
  i64 t_st = 0, t_en = 0;
};

struct Ctx {
  NetDef d;
  std::vector<int> servers, aggs, replicas, raggs;
  std::vector<i64> weights;
  i64 wsum = 0;
  bool dup_dsts = false;     // a destination list (servers / replicas) repeats a node
};

// Multi-component transfer: components reserved sequentially in destination
// order (R11) into `local` (pending on top of net - L0); t_en = max, t_st = min.
// record_all = false (a pure evaluation, nothing is applied afterwards): `local` keeps only the
// links a LATER component can share — up(src), and a later destination's own links when the
// destination list repeats a node — which is all the later transfers read.
// The walk of one send, component by component (CompRec: path, its WalkRec range, times).
struct CompRec {
  Path path;
  int w0, w1;
  i64 t_st, t_en;
};
struct SendRec {
  std::vector<CompRec> comps;
  std::vector<WalkRec> walk;
};

// the reserved segments of a recorded component (identical to its Transfer::segs)
static void rec_segs(const SendRec &rec, const CompRec &cr, std::vector<TSeg> &segs) {
  segs.clear();
  for (int w = cr.w0; w < cr.w1; ++w) segs.push_back({rec.walk[w].t0, rec.walk[w].t1, rec.walk[w].r});
}

// Multi-component transfer: components reserved sequentially in destination
// order (R11) into `local` (pending on top of net - L0); t_en = max, t_st = min.
// record_all = false (a pure evaluation, nothing is applied afterwards): `local` keeps only the
// links a LATER component can share — up(src), and a later destination's own links when the
// destination list repeats a node — which is all the later transfers read.
// rec: the walk is recorded; from > 0 resumes a recorded send whose components 0..from-1 are
// still valid on this network (their recorded reservations are replayed into `local`).
static bool send(const Net &net, const Pending *L0, const Ctx &c, const std::vector<int> &dsts, int src, i64 size,
                 i64 t_avail, Send &out, Pending &local, bool record_all = true, SendRec *rec = nullptr,
                 int from = 0) {
  Scratch &S = scratch();
  Transfer &tr = S.tr_send;
  std::vector<i64> &comp = S.comp;
  std::vector<TSeg> &segs = S.segs_send;
  component_bytes(size, c.weights, c.wsum, comp);
  local.clear();
  out.t_st = T_INF;
  out.t_en = 0;
  const i64 n = c.d.n;
  const bool all = record_all || c.dup_dsts;
  auto reserve = [&](size_t j, const Path &path, const std::vector<TSeg> &sg) {
    if (j + 1 < dsts.size() ? all : record_all) {
      for (int k = 0; k < path.nk; ++k) local.add(path.key[k], sg.data(), (int)sg.size());
    } else if (j + 1 < dsts.size() && path.nk && path.key[0] < n) {   // up(src) is always the first path link
      local.add(path.key[0], sg.data(), (int)sg.size());
    }
  };
  if (rec) {
    for (int j = 0; j < from; ++j) {
      const CompRec &cr = rec->comps[j];
      rec_segs(*rec, cr, segs);
      reserve((size_t)j, cr.path, segs);
      out.t_st = std::min(out.t_st, cr.t_st);
      out.t_en = std::max(out.t_en, cr.t_en);
    }
    rec->walk.resize(from > 0 ? rec->comps[from].w0 : 0);
    rec->comps.resize(from);
  }
  for (size_t j = from; j < dsts.size(); ++j) {
    const int w0 = rec ? (int)rec->walk.size() : 0;
    if (!transfer(net, L0, &local, comp[j], src, dsts[j], t_avail, tr, rec ? &rec->walk : nullptr)) return false;
    if (rec) rec->comps.push_back({tr.path, w0, (int)rec->walk.size(), tr.t_st, tr.t_en});
    reserve(j, tr.path, tr.segs);
    out.t_st = std::min(out.t_st, tr.t_st);
    out.t_en = std::max(out.t_en, tr.t_en);
  }
  return true;
}

// send + NetUp on `net`
static bool send_apply(Net &net, const Ctx &c, const std::vector<int> &dsts, int src, i64 size, i64 t_avail,
                       Send &out) {
  thread_local Pending P;
  if (!send(net, nullptr, c, dsts, src, size, t_avail, out, P)) return false;
  apply_pending(net, P);
  return true;
}

struct Item {
  int node;
  i64 size, version, t_avail;
  double norm;
};

// ---------------------------------------------------------------- O3 ordering
// What Alg. 3 needs from the networks Alg. 2 passes through (R10: case n starts from the
// batch-start network with the first n kept updates sent direct, which is exactly Alg. 2's NW
// after its n-th kept update).  Filled by order_final when given:
//  * snaps[j]: NW after j*kEvery kept updates (a case replays at most kEvery-1 reservations);
//  * tmax[n]: the direct prefix's t_max (the largest t_en of kept updates 0..n-1);
//  * dead[n]: case n ends at its first tail item — that item cannot reach aggs[0] by tmax[n]
//    and group 1 would be empty (R12, det_agg_tail's first step on the same network);
//  * last: NW after every kept update (the all-direct case's network).
struct AggProbe {
  static constexpr int kEvery = 8;
  const std::vector<int> *aggs = nullptr;
  std::vector<Net> snaps;
  std::vector<i64> tmax;
  std::vector<uint8_t> dead;
  std::unique_ptr<Net> last;
};

struct OrderRes {
  std::vector<int> order;
  std::vector<uint8_t> reason;
  // the reservation of every kept update, in O(U) order, on the batch-start network with the
  // earlier kept ones applied: exactly Alg. 3's direct prefix (R10), reused by plan_aggregation
  std::vector<Pending> res;
  std::vector<Send> sends;
};

// Classes an Alg. 2 scan must validate or re-evaluate before its tasks go to the pool
// (MLF_PLAN_MIN_EVALS overrides).  Measured on a B200 box's host (profiles/r02/planner_late):
// a scan has ~7 such classes, ~4 of them re-evaluated (~2.5 us each); with the claim-word pool
// a hand-off costs ~0.2 us, and config 4 / G = 8 plans fastest at a threshold of 4 (1.87 ms on
// 8 threads vs 1.97 at 8 and 2.2 at 32).
// Servers from which a look-ahead scan takes the side items (MLF_PLAN_SIDE_MIN_SERVERS overrides):
// they pay where a class's send and g*'s NetUp are long (G = 8: 1.88 -> 1.63 ms at config 4 on the
// box host) but cost hand-offs where both are short (G = 4: 0.78 vs 0.73 ms; G = 2, rank 0 in the
// 2-GPU bench: 0.87 vs 0.37 ms), since they also send scans with a single changed class to the pool
static int side_min_servers() {
  static const int v = [] {
    const char *e = getenv("MLF_PLAN_SIDE_MIN_SERVERS");
    return e && atoi(e) > 0 ? atoi(e) : 8;
  }();
  return v;
}

static int min_parallel_evals() {
  static const int v = [] {
    const char *e = getenv("MLF_PLAN_MIN_EVALS");
    return e && atoi(e) > 0 ? atoi(e) : 4;
  }();
  return v;
}

// The first component of a recorded send whose result changes when `M` is reserved on top of
// the network it was recorded on (comps.size(): none).  A component is unchanged if on every
// walk step no path link loses more than its slack; components are reserved one after another,
// so an unchanged prefix also leaves the next component's inputs unchanged.  Saturated
// stretches were skipped by the walk and stay saturated.  The unchanged components' slacks are
// reduced by what M takes, so the record describes the send on the new network; each reduction
// is appended to `log` (if given) so that it can be undone.
struct TakeLog {
  int w, k;
  i64 amount;
};
static int first_changed(SendRec &rec, const Pending &M, std::vector<TakeLog> *log = nullptr) {
  std::vector<i64> &take = scratch().take;
  for (size_t j = 0; j < rec.comps.size(); ++j) {
    const CompRec &cr = rec.comps[j];
    take.assign((size_t)(cr.w1 - cr.w0) * 3, 0);
    for (int k = 0; k < cr.path.nk; ++k) {
      const Profile *u = M.find(cr.path.key[k]);
      if (!u) continue;
      Cur cu;
      for (int w = cr.w0; w < cr.w1; ++w) {
        const WalkRec &wr = rec.walk[w];
        if (w == cr.w0) cu.seek(u, wr.t0);
        // the largest reserved rate of M on [t0, t1)
        i64 mx = cu.at(wr.t0);
        for (int q = cu.i + 1; q < cu.n && cu.p[q].t < wr.t1; ++q) mx = std::max(mx, cu.p[q].r);
        if (mx > wr.slack[k]) return (int)j;
        take[(size_t)(w - cr.w0) * 3 + k] = mx;
      }
    }
    for (int w = cr.w0; w < cr.w1; ++w)
      for (int k = 0; k < cr.path.nk; ++k) {
        const i64 t = take[(size_t)(w - cr.w0) * 3 + k];
        if (!t) continue;
        rec.walk[w].slack[k] -= t;
        if (log) log->push_back({w, k, t});
      }
  }
  return (int)rec.comps.size();
}

static OrderRes order_final(const Ctx &c, const std::vector<Item> &batch, i64 tau, i64 v_init,
                            AggProbe *probe = nullptr) {
  const int n = (int)batch.size();
  std::vector<i64> dl(n);
  for (int g = 0; g < n; ++g) dl[g] = batch[g].version + tau - v_init;
  std::vector<int> unproc(n);
  for (int g = 0; g < n; ++g) unproc[g] = g;
  OrderRes res;
  res.reason.assign(n, 0);
  Net nw(&c.d);
  i64 p = 1;
  std::vector<i64> ten(n);
  std::vector<uint8_t> ok(n);
  std::vector<int> pool, uniq, miss, rep(n, -1);
  // with one server a class's send is one transfer (~0.3 us): too little to hand to the pool
  // (config 2, tau 32: 0.13 ms serial vs 0.22 ms on 8 threads)
  const bool multi_server = c.servers.size() > 1;
  const bool use_side = multi_server && (int)c.servers.size() >= side_min_servers();
  // t_en is a pure function of (network, node, size, t_avail): updates sharing the triple
  // (virtual workers on one GPU usually share all three) form one class, evaluated once per scan
  std::vector<int> cls(n), cls_rep, cls_stamp;
  {
    std::vector<int> byk(n);
    for (int g = 0; g < n; ++g) byk[g] = g;
    std::sort(byk.begin(), byk.end(), [&](int a, int b) {
      const Item &x = batch[a], &y = batch[b];
      if (x.node != y.node) return x.node < y.node;
      if (x.size != y.size) return x.size < y.size;
      if (x.t_avail != y.t_avail) return x.t_avail < y.t_avail;
      return a < b;
    });
    int k = -1;
    for (int i = 0; i < n; ++i) {
      const Item &x = batch[byk[i]];
      if (i == 0 || x.node != batch[byk[i - 1]].node || x.size != batch[byk[i - 1]].size ||
          x.t_avail != batch[byk[i - 1]].t_avail)
        ++k;
      cls[byk[i]] = k;
    }
    cls_rep.assign(k + 1, -1);
    cls_stamp.assign(k + 1, -1);
  }
  int scan = 0;
  // Per-class result cache.  Network states get ids: nw_id = NW, la_id = NW + the look-ahead's
  // reservation of g*; NW takes la_id when g* is kept and keeps nw_id when it is dropped.
  // A look-ahead scan moves classes from NW to NW + g*; when g* is then dropped the network is
  // NW again, so the scan keeps what it overwrote: the NW record of every class it re-evaluated
  // (bk) and every slack reduction it made (takes), and a drop puts both back.
  struct ClassCache {
    int tag = -1;
    i64 t_st = 0, t_en = 0;
    SendRec rec;
    bool moved = false, backed = false;      // this look-ahead moved it to la_id / saved its record
    i64 bk_t_st = 0, bk_t_en = 0;
    SendRec bk;
    std::vector<TakeLog> takes;
  };
  std::vector<ClassCache> cache(cls_rep.size());
  PlanFail task_err{MLF_OK, ""};
  std::atomic<bool> task_failed{false};
  int nw_id = 0, la_id = 0, next_id = 1;
  std::vector<int> la_moved;                 // classes the current look-ahead moved to la_id

  // ShrtDline(pos, cands, NW + L0): the due set's argmin if any, else ShrtUp (R4, R6).
  // side(0), side(1): work that must not wait for the scan but only reads NW and L0 (see the
  // look-ahead below); when the scan's classes go to the pool it runs there as two more items,
  // else it is not run and *side_ran stays false.
  auto pick = [&](i64 pos, const std::vector<int> &cands, const Pending *L0,
                  const std::function<void(int)> *side = nullptr, bool *side_ran = nullptr) -> int {
    bool any_due = false;
    for (int g : cands)
      if (dl[g] == pos) {
        any_due = true;
        break;
      }
    pool.clear();
    for (int g : cands)
      if (!any_due || dl[g] == pos) pool.push_back(g);
    // one evaluation per class; its representative is the class's first member in the pool
    ++scan;
    uniq.clear();
    for (int g : pool) {
      const int k = cls[g];
      if (cls_stamp[k] != scan) {
        cls_stamp[k] = scan;
        cls_rep[k] = g;
        uniq.push_back(g);
      }
      rep[g] = cls_rep[k];
    }
    // a class evaluated on NW (tag nw_id) keeps its result on NW + L0 when L0 = the look-ahead's
    // reservation costs none of its walk steps more than their slack (first_changed); the others
    // are evaluated again from their first changed component.  Validation and re-evaluation of a
    // class are one task; the scan's tasks run on the pool when there are enough of them.
    const int tag = L0 ? la_id : nw_id;
    miss.clear();
    for (int g : uniq) {
      ClassCache &cc = cache[cls[g]];
      if (cc.tag == tag) {
        ok[g] = 1;
        ten[g] = cc.t_en;
      } else {
        miss.push_back(g);
      }
    }
    const int ms = (int)miss.size();
    const bool par = multi_server && (ms >= min_parallel_evals() || (side && ms >= 1));
    const int off = par && side ? 2 : 0;
    if (side_ran) *side_ran = off > 0;
    Pool::get().run(
        ms + off,
        [&](int i) {
          if (i < off) {
            try {
              (*side)(i);
            } catch (const PlanFail &e) {
              if (!task_failed.exchange(true)) task_err = e;
            }
            return;
          }
          thread_local Pending local;
          const int g = miss[i - off];
          ClassCache &cc = cache[cls[g]];
          int from = 0;
          const bool on_nw = L0 && cc.tag == nw_id;
          cc.moved = on_nw;
          cc.backed = false;
          if (on_nw) {
            cc.takes.clear();
            from = first_changed(cc.rec, *L0, &cc.takes);
            if (from == (int)cc.rec.comps.size()) {
              cc.tag = tag;
              ok[g] = 1;
              ten[g] = cc.t_en;
              return;
            }
            cc.backed = true;
            cc.bk = cc.rec;
            cc.bk_t_st = cc.t_st;
            cc.bk_t_en = cc.t_en;
          }
          Send s;                                  // the components before `from` keep their results
          try {
            ok[g] = send(nw, L0, c, c.servers, batch[g].node, batch[g].size, batch[g].t_avail, s, local, false,
                         &cc.rec, from);
          } catch (const PlanFail &e) {
            if (!task_failed.exchange(true)) task_err = e;
            ok[g] = 1;
            s.t_en = 0;
          }
          ten[g] = s.t_en;
          cc.tag = ok[g] ? tag : -1;
          cc.t_st = s.t_st;
          cc.t_en = s.t_en;
        },
        par ? 2 : std::numeric_limits<int>::max());
    if (task_failed.load()) throw task_err;
    if (L0)
      for (int g : miss)
        if (cache[cls[g]].moved) la_moved.push_back(cls[g]);
    int best = -1;
    for (int g : pool) {
      ok[g] = ok[rep[g]];
      ten[g] = ten[rep[g]];
      if (!ok[g]) throw PlanFail{MLF_E_UNSCHEDULABLE, "update path to a server is down"};
      if (best < 0 || ten[g] < ten[best]) best = g;
    }
    return best;
  };

  Pending star;
  // When g* is kept, the next step's pick at p+1 runs over exactly the look-ahead's
  // candidates (the unprocessed updates with dl >= p+1) on exactly the look-ahead's
  // network (NW with g* reserved), so its result is the look-ahead's g° (and t_en):
  // reusing it halves the scans without changing any decision.
  int cached = -1;
  std::vector<int> keep, cands;
  // What a kept g* costs after its decision (Alg. 3's probe of NW, NetUp, the copy of its
  // reservation) only reads NW and g*'s reservation, which the look-ahead scan also only reads,
  // so it runs as a side job of that scan, speculatively (a dropped g* discards it):
  //  * nw2 is a second copy of NW, brought up to date and given g*'s reservation in the side
  //    job, so a kept g* swaps the two (NetUp off the critical path); `lag` lists the
  //    reservations nw2 still has to apply (sign -1) or take back (sign +1) to equal NW —
  //    canonical profiles make the result independent of that order;
  //  * spec_res / spec_snap / spec_tm / spec_dead: the reservation's copy and the probe of NW.
  res.res.reserve(n);                       // lag keeps pointers into res.res
  std::unique_ptr<Net> nw2;
  std::vector<std::pair<const Pending *, int>> lag;
  Pending spec_res, undo_res;
  std::unique_ptr<Net> spec_snap;
  i64 spec_tm = 0;
  bool spec_dead = false, spec_has_snap = false;
  auto probe_now = [&](const Net &net, int g, i64 &tm, bool &dead, bool &has_snap, std::unique_ptr<Net> &snap) {
    const int k = (int)res.order.size();               // g*'s position in O(U)
    has_snap = k % AggProbe::kEvery == 0;
    if (has_snap) {
      if (snap) *snap = net;
      else snap = std::make_unique<Net>(net);
    }
    tm = k == 0 ? 0 : std::max(probe->tmax[k - 1], res.sends[k - 1].t_en);
    dead = false;
    if (k > 0) {
      thread_local Transfer tr;
      const Item &it = batch[g];
      try {
        dead = !transfer(net, nullptr, nullptr, it.size, it.node, (*probe->aggs)[0], it.t_avail, tr) || tr.t_en > tm;
      } catch (const PlanFail &) {
        dead = false;                                    // the case itself reports it, if it runs
      }
    }
  };
  int side_g = -1;
  // two independent side items: nw2's NetUps; the reservation's copy and the probe of NW
  const std::function<void(int)> side = [&](int j) {
    if (j == 0) {
      for (const auto &op : lag) apply_pending(*nw2, *op.first, op.second);
      apply_pending(*nw2, star);
      return;
    }
    copy_pending(spec_res, star);
    if (probe) probe_now(nw, side_g, spec_tm, spec_dead, spec_has_snap, spec_snap);
  };
  for (;;) {
    keep.clear();
    for (int g : unproc) {
      if (dl[g] < p)
        res.reason[g] = 1;                          // expired (R4)
      else
        keep.push_back(g);
    }
    unproc.swap(keep);
    if (unproc.empty()) break;
    const int g_star = cached >= 0 ? cached : pick(p, unproc, nullptr);
    const i64 t_star = ten[g_star];
    cached = -1;
    Send s_star;
    const ClassCache &cg = cache[cls[g_star]];
    if (cg.tag == nw_id) {
      // g*'s class was evaluated on exactly this network: its recorded walk is the reservation
      thread_local std::vector<TSeg> segs;
      star.clear();
      for (const CompRec &cr : cg.rec.comps) {
        rec_segs(cg.rec, cr, segs);
        for (int k = 0; k < cr.path.nk; ++k) star.add(cr.path.key[k], segs.data(), (int)segs.size());
      }
      s_star.t_st = cg.t_st;
      s_star.t_en = cg.t_en;
    } else {
      send(nw, nullptr, c, c.servers, batch[g_star].node, batch[g_star].size, batch[g_star].t_avail, s_star, star);
    }
    cands.clear();
    for (int g : unproc)
      if (g != g_star && dl[g] >= p + 1) cands.push_back(g);
    bool drop = false, side_ran = false;
    int g_next = -1;
    la_id = next_id++;
    la_moved.clear();
    if (!cands.empty()) {
      if (use_side && !nw2) nw2 = std::make_unique<Net>(nw);
      side_g = g_star;
      g_next = pick(p + 1, cands, &star, use_side ? &side : nullptr, &side_ran);   // on NetUp(NW, g*)
      if (t_star > ten[g_next]) drop = true;           // Alg. 2 line 10
    }
    unproc.erase(std::find(unproc.begin(), unproc.end(), g_star));
    if (drop) {
      res.reason[g_star] = 2;
      // back to NW: restore what the look-ahead scan overwrote
      for (int k : la_moved) {
        ClassCache &cc = cache[k];
        if (cc.backed) {
          std::swap(cc.rec, cc.bk);
          cc.t_st = cc.bk_t_st;
          cc.t_en = cc.bk_t_en;
        }
        for (const TakeLog &t : cc.takes) cc.rec.walk[t.w].slack[t.k] += t.amount;
        cc.tag = nw_id;
      }
      if (side_ran) {                                   // nw2 took g*'s reservation: take it back
        std::swap(spec_res, undo_res);                  // (the next side items rewrite spec_res)
        lag.clear();
        lag.push_back({&undo_res, +1});
      }
      continue;
    }
    if (side_ran) {
      if (probe) {
        if (spec_has_snap) probe->snaps.push_back(std::move(*spec_snap));
        probe->tmax.push_back(spec_tm);
        probe->dead.push_back(spec_dead);
      }
      std::swap(nw, *nw2);                              // NW := NW + g*; nw2 lags by g*
      res.res.emplace_back();
      std::swap(res.res.back(), spec_res);
      lag.clear();
      lag.push_back({&res.res.back(), -1});
    } else {
      if (probe) {
        i64 tm;
        bool dead, has_snap;
        std::unique_ptr<Net> snap;
        probe_now(nw, g_star, tm, dead, has_snap, snap);
        if (has_snap) probe->snaps.push_back(std::move(*snap));
        probe->tmax.push_back(tm);
        probe->dead.push_back(dead);
      }
      apply_pending(nw, star);
      res.res.emplace_back();
      copy_pending(res.res.back(), star);
      if (nw2) lag.push_back({&res.res.back(), -1});
    }
    res.order.push_back(g_star);
    nw_id = la_id;
    res.sends.push_back(s_star);
    ++p;
    cached = g_next;
  }
  if (probe) {
    const int N = (int)res.order.size();
    if (N % AggProbe::kEvery == 0) probe->snaps.push_back(nw);
    probe->tmax.push_back(N == 0 ? 0 : std::max(probe->tmax[N - 1], res.sends[N - 1].t_en));
    probe->dead.push_back(0);
    probe->last = std::make_unique<Net>(std::move(nw));
  }
  return res;
}

// ---------------------------------------------------------------- O4 aggregation
struct CommitRec {
  int first, count, group;
  Send send;
};
struct AggCase {
  int n = 0;
  bool feasible = false;
  bool record = false;              // keep the member transfers' times (distribution plans)
  i64 total = 0;
  std::vector<CommitRec> commits;
  std::vector<i64> m_st, m_en;      // [position - n]: member -> aggregator transfer times
};

// Alg. 3 DetAgg(n), continued from the state after its n direct sends (R10-R12):
// `nw` holds that network, t_max/commits the direct part.
// `cutoff`: the case only matters if its total can still be < cutoff (the argmin's best so
// far); t_max never decreases, so the walk stops as soon as t_max > cutoff (result: not feasible
// for the argmin).  T_INF = no cutoff.
static void det_agg_tail(AggCase &cs, Net &nw, i64 t_max, const std::vector<Item> &items, const Ctx &c,
                         const std::vector<int> &dsts, const std::vector<int> &aggs, i64 cutoff = T_INF) {
  const int n = cs.n;
  bool have = n > 0;
  const int k = (int)aggs.size();
  int aid = 1, i = n, gfirst = n, gcount = 0;
  i64 gsize = 0, garr = 0;
  auto flush = [&]() -> bool {                                // lines 11-12
    Send s;
    if (!send_apply(nw, c, dsts, aggs[aid - 1], gsize, garr, s)) return false;
    t_max = std::max(t_max, s.t_en);
    have = true;
    cs.commits.push_back({gfirst, gcount, aid, s});
    ++aid;
    gfirst += gcount;
    gcount = 0;
    gsize = 0;
    garr = 0;
    return true;
  };
  thread_local Transfer tr;
  while (i < (int)items.size()) {
    if (aid > k || t_max > cutoff) return;
    if (!transfer(nw, nullptr, nullptr, items[i].size, items[i].node, aggs[aid - 1], items[i].t_avail, tr)) return;
    if (have && tr.t_en > t_max) {                            // line 10
      if (gcount == 0) return;
      if (!flush()) return;
      continue;
    }
    apply_transfer(nw, tr);                                   // lines 16-18
    if (cs.record) {
      cs.m_st.push_back(tr.t_st);
      cs.m_en.push_back(tr.t_en);
    }
    if (gcount == 0) gfirst = i;
    ++gcount;
    gsize = std::max(gsize, items[i].size);
    garr = std::max(garr, tr.t_en);
    ++i;
  }
  if (gcount > 0 && !flush()) return;
  if (t_max > cutoff) return;
  cs.feasible = true;
  cs.total = t_max;
}

// The n-update direct prefix (Alg. 3 lines 3-7) applied to `nw`.
// Reservations of the direct prefix already computed by Alg. 2 (OrderRes::res / sends): item i
// of O(U) sent to the servers on the batch-start network with items 0..i-1 applied.
struct PrefixHint {
  const std::vector<Pending> *res = nullptr;
  const std::vector<Send> *sends = nullptr;
};

struct Prefix {
  Net nw;
  i64 t_max = 0;
  std::vector<CommitRec> commits;
  bool ok = true;
  const PrefixHint *hint = nullptr;
  explicit Prefix(const Net &n0, const PrefixHint *h = nullptr) : nw(n0), hint(h) {}
  void extend(const std::vector<Item> &items, int i, const Ctx &c, const std::vector<int> &dsts) {
    if (!ok) return;
    Send s;
    if (hint) {                                  // the same send_apply, replayed from Alg. 2
      apply_pending(nw, (*hint->res)[i]);
      s = (*hint->sends)[i];
    } else if (!send_apply(nw, c, dsts, items[i].node, items[i].size, items[i].t_avail, s)) {
      ok = false;
      return;
    }
    t_max = std::max(t_max, s.t_en);
    commits.push_back({i, 1, 0, s});
  }
};

static AggCase det_agg(int n, const std::vector<Item> &items, const Net &net0, const Ctx &c,
                       const std::vector<int> &dsts, const std::vector<int> &aggs, Net *net_out,
                       bool record = false) {
  Prefix pre(net0);
  for (int i = 0; i < n; ++i) pre.extend(items, i, c, dsts);
  AggCase cs;
  cs.n = n;
  cs.record = record;
  if (!pre.ok) return cs;
  cs.commits = pre.commits;
  det_agg_tail(cs, pre.nw, pre.t_max, items, c, dsts, aggs);
  if (cs.feasible && net_out) *net_out = std::move(pre.nw);
  return cs;
}

// Alg. 3 lines 21-24: all |U|+1 cases, argmin total, ties -> smallest n (R14).
static AggCase plan_aggregation_probed(const std::vector<Item> &items, const Ctx &c, const std::vector<int> &dsts,
                                       const std::vector<int> &aggs, Net *net_out, const PrefixHint &hint,
                                       AggProbe &pr);

static AggCase plan_aggregation(const std::vector<Item> &items, const Net &net0, const Ctx &c,
                                const std::vector<int> &dsts, const std::vector<int> &aggs, Net *net_out,
                                bool record = false, const PrefixHint *hint = nullptr, AggProbe *probe = nullptr) {
  const int N = (int)items.size();
  // no aggregators: every case n < |U| meets aid = 1 > k at its first tail item (R12), so
  // only the all-direct case is feasible
  if (aggs.empty()) return det_agg(N, items, net0, c, dsts, aggs, net_out, record);
  if (probe && hint && !record && (int)probe->tmax.size() == N + 1)
    return plan_aggregation_probed(items, c, dsts, aggs, net_out, *hint, *probe);
  std::vector<i64> totals(N + 1, -1);
  // contiguous ranges of n per task; the prefix states at the range starts are built in
  // one sequential pass, then every task extends its own copy incrementally
  // (small batches: one task, no dispatch overhead)
  const int tasks = (N + 1) * (int)dsts.size() < 256 ? 1 : std::max(1, std::min(N + 1, 2 * Pool::get().threads()));
  // With Alg. 2's reservations at hand (hint) every task replays its own start prefix from the
  // batch-start network (cheap merges, in parallel); otherwise the starts are sent in one
  // sequential pass and copied.
  const bool replay = hint && tasks > 1;
  std::vector<Prefix> starts;
  starts.reserve(tasks);
  if (replay) {
    for (int t = 0; t < tasks; ++t) starts.emplace_back(net0, hint);
  } else {
    Prefix pre(net0, hint);
    int done = 0;
    for (int t = 0; t < tasks; ++t) {
      const int n0 = (int)((int64_t)(N + 1) * t / tasks);
      for (; done < n0; ++done) pre.extend(items, done, c, dsts);
      starts.push_back(pre);
    }
  }
  std::atomic<bool> failed{false};
  PlanFail first_err{MLF_OK, ""};
  std::mutex err_m;
  // Exact pruning for the argmin (ties -> smallest n): a case's total is its running t_max,
  // which only grows, so a case (or its tail) whose t_max exceeds the best total found so far
  // by any task cannot be the argmin; and the direct prefix's t_max is nondecreasing in n, so
  // once it exceeds the best, every larger n of this task is pruned too.  Strict comparisons:
  // an equal total from a smaller n must still be found.  With Alg. 2's reservations at hand
  // the all-direct total (the largest kept t_en) seeds the bound.
  i64 seed = T_INF;
  if (hint && (int)hint->sends->size() == N) {
    seed = 0;
    for (const Send &x : *hint->sends) seed = std::max(seed, x.t_en);
  }
  std::atomic<i64> best_total{seed};
  // every task keeps its best case (smallest total, then smallest n) with the network after it,
  // so the argmin's plan needs no recomputation
  struct Best {
    int n = -1;
    AggCase cs;
    std::unique_ptr<Net> nw;
  };
  std::vector<Best> tbest(tasks);
  Pool::get().run(
      tasks,
      [&](int t) {
        try {
          const int n0 = (int)((int64_t)(N + 1) * t / tasks), n1 = (int)((int64_t)(N + 1) * (t + 1) / tasks);
          if (n0 >= n1) return;
          Prefix &pre = starts[t];
          if (replay)
            for (int i = 0; i < n0; ++i) pre.extend(items, i, c, dsts);
          thread_local Transfer tr;
          std::unique_ptr<Net> scratch;                // reused across cases (keeps its buffers)
          for (int n = n0; n < n1; ++n) {
            if (!pre.ok) break;
            const i64 cut = best_total.load(std::memory_order_relaxed);
            if (pre.t_max > cut) break;
            // the tail's first step, read-only: with a server-bound transfer already made
            // (n > 0) an item that cannot reach agg[0] by t_max leaves group 1 empty, and the
            // case is infeasible (R12) — most cases end here, without copying the network
            bool dead = false;
            if (n > 0 && n < N) {
              dead = !transfer(pre.nw, nullptr, nullptr, items[n].size, items[n].node, aggs[0], items[n].t_avail, tr) ||
                     tr.t_en > pre.t_max;
            }
            if (!dead) {
              AggCase cs;
              cs.n = n;
              cs.commits = pre.commits;
              if (scratch)
                *scratch = pre.nw;
              else
                scratch = std::make_unique<Net>(pre.nw);
              std::unique_ptr<Net> nw = std::move(scratch);
              det_agg_tail(cs, *nw, pre.t_max, items, c, dsts, aggs, cut);
              totals[n] = cs.feasible ? cs.total : -1;
              if (cs.feasible) {
                Best &b = tbest[t];
                if (b.n < 0 || cs.total < b.cs.total) {
                  b.n = n;
                  b.cs = std::move(cs);
                  std::swap(b.nw, nw);                 // the previous best's network becomes scratch
                }
                i64 cur = best_total.load(std::memory_order_relaxed);
                while (b.cs.total < cur &&
                       !best_total.compare_exchange_weak(cur, b.cs.total, std::memory_order_relaxed)) {
                }
              }
              if (nw) scratch = std::move(nw);
            }
            if (n < N) pre.extend(items, n, c, dsts);
          }
        } catch (const PlanFail &e) {
          std::lock_guard<std::mutex> g(err_m);
          if (!failed.exchange(true)) first_err = e;
        }
      },
      2);
  if (failed.load()) throw first_err;
  int best = -1;
  for (int n = 0; n <= N; ++n)
    if (totals[n] >= 0 && (best < 0 || totals[n] < totals[best])) best = n;
  if (best < 0) throw PlanFail{MLF_E_UNSCHEDULABLE, "no feasible aggregation case"};
  if (!record)
    for (auto &b : tbest)
      if (b.n == best) {
        if (net_out) *net_out = std::move(*b.nw);
        return std::move(b.cs);
      }
  return det_agg(best, items, net0, c, dsts, aggs, net_out, record);
}

// Alg. 3's argmin over n with Alg. 2's networks at hand (AggProbe): only the cases that get past
// their first tail item run, each from the nearest snapshot plus at most kEvery-1 replayed
// reservations, all independent (one pool task per case, in increasing n so the pruning bound
// tightens early).  Same cases, same networks, same pruning rule and tie-break as
// plan_aggregation, so the same argmin; the argmin's case is run once more for its plan.
static AggCase plan_aggregation_probed(const std::vector<Item> &items, const Ctx &c, const std::vector<int> &dsts,
                                       const std::vector<int> &aggs, Net *net_out, const PrefixHint &hint,
                                       AggProbe &pr) {
  const int N = (int)items.size();
  std::vector<int> live;
  for (int n = 0; n <= N; ++n)
    if (!pr.dead[n]) live.push_back(n);
  std::vector<i64> totals(N + 1, -1);
  totals[N] = pr.tmax[N];                        // all direct: feasible, total = the largest t_en
  std::atomic<i64> best_total{pr.tmax[N]};
  std::atomic<bool> failed{false};
  PlanFail first_err{MLF_OK, ""};
  std::mutex err_m;
  // case n on `nw`: the network after its direct prefix, then the tail
  auto run_case = [&](int n, Net &nw, i64 cut, AggCase &cs) {
    const int j = n / AggProbe::kEvery;
    nw = pr.snaps[j];
    for (int i = j * AggProbe::kEvery; i < n; ++i) apply_pending(nw, (*hint.res)[i]);
    cs.n = n;
    cs.commits.clear();
    for (int i = 0; i < n; ++i) cs.commits.push_back({i, 1, 0, (*hint.sends)[i]});
    det_agg_tail(cs, nw, pr.tmax[n], items, c, dsts, aggs, cut);
  };
  const bool small = (N + 1) * (int)dsts.size() < 256;
  // a feasible case keeps its plan and network (few cases are feasible), so the argmin's needs
  // no second run: a feasible case never exceeded the bound it ran with, so it is exactly the
  // unbounded DetAgg(n)
  std::vector<AggCase> fcase(live.size());
  std::vector<std::unique_ptr<Net>> fnet(live.size());
  Pool::get().run(
      (int)live.size(),
      [&](int q) {
        const int n = live[q];
        if (n == N) return;
        try {
          const i64 cut = best_total.load(std::memory_order_relaxed);
          if (pr.tmax[n] > cut) return;                // total >= tmax[n] > the best so far
          thread_local std::unique_ptr<Net> nw;
          if (!nw) nw = std::make_unique<Net>(pr.snaps[0]);
          AggCase cs;
          run_case(n, *nw, cut, cs);
          if (!cs.feasible) return;
          totals[n] = cs.total;
          fcase[q] = cs;
          fnet[q] = std::move(nw);                     // the next case on this thread makes a new one
          i64 cur = best_total.load(std::memory_order_relaxed);
          while (cs.total < cur && !best_total.compare_exchange_weak(cur, cs.total, std::memory_order_relaxed)) {
          }
        } catch (const PlanFail &e) {
          std::lock_guard<std::mutex> g(err_m);
          if (!failed.exchange(true)) first_err = e;
        }
      },
      small ? std::numeric_limits<int>::max() : 2);
  if (failed.load()) throw first_err;
  int best = -1;
  for (int n = 0; n <= N; ++n)
    if (totals[n] >= 0 && (best < 0 || totals[n] < totals[best])) best = n;
  AggCase cs;
  if (best == N) {
    cs.n = N;
    for (int i = 0; i < N; ++i) cs.commits.push_back({i, 1, 0, (*hint.sends)[i]});
    cs.feasible = true;
    cs.total = pr.tmax[N];
    if (net_out) *net_out = std::move(*pr.last);
    return cs;
  }
  const int qb = (int)(std::lower_bound(live.begin(), live.end(), best) - live.begin());
  if (qb >= (int)live.size() || live[qb] != best || !fnet[qb] || fcase[qb].total != totals[best])
    throw PlanFail{MLF_E_INVALID, "internal: aggregation case lost"};
  if (net_out) *net_out = std::move(*fnet[qb]);
  return std::move(fcase[qb]);
}

static std::vector<i64> chained_times(const std::vector<CommitRec> &cm) {
  std::vector<i64> out;
  i64 prev = 0;
  for (auto &x : cm) {
    prev = std::max(prev, x.send.t_en);
    out.push_back(prev);
  }
  return out;
}

// ---------------------------------------------------------------- O5 replication
// Eq. 9/12 bound with the momentum coefficients (R15); fixed evaluation order.
static double divergence_bound(const double *norms, int m, double gamma, double h0) {
  if (m == 0) return 0.0;
  thread_local std::vector<double> pw, cum;
  pw.resize(m + 1);
  cum.resize(m + 1);
  pw[0] = 1.0;
  for (int j = 1; j <= m; ++j) pw[j] = pw[j - 1] * gamma;
  double coef_h = 0.0;
  for (int j = 1; j <= m; ++j) coef_h += pw[j];
  // cum[k] = pw[0] + ... + pw[k], summed left to right: the same additions in the same order
  // as summing each coefficient on its own, so every coefficient is bitwise the same
  cum[0] = pw[0];
  for (int k = 1; k <= m; ++k) cum[k] = cum[k - 1] + pw[k];
  double d = coef_h * h0;
  for (int i = 1; i <= m; ++i) d += cum[m - i] * norms[i - 1];
  return d;
}

}  // namespace mlf

using namespace mlf;

static thread_local std::string g_plan_err;
const char *mlf_planner_last_error() { return g_plan_err.c_str(); }

static mlf_status plan_impl(const mlf_net *net, const mlf_batch *batch, const mlf_plan_params *prm,
                            mlf_plan_out *out) {
  if (!net || !batch || !prm || !out) throw PlanFail{MLF_E_INVALID, "null argument"};
  if (net->n_nodes < 1 || !net->nic_up || !net->nic_down) throw PlanFail{MLF_E_INVALID, "bad network"};
  Ctx c;
  c.d.n = net->n_nodes;
  c.d.up = net->nic_up;
  c.d.down = net->nic_down;
  c.d.bw = net->bw;
  c.d.site = net->site;
  const int nn = net->n_nodes;
  auto node_ok = [&](int x) { return x >= 0 && x < nn; };
  const int n = batch->n;
  if (n < 0) throw PlanFail{MLF_E_INVALID, "batch n < 0"};
  if (n > 0 && (!batch->node || !batch->bytes || !batch->version || !batch->t_avail_ns || !batch->norm))
    throw PlanFail{MLF_E_INVALID, "null batch array"};
  if (prm->n_servers < 1 || !prm->server) throw PlanFail{MLF_E_INVALID, "no server"};
  for (int j = 0; j < prm->n_servers; ++j) {
    if (!node_ok(prm->server[j])) throw PlanFail{MLF_E_INVALID, "server node out of range"};
    c.servers.push_back(prm->server[j]);
  }
  if (prm->k < 0 || (prm->k > 0 && !prm->agg)) throw PlanFail{MLF_E_INVALID, "aggregators"};
  for (int i = 0; i < prm->k; ++i) {
    if (!node_ok(prm->agg[i])) throw PlanFail{MLF_E_INVALID, "aggregator node out of range"};
    c.aggs.push_back(prm->agg[i]);
  }
  if (prm->n_replicas != 0 && prm->n_replicas != prm->n_servers)
    throw PlanFail{MLF_E_INVALID, "replica count must equal server count"};
  if (prm->n_replicas > 0 && !prm->replica) throw PlanFail{MLF_E_INVALID, "replica nodes"};
  for (int j = 0; j < prm->n_replicas; ++j) {
    if (!node_ok(prm->replica[j])) throw PlanFail{MLF_E_INVALID, "replica node out of range"};
    c.replicas.push_back(prm->replica[j]);
  }
  if (prm->k_r < 0 || (prm->k_r > 0 && !prm->replica_agg)) throw PlanFail{MLF_E_INVALID, "replica aggregators"};
  for (int i = 0; i < prm->k_r; ++i) {
    if (!node_ok(prm->replica_agg[i])) throw PlanFail{MLF_E_INVALID, "replica aggregator out of range"};
    c.raggs.push_back(prm->replica_agg[i]);
  }
  if (prm->replica_mode != 0 && prm->replica_mode != 1) throw PlanFail{MLF_E_INVALID, "replica_mode"};
  if (prm->sync_mode != 0 && prm->sync_mode != 1) throw PlanFail{MLF_E_INVALID, "sync_mode"};
  if (prm->tau_max < 0 || !(prm->div_max >= 0) || !(prm->gamma >= 0.0 && prm->gamma < 1.0))
    throw PlanFail{MLF_E_INVALID, "tau_max / div_max / gamma"};
  if (!(prm->hist_norm >= 0 && std::isfinite(prm->hist_norm))) throw PlanFail{MLF_E_INVALID, "hist_norm"};
  if (prm->n_carried < 0 || (prm->n_carried > 0 && (!prm->carried_node || !prm->carried_bytes || !prm->carried_norm)))
    throw PlanFail{MLF_E_INVALID, "carried items"};
  for (int j = 0; j < prm->n_servers; ++j) {
    i64 w = prm->shard_weight ? prm->shard_weight[j] : 1;
    if (w <= 0) throw PlanFail{MLF_E_INVALID, "shard weights"};
    c.weights.push_back(w);
    c.wsum += w;
  }
  auto has_dup = [](std::vector<int> v) {
    std::sort(v.begin(), v.end());
    return std::adjacent_find(v.begin(), v.end()) != v.end();
  };
  c.dup_dsts = has_dup(c.servers) || has_dup(c.replicas);
  std::vector<Item> items(n), carried(prm->n_carried);
  for (int g = 0; g < n; ++g) {
    items[g] = {batch->node[g], batch->bytes[g], batch->version[g], batch->t_avail_ns[g], batch->norm[g]};
    if (!node_ok(items[g].node)) throw PlanFail{MLF_E_INVALID, "update node out of range"};
    if (items[g].size < 0 || items[g].t_avail < 0 || !(items[g].norm >= 0 && std::isfinite(items[g].norm)))
      throw PlanFail{MLF_E_INVALID, "bad update descriptor"};
  }
  for (int g = 0; g < prm->n_carried; ++g) {
    carried[g] = {prm->carried_node[g], prm->carried_bytes[g], 0, 0, prm->carried_norm[g]};
    if (!node_ok(carried[g].node)) throw PlanFail{MLF_E_INVALID, "carried node out of range"};
    if (carried[g].size < 0 || !(carried[g].norm >= 0 && std::isfinite(carried[g].norm)))
      throw PlanFail{MLF_E_INVALID, "bad carried descriptor"};
  }
  if (out->capacity < n + prm->n_carried ||
      (n > 0 && (!out->order || !out->drop_reason || !out->group || !out->commit_first || !out->commit_count ||
                 !out->commit_t_ns)) ||
      ((n + prm->n_carried) > 0 && !out->punted) || (n > 0 && prm->k > 0 && !out->group_node) ||
      (prm->n_replicas > 0 && (n + prm->n_carried) > 0 &&
       (!out->replica_commit_first || !out->replica_commit_count || !out->replica_commit_group)))
    throw PlanFail{MLF_E_CAPACITY, "output arrays too small or missing"};
  // unschedulable pre-check (R9)
  std::vector<i64> comp;
  for (auto &it : items) {
    component_bytes(it.size, c.weights, c.wsum, comp);
    for (size_t j = 0; j < c.servers.size(); ++j)
      if (comp[j] > 0 && path_dead(c.d, it.node, c.servers[j]))
        throw PlanFail{MLF_E_UNSCHEDULABLE, "update path to a server is down"};
  }
  if (!c.replicas.empty()) {
    auto chk = [&](const Item &it) {
      component_bytes(it.size, c.weights, c.wsum, comp);
      for (size_t j = 0; j < c.replicas.size(); ++j)
        if (comp[j] > 0 && path_dead(c.d, it.node, c.replicas[j]))
          throw PlanFail{MLF_E_UNSCHEDULABLE, "update path to a replica is down"};
    };
    for (auto &it : carried) chk(it);
    for (auto &it : items) chk(it);
  }

  // 1. ordering
  // (sync mode: no ordering — the list in submission order, nothing dropped)
  OrderRes ores;
  AggProbe probe;
  probe.aggs = &c.aggs;
  if (prm->sync_mode) {
    for (int g = 0; g < n; ++g) ores.order.push_back(g);
    ores.reason.assign(n, 0);
  } else {
    ores = order_final(c, items, prm->tau_max, prm->v_init, c.aggs.empty() ? nullptr : &probe);
  }
  std::vector<Item> ordered;
  for (int g : ores.order) ordered.push_back(items[g]);
  // 2. aggregation on the batch-start network (R10)
  Net net0(&c.d);
  Net after(&c.d);
  PrefixHint hint{&ores.res, &ores.sends};
  AggCase cs = plan_aggregation(ordered, net0, c, c.servers, c.aggs, &after, false,
                                prm->sync_mode ? nullptr : &hint, prm->sync_mode ? nullptr : &probe);
  std::vector<i64> times = chained_times(cs.commits);

  out->n_commit = (int)ores.order.size();
  for (int g = 0; g < n; ++g) {
    out->drop_reason[g] = ores.reason[g];
    out->group[g] = -1;
  }
  for (size_t p = 0; p < ores.order.size(); ++p) out->order[p] = ores.order[p];
  int n_groups = 0;
  for (size_t ci = 0; ci < cs.commits.size(); ++ci) {
    auto &cm = cs.commits[ci];
    out->commit_first[ci] = cm.first;
    out->commit_count[ci] = cm.count;
    out->commit_t_ns[ci] = times[ci];
    for (int p = cm.first; p < cm.first + cm.count; ++p) out->group[ores.order[p]] = cm.group;
    if (cm.group > 0) ++n_groups;
  }
  out->n_direct = cs.n;
  out->n_groups = n_groups;
  for (int i = 0; i < n_groups; ++i) out->group_node[i] = c.aggs[i];
  out->n_server_commits = (int)cs.commits.size();
  out->replica_frozen = 0;
  out->replica_boundary_commit = -1;
  out->n_punted = 0;
  out->n_replica_commits = 0;
  out->replica_bytes = 0;
  out->sync_mode = (uint8_t)prm->sync_mode;
  out->delayed_last = 0;
  out->t_total_ns = times.empty() ? 0 : times.back();

  // 3. replication (§5.3) on the network after the server plan
  if (!c.replicas.empty()) {
    std::vector<Item> ritems(carried);
    ritems.insert(ritems.end(), ordered.begin(), ordered.end());
    const int n_c = (int)carried.size();
    AggCase rc = plan_aggregation(ritems, after, c, c.replicas, c.raggs, nullptr);
    std::vector<i64> rtimes = chained_times(rc.commits);
    i64 t_last = times.empty() ? 0 : times.back();
    std::vector<int> ends;
    int acc = 0;
    for (auto &x : rc.commits) {
      acc += x.count;
      ends.push_back(acc);
    }
    size_t n_pre = 0;
    while (n_pre < rtimes.size() && rtimes[n_pre] <= t_last) ++n_pre;
    int frozen = n_pre ? ends[n_pre - 1] : 0;
    size_t n_fc = n_pre;                                     // frozen replica commits
    std::vector<double> norms;
    for (auto &it : ritems) norms.push_back(it.norm);
    const int R = (int)ritems.size();
    double bound = divergence_bound(norms.data() + frozen, R - frozen, prm->gamma, prm->hist_norm);
    bool delayed = false;
    if (bound > prm->div_max) {
      int a_e = -1;
      for (size_t ci = n_pre; ci < rc.commits.size(); ++ci) {
        if (divergence_bound(norms.data() + ends[ci], R - ends[ci], prm->gamma, prm->hist_norm) <= prm->div_max) {
          a_e = (int)ci;
          break;
        }
      }
      if (a_e < 0) throw PlanFail{MLF_E_INVALID, "internal: no replica commit meets Div_max"};
      frozen = ends[a_e];
      n_fc = (size_t)a_e + 1;
      if (!cs.commits.empty()) {
        delayed = true;
        const Send &last = cs.commits.back().send;
        i64 shift = std::max<i64>(0, rtimes[a_e] - last.t_st);
        i64 new_end = last.t_en + shift;
        i64 prev = times.size() > 1 ? times[times.size() - 2] : 0;
        t_last = std::max(prev, new_end);
      }
    }
    // the frozen replica commits and the bytes they deliver (a direct item or one aggregate)
    int64_t rbytes = 0;
    for (size_t ci = 0; ci < n_fc; ++ci) {
      const CommitRec &x = rc.commits[ci];
      out->replica_commit_first[ci] = x.first;
      out->replica_commit_count[ci] = x.count;
      out->replica_commit_group[ci] = x.group;
      i64 mx = 0;
      for (int q = x.first; q < x.first + x.count; ++q) mx = std::max(mx, ritems[q].size);
      rbytes += mx;
    }
    out->n_replica_commits = (int)n_fc;
    out->replica_bytes = rbytes;
    // R16 mirror boundary (mode 0); replica trees (mode 1): exactly the frozen prefix
    int f_o = std::max(0, frozen - n_c), boundary, covered;
    if (prm->replica_mode == 1) {
      boundary = -1;
      covered = frozen;
    } else if (frozen == 0) {
      boundary = -1;
      covered = 0;
    } else if (f_o == 0) {
      boundary = 0;
      covered = n_c;
    } else {
      int a2 = 0;
      boundary = -1;
      for (size_t ci = 0; ci < cs.commits.size(); ++ci) {
        a2 += cs.commits[ci].count;
        if (a2 >= f_o) {
          boundary = (int)ci + 1;
          break;
        }
      }
      covered = n_c + a2;
    }
    out->replica_frozen = covered;
    out->replica_boundary_commit = boundary;
    out->n_punted = R - covered;
    for (int i = covered; i < R; ++i) out->punted[i - covered] = i;
    out->delayed_last = delayed ? 1 : 0;
    if (delayed) out->commit_t_ns[cs.commits.size() - 1] = t_last;
    out->t_total_ns = t_last;
  }
  return MLF_OK;
}

extern "C" mlf_status mlf_plan(const mlf_net *net, const mlf_batch *batch, const mlf_plan_params *params,
                               mlf_plan_out *out) {
  try {
    g_plan_err.clear();
    return plan_impl(net, batch, params, out);
  } catch (const PlanFail &e) {
    g_plan_err = e.msg;
    mlf_set_error(e.msg.c_str());
    return e.code;
  } catch (const std::exception &e) {
    g_plan_err = e.what();
    mlf_set_error(e.what());
    return MLF_E_INVALID;
  } catch (...) {
    mlf_set_error("unknown planner error");
    return MLF_E_INVALID;
  }
}

// ---------------------------------------------------------------- NEXT-4 distribution
// App. B.3 under readings R23-R25: Alg. 3 on the transposed network
// (up <-> down, pair (i, j) <-> (j, i)) over the pull requests in Alg. 1's SJF order;
// the schedule mirrored by t -> T - t is the real one.
static mlf_status plan_dist_impl(const mlf_net *net, int32_t n, const int32_t *req, const mlf_dist_params *prm,
                                 mlf_dist_out *out) {
  if (!net || !prm || !out || (n > 0 && !req)) throw PlanFail{MLF_E_INVALID, "null argument"};
  if (net->n_nodes < 1 || !net->nic_up || !net->nic_down) throw PlanFail{MLF_E_INVALID, "bad network"};
  if (n < 0 || prm->model_bytes < 0) throw PlanFail{MLF_E_INVALID, "n_requests / model_bytes"};
  const int nn = net->n_nodes;
  auto node_ok = [&](int x) { return x >= 0 && x < nn; };
  std::vector<int64_t> up(net->nic_down, net->nic_down + nn), down(net->nic_up, net->nic_up + nn), bw;
  if (net->bw) {
    bw.resize((size_t)nn * nn);
    for (int i = 0; i < nn; ++i)
      for (int j = 0; j < nn; ++j) bw[(size_t)i * nn + j] = net->bw[(size_t)j * nn + i];
  }
  Ctx c;
  c.d.n = nn;
  c.d.up = up.data();
  c.d.down = down.data();
  c.d.bw = net->bw ? bw.data() : nullptr;
  c.d.site = net->site;
  if (prm->n_servers < 1 || !prm->server) throw PlanFail{MLF_E_INVALID, "no server"};
  for (int j = 0; j < prm->n_servers; ++j) {
    if (!node_ok(prm->server[j])) throw PlanFail{MLF_E_INVALID, "server node out of range"};
    c.servers.push_back(prm->server[j]);
    const i64 w = prm->shard_weight ? prm->shard_weight[j] : 1;
    if (w <= 0) throw PlanFail{MLF_E_INVALID, "shard weights"};
    c.weights.push_back(w);
    c.wsum += w;
  }
  if (prm->k < 0 || (prm->k > 0 && !prm->distributor)) throw PlanFail{MLF_E_INVALID, "distributors"};
  for (int i = 0; i < prm->k; ++i) {
    if (!node_ok(prm->distributor[i])) throw PlanFail{MLF_E_INVALID, "distributor node out of range"};
    c.aggs.push_back(prm->distributor[i]);
  }
  auto has_dup = [](std::vector<int> v) {
    std::sort(v.begin(), v.end());
    return std::adjacent_find(v.begin(), v.end()) != v.end();
  };
  c.dup_dsts = has_dup(c.servers);
  std::vector<Item> items(n);
  for (int i = 0; i < n; ++i) {
    if (!node_ok(req[i])) throw PlanFail{MLF_E_INVALID, "request node out of range"};
    items[i] = {req[i], prm->model_bytes, 0, 0, 0.0};
  }
  if (out->capacity < n || (n > 0 && (!out->order || !out->group || !out->t_recv_ns || !out->t_start_ns)) ||
      (n > 0 && prm->k > 0 && (!out->group_node || !out->t_dist_ns)))
    throw PlanFail{MLF_E_CAPACITY, "output arrays too small or missing"};
  std::vector<i64> comp;
  component_bytes(prm->model_bytes, c.weights, c.wsum, comp);
  for (auto &it : items)
    for (size_t j = 0; j < c.servers.size(); ++j)
      if (comp[j] > 0 && path_dead(c.d, it.node, c.servers[j]))
        throw PlanFail{MLF_E_UNSCHEDULABLE, "a request's path from a server is down"};
  // R24: Alg. 1 (SJF, no deadlines) on the transposed network; requests from one node
  // are interchangeable, so each distinct node is evaluated once per step
  std::vector<int> order, unproc(n);
  for (int i = 0; i < n; ++i) unproc[i] = i;
  Net nw(&c.d);
  Pending local;
  while (!unproc.empty()) {
    std::unordered_map<int, i64> ten;
    int best = -1;
    i64 best_t = 0;
    for (int g : unproc) {
      auto it = ten.find(items[g].node);
      if (it == ten.end()) {
        Send s;
        if (!send(nw, nullptr, c, c.servers, items[g].node, items[g].size, 0, s, local, false))
          throw PlanFail{MLF_E_UNSCHEDULABLE, "a request's path from a server is down"};
        it = ten.emplace(items[g].node, s.t_en).first;
      }
      if (best < 0 || it->second < best_t) {
        best = g;
        best_t = it->second;
      }
    }
    Send s;
    send_apply(nw, c, c.servers, items[best].node, items[best].size, 0, s);
    order.push_back(best);
    unproc.erase(std::find(unproc.begin(), unproc.end(), best));
  }
  std::vector<Item> ordered(n);
  for (int p = 0; p < n; ++p) ordered[p] = items[order[p]];
  const Net net0(&c.d);
  AggCase cs = plan_aggregation(ordered, net0, c, c.servers, c.aggs, nullptr, true);
  const i64 T = cs.total;
  int n_groups = 0;
  for (auto &cm : cs.commits) {
    if (cm.group == 0) {
      const int g = order[cm.first];
      out->group[g] = 0;
      out->t_recv_ns[g] = T - cm.send.t_st;
      out->t_start_ns[g] = T - cm.send.t_en;
      continue;
    }
    out->t_dist_ns[cm.group - 1] = T - cm.send.t_st;
    out->group_node[cm.group - 1] = c.aggs[cm.group - 1];
    n_groups = std::max(n_groups, cm.group);
    for (int p = cm.first; p < cm.first + cm.count; ++p) {
      const int g = order[p];
      out->group[g] = cm.group;
      out->t_recv_ns[g] = T - cs.m_st[p - cs.n];
      out->t_start_ns[g] = T - cs.m_en[p - cs.n];
    }
  }
  for (int p = 0; p < n; ++p) out->order[p] = order[p];
  out->n_direct = cs.n;
  out->n_groups = n_groups;
  out->t_total_ns = T;
  return MLF_OK;
}

extern "C" mlf_status mlf_plan_distribution(const mlf_net *net, int32_t n_requests, const int32_t *request_node,
                                            const mlf_dist_params *params, mlf_dist_out *out) {
  try {
    g_plan_err.clear();
    return plan_dist_impl(net, n_requests, request_node, params, out);
  } catch (const PlanFail &e) {
    g_plan_err = e.msg;
    mlf_set_error(e.msg.c_str());
    return e.code;
  } catch (const std::exception &e) {
    g_plan_err = e.what();
    mlf_set_error(e.what());
    return MLF_E_INVALID;
  } catch (...) {
    mlf_set_error("unknown planner error");
    return MLF_E_INVALID;
  }
}
