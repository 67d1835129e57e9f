"""Print planner.cpp with phase timers (ordering / server aggregation / replica plan) and work
counters (transfers, walk steps, profile merges) added; planbench links it instead of the real
planner to show where a plan's time goes.  usage: python scripts/planbench/prof.py [--light] > /tmp/planner_prof.cpp
--light: the three phase timers only (no per-transfer counters, no per-scan timers), for
multi-threaded runs where contended counters would distort the timing."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
s = open(os.path.join(ROOT, "paper_1907_00434_b200", "csrc", "planner.cpp")).read()


def sub(old, new):
    global s
    assert old in s, old[:60]
    s = s.replace(old, new, 1)


sub('#include "planner.h"', '''#include "planner.h"
#include <chrono>
#include <cstdio>
static long N_tr = 0, N_it = 0, N_tr_ord = 0, N_comb = 0;
static double T_ord = 0, T_agg = 0, T_rep = 0, T_all = 0, T_scan = 0, T_star = 0, T_app = 0, T_pick = 0;
static int NCALL = 0;
struct Dump {
  ~Dump() {
    if (NCALL)
      fprintf(stderr, "per plan: all %.3f ms = ordering %.3f + aggregation %.3f + replica %.3f + rest; "
              "transfers %ld (ordering %ld), walk steps %ld, profile merges %ld\\n", T_all / NCALL, T_ord / NCALL,
              T_agg / NCALL, T_rep / NCALL, N_tr / NCALL, N_tr_ord / NCALL, N_it / NCALL, N_comb / NCALL);
    if (NCALL)
      fprintf(stderr, "  ordering: picks %.3f ms (of which class tasks %.3f), g* reservation %.3f, NetUp+copy %.3f\\n",
              T_pick / NCALL, T_scan / NCALL, T_star / NCALL, T_app / NCALL);
  }
} g_dump;
#define NOW std::chrono::steady_clock::now()
#define MS(a, b) std::chrono::duration<double, std::milli>(b - a).count()''')
sub('''    ores = order_final(c, items, prm->tau_max, prm->v_init, c.aggs.empty() ? nullptr : &probe);''',
    '''    auto t0 = NOW; long n0 = N_tr; ores = order_final(c, items, prm->tau_max, prm->v_init, c.aggs.empty() ? nullptr : &probe);
    T_ord += MS(t0, NOW); N_tr_ord += N_tr - n0;''')
sub('''  AggCase cs = plan_aggregation(ordered, net0, c, c.servers, c.aggs, &after, false,
                                prm->sync_mode ? nullptr : &hint, prm->sync_mode ? nullptr : &probe);''', '''  auto ta = NOW; AggCase cs = plan_aggregation(ordered, net0, c, c.servers, c.aggs, &after, false,
                                prm->sync_mode ? nullptr : &hint, prm->sync_mode ? nullptr : &probe); T_agg += MS(ta, NOW);''')
sub('''    AggCase rc = plan_aggregation(ritems, after, c, c.replicas, c.raggs, nullptr);''',
    '''    auto tr_ = NOW; AggCase rc = plan_aggregation(ritems, after, c, c.replicas, c.raggs, nullptr); T_rep += MS(tr_, NOW);''')
sub('''  try {
    g_plan_err.clear();
    return plan_impl(net, batch, params, out);''', '''  try {
    g_plan_err.clear();
    NCALL++; auto t2 = NOW; auto r = plan_impl(net, batch, params, out); T_all += MS(t2, NOW); return r;''')
LIGHT = "--light" in sys.argv
if LIGHT:
    def sub(old, new):  # noqa: F811 — counters and scan timers off
        pass
sub('''  const NetDef &d = *net.def;
  out.segs.clear();''', '''  const NetDef &d = *net.def;
  __atomic_add_fetch(&N_tr, 1, __ATOMIC_RELAXED);
  out.segs.clear();''')
sub('''    if (r < 0) throw PlanFail{MLF_E_INVALID, "internal: negative residual"};''', '''    __atomic_add_fetch(&N_it, 1, __ATOMIC_RELAXED);
    if (r < 0) throw PlanFail{MLF_E_INVALID, "internal: negative residual"};''')
sub('''  if (ev.empty()) return;''', '''  __atomic_add_fetch(&N_comb, 1, __ATOMIC_RELAXED);
  if (ev.empty()) return;''')
# ordering sub-phases (present in the round-2 planner; skipped silently otherwise)
def opt(old, new):
    global s
    if old in s:
        s = s.replace(old, new, 1)


if LIGHT:
    def opt(old, new):  # noqa: F811
        pass
opt('''    Pool::get().run(
        (int)miss.size(),''', '''    auto tsc = NOW;
    struct ScanT { std::chrono::steady_clock::time_point t; ~ScanT() { T_scan += MS(t, NOW); } };
    ScanT scan_t{tsc};
    Pool::get().run(
        (int)miss.size(),''')
opt('''    const int g_star = cached >= 0 ? cached : pick(p, unproc, nullptr);''', '''    auto tp0 = NOW;
    const int g_star = cached >= 0 ? cached : pick(p, unproc, nullptr);
    T_pick += MS(tp0, NOW);
    auto tst = NOW;''')
opt('''    cands.clear();
    for (int g : unproc)
      if (g != g_star && dl[g] >= p + 1) cands.push_back(g);''', '''    T_star += MS(tst, NOW);
    cands.clear();
    for (int g : unproc)
      if (g != g_star && dl[g] >= p + 1) cands.push_back(g);''')
opt('''      g_next = pick(p + 1, cands, &star, use_side ? &side : nullptr, &side_ran);   // on NetUp(NW, g*)''',
    '''      auto tp1 = NOW;
      g_next = pick(p + 1, cands, &star, use_side ? &side : nullptr, &side_ran);   // on NetUp(NW, g*)
      T_pick += MS(tp1, NOW);''')
opt('''    if (stream) probe->ord.push_back(batch[g_star]);
    if (side_ran) {''', '''    auto tap = NOW;
    if (side_ran) {''')
opt('''    if (side_ran) {
      if (probe) {''', '''    auto tap = NOW;
    if (side_ran) {
      if (probe) {''')
opt('''    res.sends.push_back(s_star);''', '''    res.sends.push_back(s_star);
    T_app += MS(tap, NOW);''')
sys.stdout.write(s)
