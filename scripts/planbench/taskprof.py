"""Print planner.cpp with an Alg. 2 scan-task profile added (items per scan, the share of scans
on the pool, wall time of the scans against the summed and the longest task per scan, task time
per thread); planbench links it instead of the real planner.
usage: python scripts/planbench/taskprof.py > /tmp/planner_taskprof.cpp"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
s = open(os.path.join(ROOT, "paper_1907_00434_b200", "csrc", "planner.cpp")).read()


def sub(old, new):
    global s
    assert s.count(old) == 1, old[:60]
    s = s.replace(old, new)


sub('namespace mlf {', '''#include <chrono>
#include <cstdio>
static double S_wall = 0, S_sum = 0, S_max = 0;
static long S_scans = 0, S_items = 0, S_par = 0;
static int S_calls = 0;
static thread_local int S_tid = -1;
static std::atomic<int> S_ntid{0};
static double S_thr[64];
struct SDump {
  ~SDump() {
    if (!S_calls) return;
    fprintf(stderr, "scans/plan %.1f items/scan %.1f parallel scans %.1f%%: wall %.3f sum %.3f max-task %.3f ms/plan\\n",
            (double)S_scans / S_calls, (double)S_items / S_scans, 100.0 * S_par / S_scans, S_wall / S_calls,
            S_sum / S_calls, S_max / S_calls);
    fprintf(stderr, "per-thread task ms/plan:");
    for (int i = 0; i < S_ntid.load() && i < 64; ++i) fprintf(stderr, " %.3f", S_thr[i] / S_calls);
    fprintf(stderr, "\\n");
  }
} g_sdump;
namespace mlf {''')
sub('''    Pool::get().run(
        (int)miss.size(),
        [&](int i) {
          thread_local Pending local;''', '''    std::vector<double> tt(miss.size());
    auto w0 = std::chrono::steady_clock::now();
    Pool::get().run(
        (int)miss.size(),
        [&](int i) {
          struct Fin {
            std::vector<double> &tt;
            int i;
            std::chrono::steady_clock::time_point t0;
            ~Fin() {
              double d = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
              tt[i] = d;
              if (S_tid < 0) S_tid = S_ntid++;
              if (S_tid < 64) S_thr[S_tid] += d;
            }
          } fin{tt, i, std::chrono::steady_clock::now()};
          thread_local Pending local;''')
sub('''    if (task_failed.load()) throw task_err;''', '''    if (task_failed.load()) throw task_err;
    S_wall += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
    {
      double sm = 0, mx = 0;
      for (double d : tt) {
        sm += d;
        mx = std::max(mx, d);
      }
      S_sum += sm;
      S_max += mx;
      S_scans++;
      S_items += miss.size();
      if (multi_server && (int)miss.size() >= min_parallel_evals()) S_par++;
    }''')
sub('''  try {
    g_plan_err.clear();
    return plan_impl(net, batch, params, out);''', '''  try {
    S_calls++;
    g_plan_err.clear();
    return plan_impl(net, batch, params, out);''')
sys.stdout.write(s)
