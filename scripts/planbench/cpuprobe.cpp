// Host CPU parallelism probe: the same fixed integer work on 1..16 threads, wall time each, and
// the round-trip latency of handing a tiny job to a spinning worker thread.  Tells whether the
// box's host gives a process several cores at once (a CPU quota shows up as wall time growing
// with the thread count).
#include <atomic>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>
static volatile unsigned long sink;
static void work(long n) {
  unsigned long x = 88172645463325252ull;
  for (long i = 0; i < n; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; }
  sink = x;
}
int main() {
  const long N = 200000000;
  for (int t : {1, 2, 4, 8, 16}) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int i = 0; i < t; ++i) th.emplace_back(work, N);
    for (auto &x : th) x.join();
    double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    printf("threads %2d: %.1f ms for %d x the same work\n", t, ms, t);
  }
  std::atomic<long> go{0}, done{0};
  std::atomic<bool> stop{false};
  std::thread w([&] { long seen = 0; while (!stop) { long g = go.load(); if (g != seen) { seen = g; done.store(g); } } });
  const int R = 100000;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 1; i <= R; ++i) { go.store(i); while (done.load() != i) {} }
  double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / R;
  stop = true; w.join();
  printf("spinning hand-off round trip: %.3f us\n", us);
}
