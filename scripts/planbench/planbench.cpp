// planbench — mlf_plan latency and bit-exactness on dumped instances (dev tool).
// build: g++ -O2 -std=c++17 -pthread -ffp-contract=off planbench.cpp ../../paper_1907_00434_b200/csrc/planner.cpp
//        -I../../include -o /tmp/planbench
// usage: planbench FILE [reps] [filter-substring]
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/mlfabric.h"

void mlf_set_error(const char *) {}

template <class T>
static std::vector<T> nums(const std::string &line, int skip = 0) {
  std::istringstream is(line);
  std::vector<T> v;
  std::string tok;
  for (int i = 0; i < skip; ++i) is >> tok;
  T x;
  while (is >> x) v.push_back(x);
  return v;
}

struct Inst {
  std::string name;
  int n_nodes;
  std::vector<int64_t> up, down, bw;
  std::vector<int32_t> site;
  bool has_bw = false, has_site = false;
  int n;
  std::vector<int32_t> node;
  std::vector<int64_t> size, version, tavail;
  std::vector<double> norm;
  std::vector<int32_t> servers, aggs, replicas, raggs;
  std::vector<int64_t> weights;
  bool has_w = false;
  int64_t v_init;
  int tau, rmode, smode;
  double div_max, gamma, hist;
  std::vector<int32_t> cnode;
  std::vector<int64_t> cbytes;
  std::vector<double> cnorm;
  std::string expect;
  int err = 0;
};

static std::string L(const int32_t *a, int n) {
  std::string s;
  for (int i = 0; i < n; ++i) s += (i ? " " : "") + std::to_string(a[i]);
  return s;
}
static std::string L8(const uint8_t *a, int n) {
  std::string s;
  for (int i = 0; i < n; ++i) s += (i ? " " : "") + std::to_string((int)a[i]);
  return s;
}
static std::string L64(const int64_t *a, int n) {
  std::string s;
  for (int i = 0; i < n; ++i) s += (i ? " " : "") + std::to_string(a[i]);
  return s;
}

int main(int argc, char **argv) {
  std::ifstream f(argv[1]);
  const int reps = argc > 2 ? atoi(argv[2]) : 1;
  const std::string filt = argc > 3 ? argv[3] : "";
  std::vector<Inst> all;
  std::string line;
  while (std::getline(f, line)) {
    if (line.rfind("instance ", 0) != 0) continue;
    Inst I;
    I.name = line.substr(9);
    std::getline(f, line); I.n_nodes = std::stoi(line);
    std::getline(f, line); I.up = nums<int64_t>(line);
    std::getline(f, line); I.down = nums<int64_t>(line);
    std::getline(f, line); I.bw = nums<int64_t>(line, 1); I.has_bw = line.size() > 2;
    std::getline(f, line); I.site = nums<int32_t>(line, 1); I.has_site = line.size() > 4;
    std::getline(f, line); I.n = std::stoi(line);
    std::getline(f, line); I.node = nums<int32_t>(line);
    std::getline(f, line); I.size = nums<int64_t>(line);
    std::getline(f, line); I.version = nums<int64_t>(line);
    std::getline(f, line); I.tavail = nums<int64_t>(line);
    std::getline(f, line); I.norm = nums<double>(line);
    std::getline(f, line); I.servers = nums<int32_t>(line);
    std::getline(f, line); I.weights = nums<int64_t>(line, 1); I.has_w = line.size() > 1;
    std::getline(f, line); I.aggs = nums<int32_t>(line, 1);
    std::getline(f, line); I.replicas = nums<int32_t>(line, 1);
    std::getline(f, line); I.raggs = nums<int32_t>(line, 1);
    std::getline(f, line);
    {
      std::istringstream is(line);
      std::string dm, g, h;
      is >> I.v_init >> I.tau >> dm >> g >> h >> I.rmode >> I.smode;
      I.div_max = std::stod(dm);
      I.gamma = std::stod(g);
      I.hist = std::stod(h);
    }
    std::getline(f, line); int nc = std::stoi(line);
    std::getline(f, line); I.cnode = nums<int32_t>(line);
    std::getline(f, line); I.cbytes = nums<int64_t>(line);
    std::getline(f, line); I.cnorm = nums<double>(line);
    (void)nc;
    std::getline(f, line);
    if (line.rfind("expect ", 0) == 0) I.expect = line.substr(7);
    else I.err = std::stoi(line.substr(6));
    if (filt.empty() || I.name.find(filt) != std::string::npos) all.push_back(std::move(I));
  }
  int bad = 0;
  std::string last_group;
  std::vector<double> grp;
  auto flush_group = [&]() {
    if (grp.empty()) return;
    std::sort(grp.begin(), grp.end());
    printf("%-28s n=%3zu (per-instance best of reps) median %8.3f ms  min %8.3f  max %8.3f\n", last_group.c_str(), grp.size(), grp[grp.size() / 2],
           grp.front(), grp.back());
    grp.clear();
  };
  double total = 0;
  for (auto &I : all) {
    const int cap = std::max(1, I.n + (int)I.cnode.size());
    std::vector<int32_t> order(cap), group(cap), gnode(cap), cf(cap), cc(cap), punted(cap), rf(cap), rc(cap), rg(cap);
    std::vector<uint8_t> drop(cap);
    std::vector<int64_t> ct(cap);
    mlf_net net{I.n_nodes, I.up.data(), I.down.data(), I.has_bw ? I.bw.data() : nullptr,
                I.has_site ? I.site.data() : nullptr};
    mlf_batch b{I.n, I.node.data(), I.size.data(), I.version.data(), I.tavail.data(), I.norm.data()};
    mlf_plan_params p{};
    p.n_servers = (int)I.servers.size();
    p.server = I.servers.data();
    p.shard_weight = I.has_w ? I.weights.data() : nullptr;
    p.k = (int)I.aggs.size();
    p.agg = I.aggs.data();
    p.n_replicas = (int)I.replicas.size();
    p.replica = I.replicas.data();
    p.k_r = (int)I.raggs.size();
    p.replica_agg = I.raggs.data();
    p.v_init = I.v_init;
    p.tau_max = I.tau;
    p.div_max = I.div_max;
    p.gamma = I.gamma;
    p.hist_norm = I.hist;
    p.n_carried = (int)I.cnode.size();
    p.carried_node = I.cnode.data();
    p.carried_bytes = I.cbytes.data();
    p.carried_norm = I.cnorm.data();
    p.replica_mode = I.rmode;
    p.sync_mode = I.smode;
    mlf_plan_out o{};
    o.capacity = cap;
    o.order = order.data(); o.drop_reason = drop.data(); o.group = group.data(); o.group_node = gnode.data();
    o.commit_first = cf.data(); o.commit_count = cc.data(); o.commit_t_ns = ct.data(); o.punted = punted.data();
    o.replica_commit_first = rf.data(); o.replica_commit_count = rc.data(); o.replica_commit_group = rg.data();
    std::string grpname = I.name.substr(0, I.name.rfind('_'));
    if (grpname != last_group) {
      flush_group();
      last_group = grpname;
    }
    double best = 1e30;
    for (int r = 0; r < reps; ++r) {
      auto t0 = std::chrono::steady_clock::now();
      mlf_status st = mlf_plan(&net, &b, &p, &o);
      double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      best = std::min(best, ms);
      total += ms;
      if (r == reps - 1) grp.push_back(best);
      if (r) continue;
      if (st != MLF_OK) {
        if (st != I.err) {
          printf("MISMATCH %s: status %d expected %s\n", I.name.c_str(), (int)st, I.expect.empty() ? "err" : "ok");
          ++bad;
        }
        continue;
      }
      std::string got = std::to_string(o.n_commit) + "|" + L(order.data(), o.n_commit) + "|" + L8(drop.data(), I.n) +
                        "|" + L(group.data(), I.n) + "|" + std::to_string(o.n_direct) + "|" +
                        std::to_string(o.n_groups) + "|" + L(gnode.data(), o.n_groups) + "|" +
                        std::to_string(o.n_server_commits) + "|" + L(cf.data(), o.n_server_commits) + "|" +
                        L(cc.data(), o.n_server_commits) + "|" + L64(ct.data(), o.n_server_commits) + "|" +
                        std::to_string(o.replica_frozen) + "|" + std::to_string(o.replica_boundary_commit) + "|" +
                        std::to_string(o.n_punted) + "|" + L(punted.data(), o.n_punted) + "|" +
                        std::to_string((int)o.delayed_last) + "|" + std::to_string(o.t_total_ns) + "|" +
                        std::to_string(o.n_replica_commits) + "|" + L(rf.data(), o.n_replica_commits) + "|" +
                        L(rc.data(), o.n_replica_commits) + "|" + L(rg.data(), o.n_replica_commits) + "|" +
                        std::to_string(o.replica_bytes);
      if (got != I.expect) {
        printf("MISMATCH %s\n  got    %s\n  expect %s\n", I.name.c_str(), got.c_str(), I.expect.c_str());
        if (++bad > 5) return 1;
      }
    }
  }
  flush_group();
  printf("%zu instances, %d mismatches, total %.1f ms\n", all.size(), bad, total);
  return bad != 0;
}
