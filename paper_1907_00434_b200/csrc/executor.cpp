// executor.cpp — the C-ABI execution half of libmlfabric: context, batch
// admission (push, Table 1), plan validation, operand tables, kernel
// launches, version accounting, pull (get), peer memory.
//
// One context per process and device.  Single GPU: the whole plan runs as one
// fused commit pass (groups folded in registers).  With
// world > 1 PS shards (App. B.2) every rank runs the same plan on
// its own slice; operands are full-length update vectors on their home GPU and
// are read through NVLink peer mappings (P2P loads inside the commit kernel), or,
// in tree mode (agg_slots > 0), groups are first summed on their aggregator's
// GPU (tree_reduce) and shards read slices of the aggregate.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <deque>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.h"
#include "planner.h"

using namespace mlf;

static thread_local std::string g_err;
void mlf_set_error(const char *msg) { g_err = msg ? msg : ""; }
extern "C" const char *mlf_last_error(void) { return g_err.c_str(); }

namespace {

struct Fail {
  mlf_status code;
  std::string msg;
};

#define CK(call)                                                                                      \
  do {                                                                                                \
    cudaError_t e_ = (call);                                                                          \
    if (e_ != cudaSuccess)                                                                            \
      throw Fail{MLF_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)};                     \
  } while (0)

template <class F>
mlf_status guard(F &&f) {
  try {
    g_err.clear();
    f();
    return MLF_OK;
  } catch (const Fail &e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception &e) {
    g_err = e.what();
    return MLF_E_INVALID;
  } catch (...) {
    g_err = "unknown error";
    return MLF_E_INVALID;
  }
}

}  // namespace

static constexpr int kCopyStreams = 4;            // concurrent copy-engine streams for staging

struct mlf_ctx {
  mlf_config cfg{};
  std::vector<void *> slot;
  std::vector<int32_t> worker_rank, node_rank, worker_node;
  std::vector<float *> agg_scratch;
  std::vector<float *> bcast;                     // fused-get destinations (full-length views)
  void *pull_host = nullptr;                      // e2e pipeline: D2H target of the new shard
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;  // copy streams of the e2e pipeline
  std::vector<cudaEvent_t> pipe_ev;
  std::vector<cudaStream_t> s_copy;                // copy-engine staging streams (world > 1)
  int64_t staged = 0;                             // bytes pulled over NVLink by the copy engines
  int sm_count = 148;
  int64_t version = 0;
  size_t elem_bytes = 4;
  cudaStream_t stream = nullptr;
  // current batch
  std::vector<int32_t> b_worker, b_node;
  std::vector<int64_t> b_bytes, b_version, b_tavail;
  std::vector<double> b_norm;
  std::vector<uint8_t> in_batch, in_flight;
  std::vector<const void *> host_src;
  // execution state
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
  cudaEvent_t ev_phase = nullptr;                 // interprocess "phase 1 done" (world > 1)
  std::vector<cudaEvent_t> peer_events;           // opened peers' phase events
  // replica trees (NEXT-2): retention pool and the carried items' slots, in carried order
  std::vector<void *> retain;                     // [world * n_retain]
  std::vector<std::vector<uint8_t>> used;         // [world][n_retain]
  std::vector<std::pair<int, int>> carried;       // (rank, slot)
  std::vector<std::pair<int, int>> to_free;       // slots released at the next batch
  int64_t retained_bytes = 0;
  bool started = false, pending = false, sticky = false, phase1_done = false;
  bool dist_p1 = false;                           // distribution phase 1 recorded ev_stop
  unsigned long long *tile_sched = nullptr;       // dynamic tile counters of the bulk commit
  bool dyn_sched = false;
  bool contig = false;                            // MLF_BULK_SCHED=contig: one range per CTA
  int32_t l2_hint = 0;                            // MLF_L2_HINT=1: evict-first operand loads
  std::deque<std::pair<cudaEvent_t, std::vector<int>>> flights;   // executed batches not yet released
  std::vector<cudaEvent_t> ev_free;                                // their recycled events
  int64_t launches = 0, h2d = 0, d2h = 0;
  CommitImpl impl = CommitImpl::kLdg;
};

static void check_ctx(mlf_ctx *c) {
  if (!c) throw Fail{MLF_E_INVALID, "null context"};
  if (c->sticky) throw Fail{MLF_E_CUDA, "context has a sticky CUDA error; destroy it"};
}

extern "C" mlf_status mlf_init(const mlf_config *cfg, int64_t v0, mlf_ctx **out) {
  return guard([&] {
    if (!cfg || !out) throw Fail{MLF_E_INVALID, "null argument"};
    *out = nullptr;
    const mlf_config &k = *cfg;
    if (k.world < 1 || k.rank < 0 || k.rank >= k.world) throw Fail{MLF_E_INVALID, "rank/world"};
    if (k.model_elems < 1 || k.shard_begin < 0 || k.shard_elems < 0 || k.shard_begin + k.shard_elems > k.model_elems)
      throw Fail{MLF_E_INVALID, "model/shard extents"};
    if (k.shard_begin % 64 != 0) throw Fail{MLF_E_INVALID, "shard_begin must be a multiple of 64 elements"};
    if (k.n_workers < 0 || (k.n_workers > 0 && !k.update_slot)) throw Fail{MLF_E_INVALID, "update slots"};
    if (k.update_dtype != MLF_F32 && k.update_dtype != MLF_BF16) throw Fail{MLF_E_INVALID, "update dtype"};
    if (k.shard_elems > 0 && !k.model_shard) throw Fail{MLF_E_INVALID, "model shard"};
    if (k.agg_slots < 0 || (k.agg_slots > 0 && !k.agg_scratch)) throw Fail{MLF_E_INVALID, "aggregate scratch"};
    if (!(k.gamma >= 0.0 && k.gamma < 1.0)) throw Fail{MLF_E_INVALID, "gamma must be in [0, 1)"};
    if (k.enforce_tau != 0 && (k.enforce_tau != 1 || k.tau_max < 0)) throw Fail{MLF_E_INVALID, "enforce_tau / tau_max"};
    if (k.replica_mode != 0 && k.replica_mode != 1) throw Fail{MLF_E_INVALID, "replica_mode"};
    if (k.n_bcast < 0 || k.n_bcast > kMaxBcast || (k.n_bcast > 0 && !k.bcast))
      throw Fail{MLF_E_INVALID, "fused get: 0..8 destinations"};
    if (k.n_bcast > 0 && k.gamma != 0.0) throw Fail{MLF_E_INVALID, "fused get is implemented for gamma = 0"};
    if (k.bcast_multicast != 0 && (k.bcast_multicast != 1 || k.n_bcast != 1))
      throw Fail{MLF_E_INVALID, "bcast_multicast needs exactly one (multicast) destination"};
    for (int i = 0; i < k.n_bcast; ++i)
      if (!k.bcast[i] || (reinterpret_cast<uintptr_t>(k.bcast[i] + k.shard_begin) & 15))
        throw Fail{MLF_E_INVALID, "fused get destination null or misaligned"};
    if (k.replica_mode == 1) {
      if (k.shard_elems > 0 && !k.backup_shard) throw Fail{MLF_E_INVALID, "replica trees need the replica shard"};
      if (k.gamma != 0.0) throw Fail{MLF_E_INVALID, "replica trees are implemented for gamma = 0"};
      if (k.n_retain < 0 || (k.n_retain > 0 && !k.retain_slot)) throw Fail{MLF_E_INVALID, "retention pool"};
      for (int i = 0; i < k.world * k.n_retain; ++i)
        if (!k.retain_slot[i] || (reinterpret_cast<uintptr_t>(k.retain_slot[i]) & 15))
          throw Fail{MLF_E_INVALID, "retention slot null or not 16-byte aligned"};
    }
    if (k.gamma != 0.0) {
      if (k.shard_elems > 0 && !k.history_shard) throw Fail{MLF_E_INVALID, "momentum needs history_shard"};
      if (k.backup_shard && !k.backup_history) throw Fail{MLF_E_INVALID, "momentum mirror needs backup_history"};
      if (k.world > 1 && k.agg_slots > 0)
        throw Fail{MLF_E_INVALID, "momentum is executed in fold mode (agg_slots = 0)"};
      if ((reinterpret_cast<uintptr_t>(k.history_shard) & 15) || (reinterpret_cast<uintptr_t>(k.backup_history) & 15))
        throw Fail{MLF_E_INVALID, "history buffers not 16-byte aligned"};
    }
    if (k.stage_bytes < 0 || (k.stage_bytes > 0 && !k.stage_buf) ||
        (reinterpret_cast<uintptr_t>(k.stage_buf) & 15))
      throw Fail{MLF_E_INVALID, "staging buffer null or not 16-byte aligned"};
    if (k.n_nodes < 1) throw Fail{MLF_E_INVALID, "n_nodes < 1"};
    for (int w = 0; w < k.n_workers; ++w) {
      int nd = k.worker_node ? k.worker_node[w] : w;
      if (nd < 0 || nd >= k.n_nodes) throw Fail{MLF_E_INVALID, "worker_node out of range"};
    }
    // the kernels move 128-bit vectors: every buffer must be 16-byte aligned
    auto misaligned = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) != 0; };
    if (misaligned(k.model_shard) || misaligned(k.backup_shard))
      throw Fail{MLF_E_INVALID, "model/backup shard not 16-byte aligned"};
    for (int w = 0; w < k.n_workers; ++w)
      if (misaligned(k.update_slot[w])) throw Fail{MLF_E_INVALID, "update slot not 16-byte aligned"};
    for (int i = 0; i < k.world * k.agg_slots; ++i)
      if (!k.agg_scratch[i] || misaligned(k.agg_scratch[i]))
        throw Fail{MLF_E_INVALID, "aggregate scratch null or not 16-byte aligned"};
    auto c = new mlf_ctx();
    c->cfg = k;
    c->version = v0;
    c->elem_bytes = k.update_dtype == MLF_BF16 ? 2 : 4;
    c->stream = static_cast<cudaStream_t>(k.stream);
    for (int w = 0; w < k.n_workers; ++w) {
      if (!k.update_slot[w]) {
        delete c;
        throw Fail{MLF_E_INVALID, "null update slot"};
      }
      c->slot.push_back(k.update_slot[w]);
      int r = k.worker_rank ? k.worker_rank[w] : 0;
      if (r < 0 || r >= k.world) {
        delete c;
        throw Fail{MLF_E_INVALID, "worker_rank out of range"};
      }
      c->worker_rank.push_back(r);
      c->worker_node.push_back(k.worker_node ? k.worker_node[w] : w);
    }
    for (int i = 0; i < k.n_nodes; ++i) {
      int r = k.node_rank ? k.node_rank[i] : 0;
      if (r < 0 || r >= k.world) {
        delete c;
        throw Fail{MLF_E_INVALID, "node_rank out of range"};
      }
      c->node_rank.push_back(r);
    }
    for (int i = 0; i < k.world * k.agg_slots; ++i) c->agg_scratch.push_back(k.agg_scratch[i]);
    for (int i = 0; i < k.n_bcast; ++i) c->bcast.push_back(k.bcast[i]);
    if (k.replica_mode == 1) {
      for (int i = 0; i < k.world * k.n_retain; ++i) c->retain.push_back(k.retain_slot[i]);
      c->used.assign(k.world, std::vector<uint8_t>(k.n_retain, 0));
    }
    c->in_batch.assign(k.n_workers, 0);
    c->in_flight.assign(k.n_workers, 0);
    c->host_src.assign(k.n_workers, nullptr);
    // default kernel: TMA bulk copies through a shared-memory ring (measured best on one GPU at
    // config 2 tau 4: 99.4% vs 98.2% of the HBM copy roofline for 128-bit LDG streaming, and
    // 675 vs 634 GB/s when operands cross NVLink); MLF_COMMIT_IMPL=ldg selects the LDG kernel
    c->impl = CommitImpl::kBulk;
    const char *impl = getenv("MLF_COMMIT_IMPL");
    if (impl && std::string(impl) == "bulk") c->impl = CommitImpl::kBulk;
    if (impl && std::string(impl) == "ldg") c->impl = CommitImpl::kLdg;
    try {
      CK(cudaSetDevice(k.device));
      CK(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, k.device));
      CK(cudaEventCreate(&c->ev_start));
      CK(cudaEventCreate(&c->ev_stop));
      if (k.world > 1) CK(cudaEventCreateWithFlags(&c->ev_phase, cudaEventInterprocess | cudaEventDisableTiming));
      CK(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
      // dynamic tile scheduling for the bulk commit (MLF_BULK_SCHED=static turns it off)
      CK(cudaMalloc(reinterpret_cast<void **>(&c->tile_sched), 2 * sizeof(unsigned long long)));
      CK(cudaMemset(c->tile_sched, 0, 2 * sizeof(unsigned long long)));
      const char *sched = getenv("MLF_BULK_SCHED");
      c->dyn_sched = !(sched && (std::string(sched) == "static" || std::string(sched) == "contig"));
      c->contig = sched && std::string(sched) == "contig";
      // evict-first L2 policy for operand loads: +0.7% / +1.3% of the HBM roofline on one GPU
      // (config 2, tau 4 / 32); over NVLink it costs 4% (2 GPUs), so only local operands get it
      const char *hint = getenv("MLF_L2_HINT");
      c->l2_hint = hint ? std::string(hint) == "1" : k.world == 1;
      if (k.stage_buf && k.stage_bytes > 0 && k.world > 1)
        for (int i = 0; i < kCopyStreams; ++i) {
          cudaStream_t s;
          CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
          c->s_copy.push_back(s);
        }
    } catch (...) {
      mlf_destroy(c);                              // releases whatever was created
      throw;
    }
    *out = c;
  });
}

extern "C" void mlf_destroy(mlf_ctx *c) {
  if (!c) return;
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  if (c->ev_stop) cudaEventDestroy(c->ev_stop);
  for (auto e : c->peer_events) cudaEventDestroy(e);
  if (c->ev_phase) cudaEventDestroy(c->ev_phase);
  for (auto e : c->pipe_ev) cudaEventDestroy(e);
  if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
  if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
  for (auto &f : c->flights) cudaEventDestroy(f.first);
  for (auto e : c->ev_free) cudaEventDestroy(e);
  for (auto s : c->s_copy) cudaStreamDestroy(s);
  if (c->tile_sched) cudaFree(c->tile_sched);
  delete c;
}

// Slots are released per executed batch, oldest first, as soon as that batch's device work
// has finished: with two slot sets a producer can submit (and the pipeline stage) batch b+1
// while batch b still commits.
static void release_if_done(mlf_ctx *c) {
  while (!c->flights.empty()) {
    cudaError_t q = cudaEventQuery(c->flights.front().first);
    if (q == cudaErrorNotReady) return;
    if (q != cudaSuccess) {
      c->sticky = true;
      throw Fail{MLF_E_CUDA, std::string("cudaEventQuery: ") + cudaGetErrorString(q)};
    }
    for (int w : c->flights.front().second) c->in_flight[w] = 0;
    c->ev_free.push_back(c->flights.front().first);
    c->flights.pop_front();
  }
  if (c->pending && cudaEventQuery(c->ev_stop) == cudaSuccess) c->pending = false;
}

extern "C" mlf_status mlf_submit_update(mlf_ctx *c, int32_t worker, int64_t version, int64_t t_avail_ns, double norm,
                                        int32_t *index_in_batch) {
  return guard([&] {
    check_ctx(c);
    if (worker < 0 || worker >= c->cfg.n_workers) throw Fail{MLF_E_INVALID, "worker out of range"};
    if (t_avail_ns < 0 || !(norm >= 0)) throw Fail{MLF_E_INVALID, "t_avail / norm"};
    if (c->phase1_done) throw Fail{MLF_E_STATE, "batch is being executed (phase 1 done)"};
    if (c->in_batch[worker]) throw Fail{MLF_E_STATE, "worker already submitted in this batch"};
    release_if_done(c);
    if (c->in_flight[worker]) throw Fail{MLF_E_STATE, "worker slot still in flight (call mlf_sync)"};
    c->in_batch[worker] = 1;
    if (index_in_batch) *index_in_batch = (int32_t)c->b_worker.size();
    c->b_worker.push_back(worker);
    c->b_node.push_back(c->worker_node[worker]);
    c->b_bytes.push_back(c->cfg.model_elems * (int64_t)c->elem_bytes);
    c->b_version.push_back(version);
    c->b_tavail.push_back(t_avail_ns);
    c->b_norm.push_back(norm);
  });
}

// push for n workers in one call (include/mlfabric.h): every descriptor is checked before any
// is appended, so on error the batch is unchanged.
extern "C" mlf_status mlf_submit_batch(mlf_ctx *c, int32_t n, const int32_t *worker, const int64_t *version,
                                       const int64_t *t_avail_ns, const double *norm) {
  return guard([&] {
    check_ctx(c);
    if (n < 0 || (n > 0 && (!worker || !version))) throw Fail{MLF_E_INVALID, "n / worker / version"};
    if (c->phase1_done) throw Fail{MLF_E_STATE, "batch is being executed (phase 1 done)"};
    release_if_done(c);
    for (int32_t i = 0; i < n; ++i) {
      const int32_t w = worker[i];
      const char *why = nullptr;
      mlf_status st = MLF_E_INVALID;
      if (w < 0 || w >= c->cfg.n_workers) why = "worker out of range";
      else if ((t_avail_ns && t_avail_ns[i] < 0) || (norm && !(norm[i] >= 0))) why = "t_avail / norm";
      else if (c->in_batch[w]) st = MLF_E_STATE, why = "worker already submitted in this batch";
      else if (c->in_flight[w]) st = MLF_E_STATE, why = "worker slot still in flight (call mlf_sync)";
      if (why) {
        for (int32_t q = 0; q < i; ++q) c->in_batch[worker[q]] = 0;   // undo this call's marks
        throw Fail{st, why};
      }
      c->in_batch[w] = 2;                        // also catches a duplicate inside this call
    }
    const int64_t bytes = c->cfg.model_elems * (int64_t)c->elem_bytes;
    for (int32_t i = 0; i < n; ++i) {
      const int32_t w = worker[i];
      c->in_batch[w] = 1;
      c->b_worker.push_back(w);
      c->b_node.push_back(c->worker_node[w]);
      c->b_bytes.push_back(bytes);
      c->b_version.push_back(version[i]);
      c->b_tavail.push_back(t_avail_ns ? t_avail_ns[i] : 0);
      c->b_norm.push_back(norm ? norm[i] : 0.0);
    }
  });
}

extern "C" mlf_status mlf_set_pull_host(mlf_ctx *c, void *host_dst) {
  return guard([&] {
    check_ctx(c);
    c->pull_host = host_dst;
  });
}

extern "C" mlf_status mlf_set_update_host(mlf_ctx *c, int32_t worker, const void *host_ptr) {
  return guard([&] {
    check_ctx(c);
    if (worker < 0 || worker >= c->cfg.n_workers) throw Fail{MLF_E_INVALID, "worker out of range"};
    c->host_src[worker] = host_ptr;
  });
}

extern "C" mlf_status mlf_batch_view(mlf_ctx *c, mlf_batch *out) {
  return guard([&] {
    check_ctx(c);
    if (!out) throw Fail{MLF_E_INVALID, "null output"};
    out->n = (int32_t)c->b_worker.size();
    out->node = c->b_node.data();
    out->bytes = c->b_bytes.data();
    out->version = c->b_version.data();
    out->t_avail_ns = c->b_tavail.data();
    out->norm = c->b_norm.data();
  });
}

extern "C" mlf_status mlf_version(mlf_ctx *c, int64_t *v) {
  return guard([&] {
    check_ctx(c);
    if (!v) throw Fail{MLF_E_INVALID, "null output"};
    *v = c->version;
  });
}

// --------------------------------------------------------------- plan checks
// Structure first (every index is range-checked before it is dereferenced), then the delay
// bound the server registered (Table 1 tau_max): no device work is enqueued for a
// plan that fails either.
static void validate_plan(const mlf_ctx *c, const mlf_plan_out *p) {
  const int n = (int)c->b_worker.size();
  if (!p) throw Fail{MLF_E_INVALID, "null plan"};
  if (p->n_commit < 0 || p->n_commit > n) throw Fail{MLF_E_INVALID, "plan n_commit inconsistent with the batch"};
  if (p->n_commit > 0 && (!p->order || !p->commit_first || !p->commit_count || !p->group))
    throw Fail{MLF_E_INVALID, "plan arrays missing"};
  std::vector<uint8_t> seen(n, 0);
  for (int i = 0; i < p->n_commit; ++i) {
    int g = p->order[i];
    if (g < 0 || g >= n || seen[g]) throw Fail{MLF_E_INVALID, "plan order is not a subset of the batch"};
    seen[g] = 1;
  }
  if (p->n_server_commits < 0 || p->n_server_commits > p->n_commit)
    throw Fail{MLF_E_INVALID, "n_server_commits out of range"};
  if (p->n_groups < 0) throw Fail{MLF_E_INVALID, "n_groups < 0"};
  int pos = 0;
  for (int ci = 0; ci < p->n_server_commits; ++ci) {
    const int cnt = p->commit_count[ci];
    if (p->commit_first[ci] != pos || cnt < 1) throw Fail{MLF_E_INVALID, "commit runs not contiguous"};
    if (pos >= p->n_commit || cnt > p->n_commit - pos) throw Fail{MLF_E_INVALID, "commit runs exceed n_commit"};
    const int gid = p->group[p->order[pos]];
    for (int q = pos; q < pos + cnt; ++q)
      if (p->group[p->order[q]] != gid) throw Fail{MLF_E_INVALID, "commit mixes groups"};
    if (gid < 0 || gid > p->n_groups) throw Fail{MLF_E_INVALID, "group id out of range"};
    if (gid > 0) {
      int node = p->group_node ? p->group_node[gid - 1] : -1;
      if (node < 0 || node >= (int)c->node_rank.size()) throw Fail{MLF_E_INVALID, "aggregator node unknown to the executor"};
    }
    pos += cnt;
  }
  if (pos != p->n_commit) throw Fail{MLF_E_INVALID, "commit runs do not cover O(U)"};
  if (p->replica_boundary_commit < -1 || p->replica_boundary_commit > p->n_server_commits)
    throw Fail{MLF_E_INVALID, "replica boundary out of range"};
  if (p->replica_boundary_commit >= 0 && !c->cfg.backup_shard)
    throw Fail{MLF_E_INVALID, "plan writes the replica but the context has no backup shard"};
  if (c->cfg.replica_mode == 1) {
    // the plan must be a replica-trees plan over this context's carried items
    const int carried = (int)c->carried.size();
    if (p->n_punted < 0 || p->replica_frozen < 0 || p->replica_frozen > carried + p->n_commit)
      throw Fail{MLF_E_INVALID, "replica_frozen / n_punted out of range"};
    const int n_c = p->replica_frozen + p->n_punted - p->n_commit;
    if (p->replica_boundary_commit != -1 || n_c != carried)
      throw Fail{MLF_E_INVALID, "plan is not a replica-trees plan over the carried items"};
    if (p->n_replica_commits < 0 || p->n_replica_commits > p->replica_frozen ||
        (p->n_replica_commits > 0 && (!p->replica_commit_first || !p->replica_commit_count)))
      throw Fail{MLF_E_INVALID, "replica commits"};
    int rpos = 0;
    for (int ci = 0; ci < p->n_replica_commits; ++ci) {
      if (p->replica_commit_first[ci] != rpos || p->replica_commit_count[ci] < 1 ||
          p->replica_commit_count[ci] > p->replica_frozen - rpos)
        throw Fail{MLF_E_INVALID, "replica commit runs not contiguous"};
      rpos += p->replica_commit_count[ci];
    }
    if (rpos != p->replica_frozen) throw Fail{MLF_E_INVALID, "replica commits do not cover the frozen prefix"};
  }
  // delay bound (R1, R2): the update at 1-based position p commits as version v + p
  if (c->cfg.enforce_tau && !p->sync_mode)
    for (int i = 0; i < p->n_commit; ++i) {
      const int64_t delay = c->version + (int64_t)(i + 1) - c->b_version[p->order[i]];
      if (delay > (int64_t)c->cfg.tau_max)
        throw Fail{MLF_E_INVALID, "plan commits update " + std::to_string(p->order[i]) + " at position " +
                                      std::to_string(i + 1) + " with delay " + std::to_string(delay) +
                                      " > tau_max " + std::to_string(c->cfg.tau_max)};
    }
}

static bool tree_mode(const mlf_ctx *c) { return c->cfg.world > 1 && c->cfg.agg_slots > 0; }

// slot of group gid among the groups aggregated on the same rank
static int agg_slot_of(const mlf_ctx *c, const mlf_plan_out *p, int gid, int *rank_out) {
  int node = p->group_node[gid - 1];
  int r = c->node_rank[node], s = 0;
  for (int g = 1; g < gid; ++g)
    if (c->node_rank[p->group_node[g - 1]] == r) ++s;
  if (s >= c->cfg.agg_slots) throw Fail{MLF_E_CAPACITY, "more groups on one rank than agg_slots"};
  *rank_out = r;
  return s;
}

static void record_start(mlf_ctx *c) {
  if (!c->started) {
    CK(cudaEventRecord(c->ev_start, c->stream));
    c->started = true;
  }
}

static void reduce_local_groups(mlf_ctx *c, const mlf_plan_out *p);
static bool pipelined(const mlf_ctx *c, const mlf_plan_out *p);

static void phase_stage(mlf_ctx *c, const mlf_plan_out *p) {
  CK(cudaSetDevice(c->cfg.device));
  // two-phase multi-GPU batches: the device window starts with the batch on every rank
  if (c->cfg.world > 1) record_start(c);
  const size_t bytes = (size_t)c->cfg.model_elems * c->elem_bytes;
  // committed host-resident updates homed on this rank move host -> device;
  // dropped ones never move ("dropped at the worker itself").
  // (one GPU: the commit phase pipelines these copies chunk by chunk instead)
  for (int i = 0; i < p->n_commit && !pipelined(c, p); ++i) {
    int w = c->b_worker[p->order[i]];
    if (c->host_src[w] && c->worker_rank[w] == c->cfg.rank) {
      record_start(c);
      CK(cudaMemcpyAsync(c->slot[w], c->host_src[w], bytes, cudaMemcpyHostToDevice, c->stream));
      c->h2d += (int64_t)bytes;
    }
  }
  if (tree_mode(c)) reduce_local_groups(c, p);
  if (c->ev_phase) CK(cudaEventRecord(c->ev_phase, c->stream));
}

static void reduce_local_groups(mlf_ctx *c, const mlf_plan_out *p) {
  // tree_reduce of the groups aggregated on this rank
  for (int ci = 0; ci < p->n_server_commits; ++ci) {
    int first = p->commit_first[ci], cnt = p->commit_count[ci];
    int gid = p->group[p->order[first]];
    if (gid <= 0) continue;
    int r;
    int s = agg_slot_of(c, p, gid, &r);
    if (r != c->cfg.rank) continue;
    if (cnt > kMaxOps) throw Fail{MLF_E_CAPACITY, "group larger than kMaxOps"};
    ReduceArgs a;
    a.sched = c->dyn_sched ? c->tile_sched : nullptr;
    a.out = c->agg_scratch[(size_t)r * c->cfg.agg_slots + s];
    a.n = c->cfg.model_elems;
    a.src_off = 0;
    a.n_ops = cnt;
    for (int q = 0; q < cnt; ++q) {
      a.op[q] = c->slot[c->b_worker[p->order[first + q]]];
      a.flag[q] = c->cfg.update_dtype == MLF_BF16 ? kOpBf16 : 0;
    }
    record_start(c);
    CK(launch_reduce(a, c->stream, c->sm_count, c->impl));
    ++c->launches;
  }
}

struct CommitOp {
  const void *ptr;
  uint8_t flag;
  int commit;      // 1-based server commit index
  int home = -1;   // rank whose HBM holds the operand (-1: unknown / local)
};

// Momentum commits (NEXT-1, Eq. 2 with gamma > 0): the aggregate form's weights per member
// and per commit (the expansion of m sequential Eq. 2 steps), from
// float64 powers of the double gamma summed left to right, each rounded once to fp32 (R21).
static void launch_momentum(mlf_ctx *c, const mlf_plan_out *p, const std::vector<CommitOp> &ops, int boundary) {
  const double g = c->cfg.gamma;
  const char *se = getenv("MLF_MOM_SINGLE");            // 0: no one-member fast path (A/B experiments)
  const bool single_ok = !(se && atoi(se) == 0);
  size_t i0 = 0;
  bool first_launch = true;
  while (i0 < ops.size() || (first_launch && c->cfg.shard_elems > 0 && boundary == 0)) {
    size_t i1 = std::min(ops.size(), i0 + (size_t)kMaxOpsM);
    if (i1 < ops.size())
      while (i1 > i0 && !(ops[i1 - 1].flag & kOpLast)) --i1;
    if (i1 == i0 && i0 < ops.size()) throw Fail{MLF_E_CAPACITY, "a single commit has more than kMaxOpsM members"};
    MomentumArgs a;
    a.sched = c->dyn_sched ? c->tile_sched : nullptr;
    a.w = c->cfg.model_shard;
    a.h = c->cfg.history_shard;
    a.backup = c->cfg.backup_shard;
    a.backup_h = c->cfg.backup_history;
    a.n = c->cfg.shard_elems;
    a.src_off = c->cfg.shard_begin;
    a.lr = c->cfg.lr;
    a.n_ops = (int32_t)(i1 - i0);
    a.backup_after = (first_launch && boundary == 0) ? -1 : -2;
    size_t q = i0;
    while (q < i1) {
      const int ci = ops[q].commit;
      size_t e = q;
      while (e < i1 && ops[e].commit == ci) ++e;
      const int m = (int)(e - q);
      std::vector<double> pw(m + 1);
      pw[0] = 1.0;
      for (int j = 1; j <= m; ++j) pw[j] = pw[j - 1] * g;
      double sh = 0.0;
      for (int j = 1; j <= m; ++j) sh += pw[j];
      for (int i = 1; i <= m; ++i) {
        double ca = 0.0;
        for (int j = 0; j <= m - i; ++j) ca += pw[j];
        const size_t o = q + i - 1 - i0;
        a.op[o] = ops[q + i - 1].ptr;
        a.flag[o] = ops[q + i - 1].flag;
        a.cA[o] = (float)ca;
        a.cB[o] = (float)pw[m - i];
        a.sh[o] = (float)sh;
        a.gm[o] = (float)pw[m];
        if (single_ok && m == 1 && a.cA[o] == 1.f && a.cB[o] == 1.f && a.sh[o] == a.gm[o]) a.flag[o] |= kOpSingle;
      }
      if (boundary > 0 && ci == boundary) a.backup_after = (int32_t)(e - 1 - i0);
      q = e;
    }
    if (a.n > 0) {
      record_start(c);
      CK(launch_commit_momentum(a, c->stream, c->sm_count));
      ++c->launches;
    }
    first_launch = false;
    i0 = i1;
    if (ops.empty()) break;
  }
}

// The fused commit pass of `ops` (commit order) over w (this rank's slice, src_off =
// shard_begin), launches split at commit boundaries when the list exceeds kMaxOps.
static void launch_ops(mlf_ctx *c, float *w, float *backup, const std::vector<CommitOp> &ops, int boundary,
                       bool bcast = false, int64_t off = 0, int64_t len = -1) {
  size_t i0 = 0;
  bool first_launch = true;
  bcast = bcast && !c->bcast.empty();
  if (len < 0) len = c->cfg.shard_elems;
  while (i0 < ops.size() || (first_launch && len > 0 && (boundary == 0 || bcast))) {
    size_t i1 = std::min(ops.size(), i0 + (size_t)kMaxOps);
    if (i1 < ops.size())
      while (i1 > i0 && !(ops[i1 - 1].flag & kOpLast)) --i1;
    if (i1 == i0 && i0 < ops.size()) throw Fail{MLF_E_CAPACITY, "a single commit has more than kMaxOps members"};
    CommitArgs a;
    a.w = w + off;
    a.backup = backup ? backup + off : nullptr;
    a.n = len;
    a.src_off = c->cfg.shard_begin + off;
    a.lr = c->cfg.lr;
    a.n_ops = (int32_t)(i1 - i0);
    a.backup_after = -2;
    if (first_launch && boundary == 0) a.backup_after = -1;
    a.n_bcast = 0;
    a.bcast_mc = c->cfg.bcast_multicast;
    a.l2_hint = c->l2_hint;
    a.sched = c->dyn_sched ? c->tile_sched : nullptr;
    a.contig = c->contig ? 1 : 0;
    if (bcast && i1 == ops.size())                  // only the pass that finishes w broadcasts it
      for (float *d : c->bcast) a.bcast[a.n_bcast++] = d + c->cfg.shard_begin + off;
    for (size_t q = i0; q < i1; ++q) {
      a.op[q - i0] = ops[q].ptr;
      a.flag[q - i0] = ops[q].flag;
      if (boundary > 0 && ops[q].commit == boundary && (ops[q].flag & kOpLast)) a.backup_after = (int32_t)(q - i0);
    }
    if (a.n > 0) {
      record_start(c);   // as late as possible: the window brackets device work only
      CK(launch_commit(a, c->stream, c->sm_count, c->impl));
      ++c->launches;
    }
    first_launch = false;
    i0 = i1;
    if (ops.empty()) break;
  }
}

// End-to-end pipeline (one GPU, host-resident updates and/or a host pull target): element
// chunks flow H2D (copy stream) -> fused commit (compute stream) -> D2H (copy stream), so
// the H2D of chunk k+1, the commit of chunk k and the D2H of chunk k-1 overlap.
static constexpr int64_t kPipeChunk = 1 << 22;     // elements per chunk (16 MB of fp32)

static bool pipelined(const mlf_ctx *c, const mlf_plan_out *p) {
  if (c->cfg.world != 1 || c->cfg.gamma != 0.0 || c->cfg.replica_mode != 0 || !c->bcast.empty()) return false;
  if (c->pull_host) return true;
  for (int i = 0; i < p->n_commit; ++i)
    if (c->host_src[c->b_worker[p->order[i]]]) return true;
  return false;
}

static cudaEvent_t pipe_event(mlf_ctx *c, size_t i) {
  while (c->pipe_ev.size() <= i) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->pipe_ev.push_back(e);
  }
  return c->pipe_ev[i];
}

static void pipeline_commit(mlf_ctx *c, const mlf_plan_out *p, const std::vector<CommitOp> &ops, int boundary) {
  if (ops.size() > (size_t)kMaxOps) {              // long lists: the plain (non-overlapped) path
    for (int i = 0; i < p->n_commit; ++i) {
      const int w = c->b_worker[p->order[i]];
      if (c->host_src[w]) {
        record_start(c);
        CK(cudaMemcpyAsync(c->slot[w], c->host_src[w], (size_t)c->cfg.model_elems * c->elem_bytes,
                           cudaMemcpyHostToDevice, c->stream));
        c->h2d += (int64_t)c->cfg.model_elems * c->elem_bytes;
      }
    }
    launch_ops(c, c->cfg.model_shard, c->cfg.backup_shard, ops, boundary);
    if (c->pull_host) {
      CK(cudaMemcpyAsync(static_cast<char *>(c->pull_host) + (size_t)c->cfg.shard_begin * 4, c->cfg.model_shard,
                         (size_t)c->cfg.shard_elems * 4, cudaMemcpyDeviceToHost, c->stream));
      c->d2h += c->cfg.shard_elems * 4;
    }
    return;
  }
  record_start(c);
  size_t ev = 0;
  const cudaEvent_t begin = pipe_event(c, ev++);
  CK(cudaEventRecord(begin, c->stream));            // w is final once earlier work is done
  // no wait for the H2D: a slot is only resubmitted after the batch that last read it has
  // finished (release_if_done), so this batch's copies may overlap the previous batch's tail
  CK(cudaStreamWaitEvent(c->s_d2h, begin, 0));
  std::vector<int> host_w;
  for (int i = 0; i < p->n_commit; ++i) {
    const int w = c->b_worker[p->order[i]];
    if (c->host_src[w]) host_w.push_back(w);
  }
  const int64_t n = c->cfg.shard_elems, e = (int64_t)c->elem_bytes;
  const char *ce = getenv("MLF_PIPE_CHUNK");          // elements per chunk (tuning experiments)
  const int64_t chunk = ce && atoll(ce) >= 4096 ? atoll(ce) / 4096 * 4096 : kPipeChunk;
  for (int64_t off = 0; off < n || (off == 0 && n == 0); off += chunk) {
    const int64_t len = std::min(chunk, n - off);
    for (int w : host_w) {
      const int64_t src = c->cfg.shard_begin + off;
      CK(cudaMemcpyAsync(static_cast<char *>(c->slot[w]) + src * e, static_cast<const char *>(c->host_src[w]) + src * e,
                         (size_t)(len * e), cudaMemcpyHostToDevice, c->s_h2d));
      c->h2d += len * e;
    }
    const cudaEvent_t in = pipe_event(c, ev++);
    CK(cudaEventRecord(in, c->s_h2d));
    CK(cudaStreamWaitEvent(c->stream, in, 0));
    // the mirror-at-pre-batch store (boundary 0) belongs to every chunk, so pass it through
    launch_ops(c, c->cfg.model_shard, c->cfg.backup_shard, ops, boundary, false, off, len);
    if (c->pull_host && len > 0) {
      const cudaEvent_t done = pipe_event(c, ev++);
      CK(cudaEventRecord(done, c->stream));
      CK(cudaStreamWaitEvent(c->s_d2h, done, 0));
      CK(cudaMemcpyAsync(static_cast<char *>(c->pull_host) + (size_t)(c->cfg.shard_begin + off) * 4,
                         c->cfg.model_shard + off, (size_t)len * 4, cudaMemcpyDeviceToHost, c->s_d2h));
      c->d2h += len * 4;
    }
    if (n == 0) break;
  }
  // the batch ends when the last D2H (and every H2D) has landed
  const cudaEvent_t fin_h = pipe_event(c, ev++), fin_d = pipe_event(c, ev++);
  CK(cudaEventRecord(fin_h, c->s_h2d));
  CK(cudaEventRecord(fin_d, c->s_d2h));
  CK(cudaStreamWaitEvent(c->stream, fin_h, 0));
  CK(cudaStreamWaitEvent(c->stream, fin_d, 0));
}

// Copy-engine staging (world > 1): the operand slices homed on other GPUs are pulled over
// NVLink by the copy engines (kCopyStreams streams) into the caller's staging buffer, chunk
// by chunk and double-buffered, while the commit kernel folds the previous chunk with the
// local operands straight from HBM.  Same arithmetic and order as the peer-load path (the
// kernel sees a different pointer per operand, nothing else); only the transport differs.
// Whole-slice staging (MLF_STAGE_WHOLE=1, when the staging buffer holds every remote slice):
// each remote operand's slice of this shard is pulled by a copy engine in ONE copy, in commit
// order over the copy streams, and the fold runs in groups of consecutive commits, each waiting
// only for its own operands' copies (w is read and written once per group).  The idea: one big
// copy per direction runs at ~775 GB/s with both directions loaded where SM peer reads reach
// ~640 (scripts/nvlink_bidir_probe.py).  Measured at config 3 on 2 GPUs it is slower than the
// fold and the chunked form (2544 vs 2707 / 2599 GB/s; 14.45 ms for 1-4 streams and 4-8 groups
// alike: 32 concurrent 287 MB copies per GPU move ~650 GB/s), so it stays an option.  Same
// kernel, order and roundings as the other transports.
static constexpr int kStageGroups = 4;

static bool staged_commit_whole(mlf_ctx *c, const std::vector<CommitOp> &ops, int boundary, float *backup) {
  const int64_t e = (int64_t)c->elem_bytes, n = c->cfg.shard_elems;
  const char *sw = getenv("MLF_STAGE_WHOLE");
  if (!(sw && atoi(sw) == 1)) return false;
  const int64_t stride = (n + 4095) / 4096 * 4096;     // elements per row: 16-byte and tile aligned
  std::vector<int> row(ops.size(), -1);
  int n_remote = 0;
  for (size_t q = 0; q < ops.size(); ++q)
    if (ops[q].home >= 0 && ops[q].home != c->cfg.rank) row[q] = n_remote++;
  if (n_remote == 0 || n == 0 || n_remote * stride * e > c->cfg.stage_bytes) return false;
  const char *gs = getenv("MLF_STAGE_GROUPS"), *ss = getenv("MLF_STAGE_STREAMS");   // A/B knobs
  const int groups = gs && atoi(gs) > 0 ? atoi(gs) : kStageGroups;
  const size_t nstreams = std::min(c->s_copy.size(), (size_t)(ss && atoi(ss) > 0 ? atoi(ss) : (int)c->s_copy.size()));
  // groups of consecutive commits with about 1/groups of the remote bytes each
  std::vector<size_t> cut;                             // group g = ops[cut[g], cut[g+1])
  cut.push_back(0);
  int seen = 0;
  for (size_t q = 0; q < ops.size(); ++q) {
    if (row[q] >= 0) ++seen;
    if ((ops[q].flag & kOpLast) && q + 1 < ops.size() &&
        seen * groups >= n_remote * (int)cut.size() && (int)cut.size() < groups)
      cut.push_back(q + 1);
  }
  cut.push_back(ops.size());
  record_start(c);
  size_t ev = 0;
  const cudaEvent_t begin = pipe_event(c, ev++);
  CK(cudaEventRecord(begin, c->stream));               // peers' updates are complete (phase events)
  for (auto s : c->s_copy) CK(cudaStreamWaitEvent(s, begin, 0));
  std::vector<CommitOp> sops = ops;
  char *stage = static_cast<char *>(c->cfg.stage_buf);
  const int64_t src = c->cfg.shard_begin;
  for (size_t g = 0; g + 1 < cut.size(); ++g) {
    for (size_t q = cut[g]; q < cut[g + 1]; ++q) {
      if (row[q] < 0) continue;
      char *dst = stage + (size_t)row[q] * stride * e;
      CK(cudaMemcpyAsync(dst, static_cast<const char *>(ops[q].ptr) + src * e, (size_t)(n * e),
                         cudaMemcpyDeviceToDevice, c->s_copy[row[q] % nstreams]));
      c->staged += n * e;
      // the kernel reads op + src_off * e: shift the row pointer so that lands on the row
      sops[q].ptr = reinterpret_cast<const void *>(reinterpret_cast<uintptr_t>(dst) - (uintptr_t)(src * e));
    }
    for (size_t k = 0; k < nstreams; ++k) {
      const cudaEvent_t in = pipe_event(c, ev++);
      CK(cudaEventRecord(in, c->s_copy[k]));
      CK(cudaStreamWaitEvent(c->stream, in, 0));
    }
    const std::vector<CommitOp> part(sops.begin() + (std::ptrdiff_t)cut[g], sops.begin() + (std::ptrdiff_t)cut[g + 1]);
    // the pre-batch mirror store (boundary 0) belongs to the first pass, the fused get to the last
    const int b = boundary == 0 ? (g == 0 ? 0 : -1) : boundary;
    launch_ops(c, c->cfg.model_shard, backup, part, b, g + 2 == cut.size());
  }
  return true;
}

static void staged_commit(mlf_ctx *c, const std::vector<CommitOp> &ops, int boundary, float *backup) {
  if (staged_commit_whole(c, ops, boundary, backup)) return;
  const int64_t e = (int64_t)c->elem_bytes, n = c->cfg.shard_elems;
  // MLF_STAGE_EVERY=k (A/B knob, default 1): only every k-th remote operand is pulled by the
  // copy engines, the others stay SM peer loads in the same kernel — the two transports then
  // share the NVLink ingress
  // (MLF_STAGE_SKIP=k: the opposite split — every remote operand except every k-th is staged)
  const char *se = getenv("MLF_STAGE_EVERY"), *sk = getenv("MLF_STAGE_SKIP");
  const int every = se && atoi(se) > 0 ? atoi(se) : 1, skip = sk && atoi(sk) > 1 ? atoi(sk) : 0;
  std::vector<int> row(ops.size(), -1);
  int n_remote = 0, seen_remote = 0;
  for (size_t q = 0; q < ops.size(); ++q) {
    if (ops[q].home < 0 || ops[q].home == c->cfg.rank) continue;
    const int r = seen_remote++;
    if (skip ? r % skip != 0 : r % every == 0) row[q] = n_remote++;
  }
  constexpr int64_t kAlign = 4096;                 // elements: keeps every row 16-byte (and tile) aligned
  int64_t C = n_remote ? c->cfg.stage_bytes / (2 * n_remote * e) : 0;
  // at least 4 chunks per shard (MLF_STAGE_CHUNKS; the last chunk's fold is not overlapped);
  // larger copies run closer to the copy engine's peak (measured per-copy: 16 MiB 586, 64 MiB
  // 691, 1 GiB 732 GB/s)
  const char *sc = getenv("MLF_STAGE_CHUNKS");
  const int64_t chunks = sc && atoi(sc) > 0 ? atoi(sc) : 4;
  C = std::min(C, std::max(kAlign, ((n + chunks - 1) / chunks + kAlign - 1) / kAlign * kAlign));
  // MLF_STAGE_FIRST_DIRECT=1: the first chunk is folded with every operand read over the peer
  // mappings (nothing to wait for), while the copy engines already pull the second chunk
  const char *fd = getenv("MLF_STAGE_FIRST_DIRECT");
  const bool first_direct = fd && atoi(fd) == 1;
  C -= C % kAlign;
  if (n_remote == 0 || n == 0 || C < kAlign) {     // nothing remote, or staging too small: SM peer loads
    launch_ops(c, c->cfg.model_shard, backup, ops, boundary, true);
    return;
  }
  record_start(c);
  size_t ev = 0;
  const cudaEvent_t begin = pipe_event(c, ev++);
  CK(cudaEventRecord(begin, c->stream));           // peers' updates are complete (phase events)
  for (auto s : c->s_copy) CK(cudaStreamWaitEvent(s, begin, 0));
  std::vector<cudaEvent_t> kdone;
  std::vector<CommitOp> sops = ops;
  char *stage = static_cast<char *>(c->cfg.stage_buf);
  int k = 0;
  for (int64_t off = 0; off < n; off += C, ++k) {
    const int64_t len = std::min(C, n - off), src = c->cfg.shard_begin + off;
    if (k == 0 && first_direct) {
      launch_ops(c, c->cfg.model_shard, backup, ops, boundary, true, off, len);
      kdone.push_back(pipe_event(c, ev++));
      CK(cudaEventRecord(kdone.back(), c->stream));
      continue;
    }
    char *base = stage + (size_t)(k % 2) * n_remote * C * e;
    if (k >= 2)                                    // the buffer's previous chunk has been folded
      for (auto s : c->s_copy) CK(cudaStreamWaitEvent(s, kdone[k - 2], 0));
    for (size_t q = 0; q < ops.size(); ++q) {
      if (row[q] < 0) continue;
      char *dst = base + (size_t)row[q] * C * e;
      CK(cudaMemcpyAsync(dst, static_cast<const char *>(ops[q].ptr) + src * e, (size_t)(len * e),
                         cudaMemcpyDeviceToDevice, c->s_copy[row[q] % c->s_copy.size()]));
      c->staged += len * e;
      // the kernel reads op + src_off * e: shift the row pointer so that lands on the row
      sops[q].ptr = reinterpret_cast<const void *>(reinterpret_cast<uintptr_t>(dst) - (uintptr_t)(src * e));
    }
    for (auto s : c->s_copy) {
      const cudaEvent_t in = pipe_event(c, ev++);
      CK(cudaEventRecord(in, s));
      CK(cudaStreamWaitEvent(c->stream, in, 0));
    }
    launch_ops(c, c->cfg.model_shard, backup, sops, boundary, true, off, len);
    kdone.push_back(pipe_event(c, ev++));
    CK(cudaEventRecord(kdone.back(), c->stream));
  }
}

// Replica trees (NEXT-2): apply the frozen replica commits (the replica's own Alg. 3
// grouping over carried ++ order) to the replica shard, then retain the punted updates.
static void replicate_trees(mlf_ctx *c, const mlf_plan_out *p) {
  const int n_c = (int)c->carried.size();
  const uint8_t dflag = c->cfg.update_dtype == MLF_BF16 ? kOpBf16 : 0;
  auto item_ptr = [&](int i) -> void * {
    if (i < n_c) return c->retain[(size_t)c->carried[i].first * c->cfg.n_retain + c->carried[i].second];
    return c->slot[c->b_worker[p->order[i - n_c]]];
  };
  std::vector<CommitOp> rops;
  for (int ci = 0; ci < p->n_replica_commits; ++ci) {
    const int f = p->replica_commit_first[ci], k = p->replica_commit_count[ci];
    for (int q = 0; q < k; ++q) {
      uint8_t fl = dflag;
      if (q == 0) fl |= kOpFirst;
      if (q == k - 1) fl |= kOpLast;
      rops.push_back({item_ptr(f + q), fl, ci + 1});
    }
  }
  if (!rops.empty()) launch_ops(c, c->cfg.backup_shard, nullptr, rops, -1);
  // retention: punted items stay readable for the next batch (the worker "retains" its
  // update until the replica has it)
  const size_t bytes = (size_t)c->cfg.model_elems * c->elem_bytes;
  std::vector<std::pair<int, int>> next;
  // slots whose carried item the previous batch froze become free only now: in that batch
  // another rank's replica kernel may still have been reading them
  for (auto &rs : c->to_free) c->used[rs.first][rs.second] = 0;
  c->to_free.clear();
  for (int i = 0; i < p->replica_frozen && i < n_c; ++i) c->to_free.push_back(c->carried[i]);
  for (int i = p->replica_frozen; i < n_c + p->n_commit; ++i) {
    if (i < n_c) {
      next.push_back(c->carried[i]);
      continue;
    }
    const int w = c->b_worker[p->order[i - n_c]];
    const int r = c->worker_rank[w];
    int s = 0;
    while (s < c->cfg.n_retain && c->used[r][s]) ++s;
    if (s == c->cfg.n_retain) throw Fail{MLF_E_CAPACITY, "retention pool exhausted (punted updates)"};
    c->used[r][s] = 1;
    next.push_back({r, s});
    if (r == c->cfg.rank) {
      record_start(c);
      CK(cudaMemcpyAsync(c->retain[(size_t)r * c->cfg.n_retain + s], c->slot[w], bytes, cudaMemcpyDeviceToDevice,
                         c->stream));
      c->retained_bytes += (int64_t)bytes;
    }
  }
  c->carried.swap(next);
}

static void phase_commit(mlf_ctx *c, const mlf_plan_out *p) {
  CK(cudaSetDevice(c->cfg.device));
  // aggregates / staged updates of the other ranks are complete (phase events)
  for (auto e : c->peer_events) CK(cudaStreamWaitEvent(c->stream, e, 0));
  const bool tree = tree_mode(c);
  const uint8_t dflag = c->cfg.update_dtype == MLF_BF16 ? kOpBf16 : 0;
  // operand table in commit order
  std::vector<CommitOp> ops;
  for (int ci = 0; ci < p->n_server_commits; ++ci) {
    int first = p->commit_first[ci], cnt = p->commit_count[ci];
    int gid = p->group[p->order[first]];
    if (tree && gid > 0) {
      int r;
      int s = agg_slot_of(c, p, gid, &r);
      ops.push_back({c->agg_scratch[(size_t)r * c->cfg.agg_slots + s], (uint8_t)(kOpFirst | kOpLast), ci + 1, r});
      continue;
    }
    for (int q = 0; q < cnt; ++q) {
      uint8_t f = dflag;
      if (q == 0) f |= kOpFirst;
      if (q == cnt - 1) f |= kOpLast;
      const int w = c->b_worker[p->order[first + q]];
      ops.push_back({c->slot[w], f, ci + 1, c->worker_rank[w]});
    }
  }
  const bool trees = c->cfg.replica_mode == 1;
  const int boundary = (c->cfg.backup_shard && !trees) ? p->replica_boundary_commit : -1;
  if (c->cfg.gamma != 0.0)
    launch_momentum(c, p, ops, boundary);
  else if (pipelined(c, p))
    pipeline_commit(c, p, ops, boundary);
  else if (!c->s_copy.empty())
    staged_commit(c, ops, boundary, trees ? nullptr : c->cfg.backup_shard);
  else
    launch_ops(c, c->cfg.model_shard, trees ? nullptr : c->cfg.backup_shard, ops, boundary, true);
  if (trees) replicate_trees(c, p);
  record_start(c);
  CK(cudaEventRecord(c->ev_stop, c->stream));
  // this batch's slots are released when its own work is done (release_if_done)
  cudaEvent_t done;
  if (c->ev_free.empty()) {
    CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  } else {
    done = c->ev_free.back();
    c->ev_free.pop_back();
  }
  CK(cudaEventRecord(done, c->stream));
  c->flights.emplace_back(done, c->b_worker);
  c->started = false;
  c->pending = true;
  // version accounting (R2): every committed update advances the version
  c->version += p->sync_mode ? (p->n_commit > 0 ? 1 : 0) : p->n_commit;   // R22 / R2
  for (int w : c->b_worker) {
    c->in_flight[w] = 1;
    c->in_batch[w] = 0;
  }
  c->b_worker.clear();
  c->b_node.clear();
  c->b_bytes.clear();
  c->b_version.clear();
  c->b_tavail.clear();
  c->b_norm.clear();
  c->phase1_done = false;
}

extern "C" mlf_status mlf_execute_phase(mlf_ctx *c, const mlf_plan_out *p, int32_t phase) {
  mlf_status st = guard([&] {
    check_ctx(c);
    validate_plan(c, p);
    if ((phase & MLF_PHASE_AGGREGATE) && (phase & MLF_PHASE_COMMIT) && c->cfg.world > 1) {
      // one call for both phases gives the peers no point to order against: their phase 2
      // could read our aggregates / staged updates before they exist
      bool staged = false;
      for (int i = 0; i < p->n_commit && !staged; ++i) {
        const int w = c->b_worker[p->order[i]];
        staged = c->host_src[w] && c->worker_rank[w] == c->cfg.rank;
      }
      if (tree_mode(c) || staged)
        throw Fail{MLF_E_STATE, "tree mode / host-resident updates with world > 1 need two-phase execution "
                                "(phase 1, a barrier across ranks, phase 2)"};
    }
    if (phase & MLF_PHASE_AGGREGATE) {
      if (c->phase1_done) throw Fail{MLF_E_STATE, "phase 1 already ran for this batch"};
      phase_stage(c, p);
      c->phase1_done = true;
    }
    if (phase & MLF_PHASE_COMMIT) {
      if (!c->phase1_done) throw Fail{MLF_E_STATE, "phase 2 before phase 1"};
      phase_commit(c, p);
    }
  });
  if (st == MLF_E_CUDA && c) c->sticky = true;
  return st;
}

extern "C" mlf_status mlf_phase_event_export(mlf_ctx *c, mlf_ipc_event *out) {
  return guard([&] {
    check_ctx(c);
    if (!out) throw Fail{MLF_E_INVALID, "null output"};
    if (!c->ev_phase) throw Fail{MLF_E_STATE, "phase events exist only when world > 1"};
    cudaIpcEventHandle_t h;
    CK(cudaIpcGetEventHandle(&h, c->ev_phase));
    static_assert(sizeof(h) == 64, "ipc event handle size");
    std::memcpy(out->handle, &h, 64);
  });
}

extern "C" mlf_status mlf_phase_events_open(mlf_ctx *c, int32_t n, const mlf_ipc_event *peers) {
  return guard([&] {
    check_ctx(c);
    if (n < 0 || (n > 0 && !peers)) throw Fail{MLF_E_INVALID, "peer events"};
    CK(cudaSetDevice(c->cfg.device));
    for (auto e : c->peer_events) cudaEventDestroy(e);
    c->peer_events.clear();
    for (int i = 0; i < n; ++i) {
      cudaIpcEventHandle_t h;
      std::memcpy(&h, peers[i].handle, 64);
      cudaEvent_t e;
      CK(cudaIpcOpenEventHandle(&e, h));
      c->peer_events.push_back(e);
    }
  });
}

extern "C" mlf_status mlf_execute(mlf_ctx *c, const mlf_plan_out *p) {
  return mlf_execute_phase(c, p, MLF_PHASE_AGGREGATE | MLF_PHASE_COMMIT);
}

extern "C" mlf_status mlf_sync(mlf_ctx *c, float *device_ms) {
  mlf_status st = guard([&] {
    check_ctx(c);
    if (device_ms) *device_ms = 0.f;
    if (!c->pending) return;
    CK(cudaEventSynchronize(c->ev_stop));
    if (device_ms) CK(cudaEventElapsedTime(device_ms, c->ev_start, c->ev_stop));
    c->pending = false;
    std::fill(c->in_flight.begin(), c->in_flight.end(), 0);
    for (auto &f : c->flights) c->ev_free.push_back(f.first);   // all stream-ordered before ev_stop
    c->flights.clear();
  });
  if (st == MLF_E_CUDA && c) c->sticky = true;
  return st;
}

extern "C" mlf_status mlf_release(mlf_ctx *c, int32_t max_batches) {
  mlf_status st = guard([&] {
    check_ctx(c);
    if (max_batches < 0) throw Fail{MLF_E_INVALID, "max_batches < 0"};
    while ((int32_t)c->flights.size() > max_batches) {
      CK(cudaEventSynchronize(c->flights.front().first));
      for (int w : c->flights.front().second) c->in_flight[w] = 0;
      c->ev_free.push_back(c->flights.front().first);
      c->flights.pop_front();
    }
    release_if_done(c);
  });
  if (st == MLF_E_CUDA && c) c->sticky = true;
  return st;
}

extern "C" mlf_status mlf_pull_model(mlf_ctx *c, void *dst, int32_t dst_is_host, int64_t *version) {
  mlf_status st = guard([&] {
    check_ctx(c);
    if (!dst) throw Fail{MLF_E_INVALID, "null destination"};
    CK(cudaSetDevice(c->cfg.device));
    const size_t bytes = (size_t)c->cfg.shard_elems * 4;
    char *d = static_cast<char *>(dst) + (size_t)c->cfg.shard_begin * 4;
    if (bytes) {
      CK(cudaMemcpyAsync(d, c->cfg.model_shard, bytes, dst_is_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                         c->stream));
      if (dst_is_host) c->d2h += (int64_t)bytes;
    }
    CK(cudaStreamSynchronize(c->stream));
    if (version) *version = c->version;
  });
  if (st == MLF_E_CUDA && c) c->sticky = true;
  return st;
}

extern "C" mlf_status mlf_stats(mlf_ctx *c, int64_t *kl, int64_t *h2d, int64_t *d2h) {
  return guard([&] {
    if (!c) throw Fail{MLF_E_INVALID, "null context"};
    if (kl) *kl = c->launches;
    if (h2d) *h2d = c->h2d;
    if (d2h) *d2h = c->d2h;
  });
}

// --------------------------------------------------------------- peer memory
typedef CUresult (*PFN_range)(CUdeviceptr *, size_t *, CUdeviceptr);

static void alloc_base(const void *p, char **base) {
  static PFN_range fn = nullptr;
  if (!fn) {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess) throw Fail{MLF_E_CUDA, "cuMemGetAddressRange unavailable"};
    fn = reinterpret_cast<PFN_range>(f);
  }
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (CUdeviceptr)p) != CUDA_SUCCESS) throw Fail{MLF_E_CUDA, "cuMemGetAddressRange failed"};
  *base = reinterpret_cast<char *>(b);
}

extern "C" mlf_status mlf_ipc_export(int32_t device, const void *ptr, mlf_ipc_handle *out) {
  return guard([&] {
    if (!ptr || !out) throw Fail{MLF_E_INVALID, "null argument"};
    CK(cudaSetDevice(device));
    char *base = nullptr;
    alloc_base(ptr, &base);
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, base));
    static_assert(sizeof(h) == 64, "ipc handle size");
    std::memcpy(out->handle, &h, 64);
    out->offset = static_cast<const char *>(ptr) - base;
  });
}

extern "C" mlf_status mlf_ipc_open(int32_t device, const mlf_ipc_handle *h, void **ptr) {
  return guard([&] {
    if (!h || !ptr) throw Fail{MLF_E_INVALID, "null argument"};
    CK(cudaSetDevice(device));
    cudaIpcMemHandle_t hh;
    std::memcpy(&hh, h->handle, 64);
    void *base = nullptr;
    CK(cudaIpcOpenMemHandle(&base, hh, cudaIpcMemLazyEnablePeerAccess));
    *ptr = static_cast<char *>(base) + h->offset;
  });
}

extern "C" mlf_status mlf_ipc_close(int32_t device, void *ptr, int64_t offset) {
  return guard([&] {
    CK(cudaSetDevice(device));
    CK(cudaIpcCloseMemHandle(static_cast<char *>(ptr) - offset));
  });
}

// --------------------------------------------------------------- test infrastructure
extern "C" mlf_status mlf_synth_fill(int32_t device, void *dst, int64_t n, int64_t elem_offset, mlf_dtype dtype,
                                     uint64_t seed, int32_t kind, int64_t a, int64_t b, int32_t variant,
                                     void *stream) {
  return guard([&] {
    if (!dst && n > 0) throw Fail{MLF_E_INVALID, "null destination"};
    if (kind != 1 && kind != 2) throw Fail{MLF_E_INVALID, "kind must be 1 (update) or 2 (w0)"};
    if (variant != 0 && variant != 1) throw Fail{MLF_E_INVALID, "variant"};
    CK(cudaSetDevice(device));
    uint64_t key = synth_stream_key(seed, (uint64_t)kind, (uint64_t)a, (uint64_t)b);
    CK(launch_synth(dst, n, elem_offset, (int)dtype, key, kind, variant, static_cast<cudaStream_t>(stream)));
  });
}

extern "C" mlf_status mlf_copy_kernel(int32_t device, void *dst, const void *src, int64_t bytes, void *stream) {
  return guard([&] {
    if (bytes % 16 != 0) throw Fail{MLF_E_INVALID, "bytes % 16 != 0"};
    CK(cudaSetDevice(device));
    int sm = 148;
    CK(cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, device));
    CK(launch_copy(dst, src, bytes, static_cast<cudaStream_t>(stream), sm));
  });
}

// The whole model from its shards into dst (one gather launch over every 16-byte-aligned
// body; ragged tails and overflow shards on the copy engine).
static void gather_into(float *dst, int32_t n, const float *const *shard, const int64_t *begin, const int64_t *elems,
                        int32_t copy_engine, cudaStream_t s, int sm) {
  GatherArgs g{};
  BulkSegs t{};
  for (int i = 0; i < n; ++i) {
    if (elems[i] < 0 || begin[i] < 0 || (elems[i] > 0 && !shard[i])) throw Fail{MLF_E_INVALID, "gather shard"};
    float *d = dst + begin[i];
    const int64_t bytes = elems[i] * 4;
    const bool aligned = ((reinterpret_cast<uintptr_t>(d) | reinterpret_cast<uintptr_t>(shard[i])) & 15) == 0;
    const int used = copy_engine == 2 ? g.n : t.n;
    if (copy_engine == 1 || !aligned || used == kMaxShards) {
      if (bytes) CK(cudaMemcpyAsync(d, shard[i], (size_t)bytes, cudaMemcpyDeviceToDevice, s));
      continue;
    }
    const int64_t body = bytes & ~int64_t(15);
    if (copy_engine == 2) {
      g.vstart[g.n] = g.total_v;
      g.dst[g.n] = d;
      g.src[g.n] = shard[i];
      g.total_v += body / 16;
      ++g.n;
    } else if (body > 0) {
      t.cstart[t.n + 1] = t.cstart[t.n] + (body + kBulkChunk - 1) / kBulkChunk;
      t.dst[t.n] = reinterpret_cast<char *>(d);
      t.src[t.n] = reinterpret_cast<const char *>(shard[i]);
      t.bytes[t.n] = body;
      ++t.n;
    }
    if (bytes > body)
      CK(cudaMemcpyAsync(reinterpret_cast<char *>(d) + body, reinterpret_cast<const char *>(shard[i]) + body,
                         (size_t)(bytes - body), cudaMemcpyDeviceToDevice, s));
  }
  if (copy_engine == 2) CK(launch_gather(g, s, sm));
  else CK(launch_bulk_segs(t, s, sm));
}

extern "C" mlf_status mlf_gather(int32_t device, float *dst, int32_t n, const float *const *shard,
                                 const int64_t *begin, const int64_t *elems, int32_t copy_engine, void *stream) {
  return guard([&] {
    if (!dst || n < 0 || (n > 0 && (!shard || !begin || !elems))) throw Fail{MLF_E_INVALID, "gather arguments"};
    CK(cudaSetDevice(device));
    int sm = 148;
    CK(cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, device));
    gather_into(dst, n, shard, begin, elems, copy_engine, static_cast<cudaStream_t>(stream), sm);
  });
}

// NEXT-4: a distribution plan executed on the box (header: mlf_distribute_phase).
extern "C" mlf_status mlf_distribute_phase(mlf_ctx *c, const mlf_dist_out *p, int32_t n, const int32_t *req,
                                           float *const *view, const float *const *shard, const int64_t *begin,
                                           const int64_t *elems, int32_t phase, int32_t *source) {
  mlf_status st = guard([&] {
    check_ctx(c);
    const int world = c->cfg.world, r = c->cfg.rank;
    if (!p || n < 0 || (n > 0 && (!req || !p->order || !p->group)) || !view || !shard || !begin || !elems)
      throw Fail{MLF_E_INVALID, "distribute arguments"};
    if (p->n_groups < 0 || (p->n_groups > 0 && !p->group_node)) throw Fail{MLF_E_INVALID, "distribution groups"};
    const int nn = (int)c->node_rank.size();
    for (int i = 0; i < n; ++i)
      if (req[i] < 0 || req[i] >= nn || p->group[i] < 0 || p->group[i] > p->n_groups)
        throw Fail{MLF_E_INVALID, "request node or group out of range"};
    for (int g = 0; g < p->n_groups; ++g)
      if (p->group_node[g] < 0 || p->group_node[g] >= nn) throw Fail{MLF_E_INVALID, "distributor node unknown"};
    for (int j = 0; j < world; ++j)
      if (!view[j] || (reinterpret_cast<uintptr_t>(view[j]) & 15) || (elems[j] > 0 && !shard[j]))
        throw Fail{MLF_E_INVALID, "null or misaligned view, or null shard"};
    // this GPU's view is written once, by its earliest hop: from the servers if it hosts a
    // distributor of a non-empty group or a direct request (phase 1), else from the
    // distributor of its first request in O (phase 2)
    bool from_servers = false;
    int src = -1;
    std::vector<uint8_t> used(p->n_groups + 1, 0);
    for (int i = 0; i < n; ++i) used[p->group[i]] = 1;
    for (int g = 1; g <= p->n_groups; ++g)
      if (used[g] && c->node_rank[p->group_node[g - 1]] == r) from_servers = true;
    for (int q = 0; q < n; ++q) {
      const int i = p->order[q];
      if (i < 0 || i >= n) throw Fail{MLF_E_INVALID, "distribution order"};
      if (c->node_rank[req[i]] != r) continue;
      if (p->group[i] == 0) from_servers = true;
      else if (src < 0) src = c->node_rank[p->group_node[p->group[i] - 1]];
    }
    if (from_servers || src == r) src = -1, from_servers = true;
    if (source) *source = from_servers ? -1 : (src >= 0 ? src : -2);
    CK(cudaSetDevice(c->cfg.device));
    if (phase & MLF_PHASE_AGGREGATE) {
      record_start(c);
      if (from_servers) {
        gather_into(view[r], world, shard, begin, elems, 0, c->stream, c->sm_count);
        ++c->launches;
      }
      if (c->ev_phase) CK(cudaEventRecord(c->ev_phase, c->stream));
      // a GPU without a phase-2 hop is done here (its window must not include the host
      // barrier between the phases)
      CK(cudaEventRecord(c->ev_stop, c->stream));
      c->pending = true;
      c->dist_p1 = true;
    }
    if (phase & MLF_PHASE_COMMIT) {
      record_start(c);
      if (src >= 0) {                             // TMA bulk copy of the distributor's view
        for (auto e : c->peer_events) CK(cudaStreamWaitEvent(c->stream, e, 0));
        const int64_t bytes = c->cfg.model_elems * 4, body = bytes & ~int64_t(15);
        CK(launch_bulk_copy(view[r], view[src], body, c->stream, c->sm_count));
        ++c->launches;
        if (bytes > body)
          CK(cudaMemcpyAsync(reinterpret_cast<char *>(view[r]) + body, reinterpret_cast<const char *>(view[src]) + body,
                             (size_t)(bytes - body), cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaEventRecord(c->ev_stop, c->stream));
      } else if (!c->dist_p1) {
        CK(cudaEventRecord(c->ev_stop, c->stream));
      }
      c->dist_p1 = false;
      c->started = false;
      c->pending = true;
    }
  });
  if (st == MLF_E_CUDA && c) c->sticky = true;
  return st;
}

extern "C" mlf_status mlf_copy_bulk(int32_t device, void *dst, const void *src, int64_t bytes, void *stream) {
  return guard([&] {
    if (bytes % 16 != 0 || ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15))
      throw Fail{MLF_E_INVALID, "bulk copy needs 16-byte aligned pointers and sizes"};
    CK(cudaSetDevice(device));
    int sm = 148;
    CK(cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, device));
    CK(launch_bulk_copy(dst, src, bytes, static_cast<cudaStream_t>(stream), sm));
  });
}

extern "C" mlf_status mlf_read_probe(int32_t device, const void *src, int64_t bytes, void *stream) {
  return guard([&] {
    if (bytes % 16 != 0 || (reinterpret_cast<uintptr_t>(src) & 15))
      throw Fail{MLF_E_INVALID, "read probe needs a 16-byte aligned pointer and size"};
    CK(cudaSetDevice(device));
    int sm = 148;
    CK(cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, device));
    CK(launch_bulk_read(src, bytes, static_cast<cudaStream_t>(stream), sm));
  });
}

extern "C" mlf_status mlf_copy_engine(int32_t device, void *dst, const void *src, int64_t bytes, void *stream) {
  return guard([&] {
    if (bytes < 0 || (!dst && bytes) || (!src && bytes)) throw Fail{MLF_E_INVALID, "copy arguments"};
    CK(cudaSetDevice(device));
    CK(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
  });
}
