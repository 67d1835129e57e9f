// kernels.h — launch interface between the executor (host C++) and the sm_100a kernels.
#pragma once
#include <atomic>
#include <cstdint>

#include <cuda_runtime_api.h>

namespace mlf {

// Operands per fused-commit launch (kernel parameter space, CUDA >= 12.1 allows
// 32 KB of parameters).  Longer commit lists are split at commit boundaries.
constexpr int kMaxOps = 1024;
constexpr int kMaxBcast = 8;

// flag bits per operand
constexpr uint8_t kOpFirst = 1;   // first member of its commit: x = u (not x += u)
constexpr uint8_t kOpLast = 2;    // last member of its commit: w <- w - lr*x after it
constexpr uint8_t kOpBf16 = 4;    // operand is bf16 (widened exactly), else fp32
// momentum only: a one-member commit whose weights are cA = cB = 1 and sh = gm (every m = 1
// commit: cA = g^0, cB = g^0, sh = gm = g).  Its two weighted sums reduce exactly to
// h' = gm*h + u, w' = w + h' (1*u == u and -0 + u == u bitwise), which the kernels evaluate
// directly: one product and two sums per element instead of five products and four sums.
constexpr uint8_t kOpSingle = 8;

// The fused reduce + scale + apply (+ mirror store) pass over one shard slice.
// Dynamic shared memory above 48 KB must be opted into per kernel and per device.  One bit
// per device records that it was; setting it twice (two threads racing) is harmless.
template <typename K>
inline cudaError_t ensure_smem(K kernel, size_t smem, std::atomic<uint64_t> &done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

struct CommitArgs {
  float *w;             // [n] shard slice, read once, written once
  float *backup;        // [n] mirror target (local or peer), or nullptr
  int64_t n;            // slice length (elements)
  int64_t src_off;      // element offset of the slice inside every operand vector
  float lr;
  int32_t n_ops;
  int32_t backup_after; // -2: no mirror store; -1: store the loaded w; k: store w after op k
  const void *op[kMaxOps];
  uint8_t flag[kMaxOps];
  // fused get (bulk kernel only): the final w of every tile is also stored to these
  // destinations (already offset to this shard; local or peer), i.e. the all-gather of the
  // new model happens tile by tile inside the commit pass
  int32_t n_bcast;
  float *bcast[kMaxBcast];
  int32_t bcast_mc;     // 1: bcast[0] is an NVLS multicast address (multimem.st, the switch replicates)
  int32_t l2_hint;      // 1: operand tiles are loaded with an L2 evict-first policy
  // dynamic tile scheduling (bulk kernel): [0] next tile, [1] CTAs done; zero between launches
  // (the last CTA resets both).  nullptr = static round-robin tiles.
  unsigned long long *sched;
  // 1 (bulk kernel, sched == nullptr): every CTA walks ONE contiguous range of n / grid elements
  // (multiples of 8) in tiles, so every CTA moves the same bytes (no last-wave tile imbalance)
  int32_t contig;
};

// tree_reduce: out[i] = left fold of members, fp32 (an aggregator's sum).
struct ReduceArgs {
  float *out;           // [n]
  int64_t n;
  int64_t src_off;
  int32_t n_ops;
  const void *op[kMaxOps];
  uint8_t flag[kMaxOps];
  unsigned long long *sched;  // dynamic tile counters (bulk reduce; as CommitArgs::sched) or nullptr
};

// Momentum commit (Eq. 2 with gamma > 0, aggregate form): per operand the weights of the two
// weighted sums, per commit (stored at its last operand) the history weights.
constexpr int kMaxOpsM = 512;
struct MomentumArgs {
  float *w, *h;              // [n] shard slice and its history, read once, written once
  float *backup, *backup_h;  // mirror targets or nullptr
  int64_t n, src_off;
  float lr;
  int32_t n_ops, backup_after;
  const void *op[kMaxOpsM];
  uint8_t flag[kMaxOpsM];
  float cA[kMaxOpsM];        // sum_{j=0..m-i} g^j   (w's weight of member i)
  float cB[kMaxOpsM];        // g^(m-i)              (h's weight of member i)
  float sh[kMaxOpsM];        // sum_{j=1..m} g^j     (at the commit's last operand)
  float gm[kMaxOpsM];        // g^m                  (at the commit's last operand)
  unsigned long long *sched; // dynamic tile counters (as CommitArgs::sched) or nullptr
};

enum class CommitImpl : int { kLdg = 0, kBulk = 1 };

cudaError_t launch_commit_momentum(const MomentumArgs &a, cudaStream_t s, int sm_count);

cudaError_t launch_commit(const CommitArgs &a, cudaStream_t s, int sm_count, CommitImpl impl);
cudaError_t launch_commit_bulk(const CommitArgs &a, cudaStream_t s, int sm_count);
// tree reduce: TMA ring (kBulk, default) or 128-bit LDG streaming (kLdg)
cudaError_t launch_reduce(const ReduceArgs &a, cudaStream_t s, int sm_count, CommitImpl impl);
cudaError_t launch_reduce_bulk(const ReduceArgs &a, cudaStream_t s, int sm_count);
cudaError_t launch_synth(void *dst, int64_t n, int64_t elem_offset, int dtype, uint64_t key, int kind,
                         int variant, cudaStream_t s);
cudaError_t launch_copy(void *dst, const void *src, int64_t bytes, cudaStream_t s, int sm_count);
cudaError_t launch_bulk_copy(void *dst, const void *src, int64_t bytes, cudaStream_t s, int sm_count);
cudaError_t launch_bulk_read(const void *src, int64_t bytes, cudaStream_t s, int sm_count);

// one launch gathering up to kMaxShards 16-byte-aligned pieces (float4 counts)
constexpr int kMaxShards = 16;
struct GatherArgs {
  int32_t n;
  int64_t total_v;                 // float4s over all pieces
  int64_t vstart[kMaxShards];      // prefix sums of the pieces' float4 counts
  float *dst[kMaxShards];
  const float *src[kMaxShards];
};
cudaError_t launch_gather(const GatherArgs &a, cudaStream_t s, int sm_count);

// TMA bulk copies of up to kMaxShards (dst, src, bytes) segments in one launch: 16 KB chunks
// global -> shared -> global, 12 in flight per SM.  Pointers and sizes 16-byte aligned.
constexpr int kBulkChunk = 16384;
struct BulkSegs {
  int32_t n;
  int64_t cstart[kMaxShards + 1];  // prefix sums of the segments' chunk counts
  char *dst[kMaxShards];
  const char *src[kMaxShards];
  int64_t bytes[kMaxShards];
};
cudaError_t launch_bulk_segs(const BulkSegs &a, cudaStream_t s, int sm_count);

// host-side splitmix64 key derivation (same definition as synthgen.stream_key)
uint64_t synth_stream_key(uint64_t seed, uint64_t kind, uint64_t a, uint64_t b);

}  // namespace mlf
