// commit.cu — the fused ordered-commit kernel and the aggregator tree_reduce (sm_100a).
//
// What it computes: every server commit c of the plan, in O(U)
// order, applies Eq. 2 with gamma = 0 and the north-star sign:
//     x_c = (((u_1 + u_2) + u_3) + ...)      left fold of the commit's members,
//                                             aggregators "compute the (weighted) sum"
//                                              in O(U) order
//     w   = w - (lr * x_c)                    two fp32 roundings, never an FMA (R17)
// and the replica mirror (R16) stores w at the plan's boundary commit.
//
// How (B200): the path is HBM-bound (<= 0.5 flop/byte); there is
// no contraction, so no tensor cores.  One pass: each thread owns float4 chunks
// of the shard slice, reads w once, streams every operand's chunk once
// (128-bit ld.global.cs: read-once data, evict-first), folds in registers in
// the pinned order, writes w once (and the mirror once).  Loads of up to U
// operands are issued back to back before the dependent adds (the adds keep
// their order; the loads need not), giving U+1 independent 16-byte requests in
// flight per thread.  Grid = SM count x resident blocks, grid-stride.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace mlf {

__device__ __forceinline__ float4 ld_f32x4(const float *p) { return __ldcs(reinterpret_cast<const float4 *>(p)); }

__device__ __forceinline__ float4 ld_bf16x4(const uint16_t *p) {
  const uint2 u = __ldcs(reinterpret_cast<const uint2 *>(p));
  float4 r;  // exact widening: u32 = u16 << 16 (little endian: element 0 = low half)
  r.x = __uint_as_float(u.x << 16);
  r.y = __uint_as_float(u.x & 0xffff0000u);
  r.z = __uint_as_float(u.y << 16);
  r.w = __uint_as_float(u.y & 0xffff0000u);
  return r;
}

__device__ __forceinline__ float4 load_op(const void *ptr, uint8_t flag, int64_t elem) {
  if (flag & kOpBf16) return ld_bf16x4(static_cast<const uint16_t *>(ptr) + elem);
  return ld_f32x4(static_cast<const float *>(ptr) + elem);
}

__device__ __forceinline__ float load_op1(const void *ptr, uint8_t flag, int64_t elem) {
  if (flag & kOpBf16) return __uint_as_float(uint32_t(static_cast<const uint16_t *>(ptr)[elem]) << 16);
  return static_cast<const float *>(ptr)[elem];
}

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
// w - (lr * x): product rounded, then difference rounded
__device__ __forceinline__ float4 apply4(float4 w, float lr, float4 x) {
  return make_float4(__fsub_rn(w.x, __fmul_rn(lr, x.x)), __fsub_rn(w.y, __fmul_rn(lr, x.y)),
                     __fsub_rn(w.z, __fmul_rn(lr, x.z)), __fsub_rn(w.w, __fmul_rn(lr, x.w)));
}

template <int U>
__global__ void __launch_bounds__(256) fused_commit_ldg(const __grid_constant__ CommitArgs a) {
  const int64_t nv = a.n >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride) {
    const int64_t e = v << 2;
    float4 w = __ldcs(reinterpret_cast<const float4 *>(a.w + e));
    if (a.backup_after == -1) __stcs(reinterpret_cast<float4 *>(a.backup + e), w);
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j0 = 0; j0 < a.n_ops; j0 += U) {
      float4 buf[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j0 + u < a.n_ops) buf[u] = load_op(a.op[j0 + u], a.flag[j0 + u], a.src_off + e);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + u;
        if (j < a.n_ops) {
          const uint8_t f = a.flag[j];
          x = (f & kOpFirst) ? buf[u] : add4(x, buf[u]);
          if (f & kOpLast) {
            w = apply4(w, a.lr, x);
            if (j == a.backup_after) __stcs(reinterpret_cast<float4 *>(a.backup + e), w);
          }
        }
      }
    }
    __stcs(reinterpret_cast<float4 *>(a.w + e), w);
  }
  // ragged tail (< 4 elements)
  const int64_t tail = a.n & 3;
  if (blockIdx.x == 0 && threadIdx.x < tail) {
    const int64_t e = (nv << 2) + threadIdx.x;
    float w = a.w[e];
    if (a.backup_after == -1) a.backup[e] = w;
    float x = 0.f;
    for (int j = 0; j < a.n_ops; ++j) {
      const uint8_t f = a.flag[j];
      const float u = load_op1(a.op[j], f, a.src_off + e);
      x = (f & kOpFirst) ? u : __fadd_rn(x, u);
      if (f & kOpLast) {
        w = __fsub_rn(w, __fmul_rn(a.lr, x));
        if (j == a.backup_after) a.backup[e] = w;
      }
    }
    a.w[e] = w;
  }
}

template <int U>
__global__ void __launch_bounds__(256) tree_reduce_ldg(const __grid_constant__ ReduceArgs a) {
  const int64_t nv = a.n >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride) {
    const int64_t e = v << 2;
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j0 = 0; j0 < a.n_ops; j0 += U) {
      float4 buf[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j0 + u < a.n_ops) buf[u] = load_op(a.op[j0 + u], a.flag[j0 + u], a.src_off + e);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j0 + u < a.n_ops) x = (j0 + u == 0) ? buf[u] : add4(x, buf[u]);
    }
    __stcs(reinterpret_cast<float4 *>(a.out + e), x);
  }
  const int64_t tail = a.n & 3;
  if (blockIdx.x == 0 && threadIdx.x < tail) {
    const int64_t e = (nv << 2) + threadIdx.x;
    float x = 0.f;
    for (int j = 0; j < a.n_ops; ++j) {
      const float u = load_op1(a.op[j], a.flag[j], a.src_off + e);
      x = (j == 0) ? u : __fadd_rn(x, u);
    }
    a.out[e] = x;
  }
}

static int blocks_for(const void *fn, int sm_count, int threads) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0) != cudaSuccess || per_sm < 1) per_sm = 1;
  return sm_count * per_sm;
}

cudaError_t launch_commit(const CommitArgs &a, cudaStream_t s, int sm_count, CommitImpl impl) {
  if (impl == CommitImpl::kBulk || a.n_bcast > 0) return launch_commit_bulk(a, s, sm_count);
  constexpr int kThreads = 256;
  constexpr int kU = 8;
  static int grid = 0;
  if (grid == 0) grid = blocks_for((const void *)fused_commit_ldg<kU>, sm_count, kThreads);
  int64_t need = ((a.n >> 2) + kThreads - 1) / kThreads;
  int g = (int)((need < grid) ? (need > 0 ? need : 1) : grid);
  fused_commit_ldg<kU><<<g, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_reduce(const ReduceArgs &a, cudaStream_t s, int sm_count, CommitImpl impl) {
  if (impl == CommitImpl::kBulk) return launch_reduce_bulk(a, s, sm_count);
  constexpr int kThreads = 256;
  constexpr int kU = 8;
  static int grid = 0;
  if (grid == 0) grid = blocks_for((const void *)tree_reduce_ldg<kU>, sm_count, kThreads);
  int64_t need = ((a.n >> 2) + kThreads - 1) / kThreads;
  int g = (int)((need < grid) ? (need > 0 ? need : 1) : grid);
  tree_reduce_ldg<kU><<<g, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace mlf
