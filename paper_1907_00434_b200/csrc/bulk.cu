// bulk.cu — fused ordered commit with TMA bulk copies (cp.async.bulk) into a
// shared-memory ring, warp-specialised (sm_100a).
//
// Same arithmetic as fused_commit_ldg (commit.cu; Eq. 2 P:278 with
// gamma = 0, in-group left fold in O(U) order P:712-715/P:1069-1070, two fp32
// roundings per commit R17, mirror store R16), different data movement:
//   * one persistent CTA per SM; a producer warp (one elected lane) streams, for
//     every tile of kTile elements of the shard, the w tile and then each
//     operand's tile, in commit order, into a kStages-deep ring of shared-memory
//     stages with cp.async.bulk.shared::cluster.global.mbarrier::complete_tx
//     (SASS UBLKCP) — tens of KB in flight per SM independent of register
//     pressure and operand count, one instruction per 8 KB;
//   * 8 consumer warps wait on the stage's full mbarrier, fold the tile from
//     shared memory in the pinned order, release the stage (empty mbarrier),
//     and write w (and the mirror) back with 128-bit streaming stores.
// Tiles come from a global counter when a tile loads >= 64 KB (one atomic per tile, fetched a
// tile ahead, the last CTA resets the counter; the tile index rides with the first stage of
// the tile), else round-robin (tile = cta + k * grid).  A stage is refilled only after
// fence.proxy.async: its reuse is a write-after-read across proxies.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kernels.h"

namespace mlf {
namespace bulk {

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kThreads = kConsumers + 32;       // + 1 producer warp
constexpr size_t smem_bytes(int tile, int stages) {
  return (size_t)stages * tile * 4 + 3 * stages * sizeof(uint64_t);   // stages, full, empty, tile ids
}

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
// Stage reuse is a write-after-read across proxies: the consumers read a stage with generic
// loads, the producer then overwrites it with an async-proxy bulk copy.  The empty-barrier
// acquire orders the reads only for the generic proxy; fence.proxy.async extends the order to
// the bulk copy (without it, stages were measurably overwritten early under concurrent
// copy-engine traffic: scripts/dbg_concurrent.py).
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// the same copy with an L2 eviction-priority hint (operands are read exactly once)
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// fused-get store of one float4: a plain streaming store to a peer view, or one multimem
// store to an NVLS multicast address that NVSwitch replicates into every GPU's view
__device__ __forceinline__ void store_get(float *dst, float4 v, bool mc) {
  if (mc)
    asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
  else
    __stcs(reinterpret_cast<float4 *>(dst), v);
}
__device__ __forceinline__ void store_get1(float *dst, float v, bool mc) {
  if (mc)
    asm volatile("multimem.st.weak.global.f32 [%0], %1;" ::"l"(dst), "f"(v) : "memory");
  else
    *dst = v;
}

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 apply4(float4 w, float lr, float4 x) {
  return make_float4(__fsub_rn(w.x, __fmul_rn(lr, x.x)), __fsub_rn(w.y, __fmul_rn(lr, x.y)),
                     __fsub_rn(w.z, __fmul_rn(lr, x.z)), __fsub_rn(w.w, __fmul_rn(lr, x.w)));
}
__device__ __forceinline__ float4 widen_bf16x4(uint2 u) {
  return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u), __uint_as_float(u.y << 16),
                     __uint_as_float(u.y & 0xffff0000u));
}

// kTile elements per tile (one fp32 tile per stage; bf16 tiles use half), kStages-deep ring;
// kHint: operand copies carry an L2 evict-first policy (a.l2_hint), else the plain copy form
template <int kTile, int kStages, bool kHint>
__global__ void __launch_bounds__(kThreads, 1) fused_commit_bulk(const __grid_constant__ CommitArgs a) {
  constexpr int kStageBytes = kTile * 4;
  constexpr int kChunks = kTile / 4 / kConsumers;   // float4 chunks per consumer thread per tile
  static_assert(kChunks >= 1 && kTile % (4 * kConsumers) == 0, "tile must be a multiple of 4 * consumers");
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)kStages * kStageBytes);
  uint64_t *empty = full + kStages;
  int64_t *tile_of = reinterpret_cast<int64_t *>(empty + kStages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_bulk = a.n & ~int64_t(7);       // bulk region: whole 8-element groups (16 B for bf16)
  const int64_t n_tiles = (n_bulk + kTile - 1) / kTile;
  // contiguous mode: this CTA's range [r_begin, r_end); tiles are offsets into it, and the tile
  // "index" handed to the consumers is the element offset itself
  const bool contig = a.contig && !a.sched;
  const int64_t r_begin = contig ? (n_bulk / 8) * blockIdx.x / gridDim.x * 8 : 0;
  const int64_t r_end = contig ? (n_bulk / 8) * (blockIdx.x + 1) / gridDim.x * 8 : n_bulk;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ producer
    // Tiles come round-robin (static) or from a global counter (a.sched: a CTA slowed by a
    // hot peer link takes fewer tiles).  The w stage of each tile carries its index to the
    // consumers; index -1 (no stage data) ends them.
    if (lane == 0) {
      uint32_t L = 0;
      // operands are read once: evict-first under kHint.  One instruction form per
      // instantiation: a per-copy branch costs the producer, and the hinted form
      // even with the normal policy costs ~4% on peer (NVLink) reads
      const uint64_t pol_w = kHint ? policy_evict_normal() : 0;
      const uint64_t pol_op = kHint ? policy_evict_first() : 0;
      int64_t t = contig ? 0 : (a.sched ? (int64_t)atomicAdd(&a.sched[0], 1ull) : (int64_t)blockIdx.x);
      for (;;) {
        const int64_t e0 = contig ? r_begin + t * kTile : t * kTile;
        const bool live = contig ? e0 < r_end : t < n_tiles;
        const uint32_t cnt = live ? (uint32_t)(r_end - e0 < kTile ? r_end - e0 : kTile) : 0u;
        // fetch the next tile now: the atomic's latency hides behind this tile's issues
        int64_t t_next = 0;
        if (live) t_next = (a.sched && !contig) ? (int64_t)atomicAdd(&a.sched[0], 1ull) : t + (contig ? 1 : gridDim.x);
        for (int j = -1; j < a.n_ops; ++j, ++L) {
          const uint32_t s = L % kStages;
          if (L >= (uint32_t)kStages) {
            mbar_wait(&empty[s], ((L / kStages) & 1) ^ 1);
            fence_proxy_async_smem();
          }
          const void *src;
          uint32_t bytes;
          if (j < 0) {
            tile_of[s] = live ? e0 : -1;             // the consumers get the tile's element offset
            if (!live) {
              mbar_arrive(&full[s]);                  // release: the consumers read -1
              break;
            }
            src = a.w + e0;
            bytes = cnt * 4;
          } else if (a.flag[j] & kOpBf16) {
            src = static_cast<const uint16_t *>(a.op[j]) + a.src_off + e0;
            bytes = cnt * 2;
          } else {
            src = static_cast<const float *>(a.op[j]) + a.src_off + e0;
            bytes = cnt * 4;
          }
          mbar_expect_tx(&full[s], bytes);
          if constexpr (kHint)
            bulk_g2s_hint(smem + (size_t)s * kStageBytes, src, bytes, &full[s], j < 0 ? pol_w : pol_op);
          else
            bulk_g2s(smem + (size_t)s * kStageBytes, src, bytes, &full[s]);
        }
        if (!live) break;
        t = t_next;
      }
      if (a.sched && !contig) {
        // every CTA has made its last fetch: the last one resets the counters for the next
        // launch on this stream
        __threadfence();
        if (atomicAdd(&a.sched[1], 1ull) == gridDim.x - 1) {
          a.sched[0] = 0;
          a.sched[1] = 0;
          __threadfence();
        }
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    const int tid = threadIdx.x;
    uint32_t L = 0;
    for (;;) {
      const uint32_t s0 = L % kStages;
      mbar_wait(&full[s0], (L / kStages) & 1);
      const int64_t e0 = tile_of[s0];
      if (e0 < 0) break;
      const int cnt = (int)(r_end - e0 < kTile ? r_end - e0 : kTile);
      float4 w[kChunks], x[kChunks];
      {
        const uint32_t s = s0;
        const float4 *sw = reinterpret_cast<const float4 *>(smem + (size_t)s * kStageBytes);
#pragma unroll
        for (int k = 0; k < kChunks; ++k) {
          const int c = tid + k * kConsumers;
          if (c * 4 < cnt) w[k] = sw[c];
          x[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        ++L;
      }
      if (a.backup_after == -1) {
#pragma unroll
        for (int k = 0; k < kChunks; ++k) {
          const int c = tid + k * kConsumers;
          if (c * 4 < cnt) __stcs(reinterpret_cast<float4 *>(a.backup + e0) + c, w[k]);
        }
      }
      for (int j = 0; j < a.n_ops; ++j, ++L) {
        const uint32_t s = L % kStages;
        const uint8_t f = a.flag[j];
        mbar_wait(&full[s], (L / kStages) & 1);
        const uint8_t *st = smem + (size_t)s * kStageBytes;
#pragma unroll
        for (int k = 0; k < kChunks; ++k) {
          const int c = tid + k * kConsumers;
          if (c * 4 < cnt) {
            const float4 u = (f & kOpBf16) ? widen_bf16x4(reinterpret_cast<const uint2 *>(st)[c])
                                           : reinterpret_cast<const float4 *>(st)[c];
            x[k] = (f & kOpFirst) ? u : add4(x[k], u);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (f & kOpLast) {
#pragma unroll
          for (int k = 0; k < kChunks; ++k) w[k] = apply4(w[k], a.lr, x[k]);
          if (j == a.backup_after) {
#pragma unroll
            for (int k = 0; k < kChunks; ++k) {
              const int c = tid + k * kConsumers;
              if (c * 4 < cnt) __stcs(reinterpret_cast<float4 *>(a.backup + e0) + c, w[k]);
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kChunks; ++k) {
        const int c = tid + k * kConsumers;
        if (c * 4 < cnt) __stcs(reinterpret_cast<float4 *>(a.w + e0) + c, w[k]);
      }
      // fused get: the new model tile goes straight to every destination (NVLink stores)
      for (int b = 0; b < a.n_bcast; ++b) {
#pragma unroll
        for (int k = 0; k < kChunks; ++k) {
          const int c = tid + k * kConsumers;
          if (c * 4 < cnt) store_get(a.bcast[b] + e0 + 4 * c, w[k], a.bcast_mc != 0);
        }
      }
    }
    // ragged tail (< 8 elements) on CTA 0
    const int64_t tail = a.n - n_bulk;
    if (blockIdx.x == 0 && tid < tail) {
      const int64_t e = n_bulk + tid;
      float wv = a.w[e];
      if (a.backup_after == -1) a.backup[e] = wv;
      float xv = 0.f;
      for (int j = 0; j < a.n_ops; ++j) {
        const uint8_t f = a.flag[j];
        const float u = (f & kOpBf16)
                            ? __uint_as_float(uint32_t(static_cast<const uint16_t *>(a.op[j])[a.src_off + e]) << 16)
                            : static_cast<const float *>(a.op[j])[a.src_off + e];
        xv = (f & kOpFirst) ? u : __fadd_rn(xv, u);
        if (f & kOpLast) {
          wv = __fsub_rn(wv, __fmul_rn(a.lr, xv));
          if (j == a.backup_after) a.backup[e] = wv;
        }
      }
      a.w[e] = wv;
      for (int b = 0; b < a.n_bcast; ++b) store_get1(a.bcast[b] + e, wv, a.bcast_mc != 0);
    }
    if (a.bcast_mc) __threadfence_system();        // multimem stores visible system-wide at exit
  }
}

// ---------------------------------------------------------------------------------------
// Momentum (NEXT-1): Eq. 2 with gamma > 0 in its aggregate form, evaluated in the fp32 order
// DESIGN.md R21 pins (u = -(lr*g), two left folds, then w and h).  Same pipeline; each tile streams w, h and
// the operands; per commit c with members u_i = -(lr*g_i):
//   A = fold(cA_i * u_i), B = fold(cB_i * u_i), w += sh*h + A, h = gm*h + B.
__device__ __forceinline__ float4 mul4(float s, float4 x) {
  return make_float4(__fmul_rn(s, x.x), __fmul_rn(s, x.y), __fmul_rn(s, x.z), __fmul_rn(s, x.w));
}
__device__ __forceinline__ float4 neg4(float4 x) { return make_float4(-x.x, -x.y, -x.z, -x.w); }
// kBf instantiations (every operand bf16): the consumers are the limit there (16 elements per
// thread per 8 KB stage, the same work as a 16 KB fp32 stage), so their fold is branch-free.
// A commit's folds start at -0: (-0) + p == p bitwise for every p (+0 and -0 included), so
// the first member needs no select; whole tiles skip the per-chunk bounds checks.
#define kNegZero4 make_float4(-0.f, -0.f, -0.f, -0.f)
// one bf16 operand tile into A and B: u = -(lr*g), A += cA*u, B += cB*u (the pinned roundings)
// Packed fp32 pairs (sm_100a FMUL2): each lane rounds as mul.rn, so the products are bitwise
// those of the scalar op at half the instruction count.  The adds stay scalar: ptxas 12.9
// contracts mul.rn.f32x2 followed by add.rn.f32x2 into FFMA2 (one rounding), which breaks
// the pinned order; scalar add.rn is never contracted (checked in the SASS: FMUL2 + FADD)
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 x, y, z;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %5};\n\t"
      "mul.rn.f32x2 z, x, y;\n\tmov.b64 {%0, %1}, z;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
// packed sum of two fp32 pairs, each lane rounded as add.rn.  Only for sums whose operands are
// not products: ptxas contracts a mul.rn.f32x2 feeding add.rn.f32x2 into FFMA2 (R17 forbids
// fusing), but a sum of sums stays FADD2 (tests/test_sass_guard.py)
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 x, y, z;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %5};\n\t"
      "add.rn.f32x2 z, x, y;\n\tmov.b64 {%0, %1}, z;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float4 cat2(float2 lo, float2 hi) { return make_float4(lo.x, lo.y, hi.x, hi.y); }
__device__ __forceinline__ float2 lo2(float4 v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(float4 v) { return make_float2(v.z, v.w); }

template <bool kFull, int kChunks>
__device__ __forceinline__ void mom_fold_bf16(const uint8_t *st, int tid, int cnt, float lr, float ca, float cb,
                                              float4 *A, float4 *B) {
  const float2 nlr = make_float2(-lr, -lr), ca2 = make_float2(ca, ca), cb2 = make_float2(cb, cb);
#pragma unroll
  for (int k = 0; k < kChunks; ++k) {
    const int c = tid + k * kConsumers;
    if (kFull || c * 4 < cnt) {
      // u = -(lr*g) = (-lr)*g exactly (negation commutes with round-to-nearest)
      const float4 g = widen_bf16x4(reinterpret_cast<const uint2 *>(st)[c]);
      const float2 u0 = mul2(nlr, lo2(g)), u1 = mul2(nlr, hi2(g));
      A[k] = add4(A[k], cat2(mul2(ca2, u0), mul2(ca2, u1)));
      B[k] = add4(B[k], cat2(mul2(cb2, u0), mul2(cb2, u1)));
    }
  }
}

// a kOpSingle commit (see kernels.h): u = -(lr*g); h = gm*h + u; w = w + h, the same roundings
// as the weighted-sum form of a one-member commit
template <bool kFull, int kChunks, int kCons>
__device__ __forceinline__ void mom_single(const uint8_t *st, bool bf, int tid, int cnt, float lr, float gm,
                                           float4 *w, float4 *h) {
#pragma unroll
  for (int k = 0; k < kChunks; ++k) {
    const int c = tid + k * kCons;
    if (kFull || c * 4 < cnt) {
      const float4 g = bf ? widen_bf16x4(reinterpret_cast<const uint2 *>(st)[c]) : reinterpret_cast<const float4 *>(st)[c];
      const float2 nlr = make_float2(-lr, -lr), gm2 = make_float2(gm, gm);
      const float4 u = cat2(mul2(nlr, lo2(g)), mul2(nlr, hi2(g)));
      // gm*h packed too (each lane rounds as mul.rn); the adds stay scalar (no FFMA2, R17)
      h[k] = add4(cat2(mul2(gm2, lo2(h[k])), mul2(gm2, hi2(h[k]))), u);
      w[k] = cat2(add2(lo2(w[k]), lo2(h[k])), add2(hi2(w[k]), hi2(h[k])));   // w + h: no product
    }
  }
}

template <int kTile, int kStages, bool kBf>
__global__ void __launch_bounds__(kThreads, 1) fused_commit_momentum(const __grid_constant__ MomentumArgs a) {
  constexpr int kStageBytes = kTile * 4;
  constexpr int kChunks = kTile / 4 / kConsumers;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)kStages * kStageBytes);
  uint64_t *empty = full + kStages;
  int64_t *tile_of = reinterpret_cast<int64_t *>(empty + kStages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_bulk = a.n & ~int64_t(7);
  const int64_t n_tiles = (n_bulk + kTile - 1) / kTile;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kConsumerWarps) {
    if (lane == 0) {
      uint32_t L = 0;
      int64_t t = a.sched ? (int64_t)atomicAdd(&a.sched[0], 1ull) : (int64_t)blockIdx.x;
      for (;;) {
        const int64_t e0 = t * kTile;
        const uint32_t cnt = t < n_tiles ? (uint32_t)(n_bulk - e0 < kTile ? n_bulk - e0 : kTile) : 0u;
        // fetch the next tile now: the atomic's latency hides behind this tile's issues
        int64_t t_next = 0;
        if (t < n_tiles) t_next = a.sched ? (int64_t)atomicAdd(&a.sched[0], 1ull) : t + gridDim.x;
        for (int j = -2; j < a.n_ops; ++j, ++L) {
          const uint32_t s = L % kStages;
          if (L >= (uint32_t)kStages) {
            mbar_wait(&empty[s], ((L / kStages) & 1) ^ 1);
            fence_proxy_async_smem();
          }
          const void *src;
          uint32_t bytes = cnt * 4;
          if (j == -2) {
            tile_of[s] = t < n_tiles ? t : -1;       // the w stage carries the tile index
            if (t >= n_tiles) {
              mbar_arrive(&full[s]);
              break;
            }
            src = a.w + e0;
          } else if (j == -1) {
            src = a.h + e0;
          } else if (a.flag[j] & kOpBf16) {
            src = static_cast<const uint16_t *>(a.op[j]) + a.src_off + e0;
            bytes = cnt * 2;
          } else {
            src = static_cast<const float *>(a.op[j]) + a.src_off + e0;
          }
          mbar_expect_tx(&full[s], bytes);
          bulk_g2s(smem + (size_t)s * kStageBytes, src, bytes, &full[s]);
        }
        if (t >= n_tiles) break;
        t = t_next;
      }
      if (a.sched) {                                  // the last CTA resets the counters
        __threadfence();
        if (atomicAdd(&a.sched[1], 1ull) == gridDim.x - 1) {
          a.sched[0] = 0;
          a.sched[1] = 0;
          __threadfence();
        }
      }
    }
    return;
  }
  const int tid = threadIdx.x;
  uint32_t L = 0;
  for (;;) {
    mbar_wait(&full[L % kStages], (L / kStages) & 1);
    const int64_t t = tile_of[L % kStages];
    if (t < 0) break;
    const int64_t e0 = t * kTile;
    const int cnt = (int)(n_bulk - e0 < kTile ? n_bulk - e0 : kTile);
    float4 w[kChunks], h[kChunks], A[kChunks], B[kChunks];
    const bool full_tile = cnt == kTile;
    if constexpr (kBf) {
#pragma unroll
      for (int k = 0; k < kChunks; ++k) A[k] = B[k] = kNegZero4;
    }
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      const uint32_t s = L % kStages;
      mbar_wait(&full[s], (L / kStages) & 1);
      const float4 *sp = reinterpret_cast<const float4 *>(smem + (size_t)s * kStageBytes);
#pragma unroll
      for (int k = 0; k < kChunks; ++k) {
        const int c = tid + k * kConsumers;
        if (c * 4 < cnt) (which == 0 ? w[k] : h[k]) = sp[c];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      ++L;
    }
    if (a.backup_after == -1) {
#pragma unroll
      for (int k = 0; k < kChunks; ++k) {
        const int c = tid + k * kConsumers;
        if (c * 4 < cnt) {
          __stcs(reinterpret_cast<float4 *>(a.backup + e0) + c, w[k]);
          __stcs(reinterpret_cast<float4 *>(a.backup_h + e0) + c, h[k]);
        }
      }
    }
    for (int j = 0; j < a.n_ops; ++j, ++L) {
      const uint32_t s = L % kStages;
      const uint8_t f = a.flag[j];
      const float ca = a.cA[j], cb = a.cB[j];
      mbar_wait(&full[s], (L / kStages) & 1);
      const uint8_t *st = smem + (size_t)s * kStageBytes;
      // the one-member fast path only in the all-bf16 (consumer-bound) instantiation: in the
      // generic one its extra code measured 13% slower at config 2 fp32 tau 32 (profiles/r02)
      const bool single = kBf && (f & kOpSingle);
      if (single) {
        if (full_tile) mom_single<true, kChunks, kConsumers>(st, true, tid, cnt, a.lr, a.gm[j], w, h);
        else mom_single<false, kChunks, kConsumers>(st, true, tid, cnt, a.lr, a.gm[j], w, h);
      } else if constexpr (kBf) {
        if (full_tile) mom_fold_bf16<true, kChunks>(st, tid, cnt, a.lr, ca, cb, A, B);
        else mom_fold_bf16<false, kChunks>(st, tid, cnt, a.lr, ca, cb, A, B);
      } else {
#pragma unroll
        for (int k = 0; k < kChunks; ++k) {
          const int c = tid + k * kConsumers;
          if (c * 4 < cnt) {
            const float4 g = (f & kOpBf16) ? widen_bf16x4(reinterpret_cast<const uint2 *>(st)[c])
                                           : reinterpret_cast<const float4 *>(st)[c];
            const float4 u = neg4(mul4(a.lr, g));
            const float4 pa = mul4(ca, u), pb = mul4(cb, u);
            A[k] = (f & kOpFirst) ? pa : add4(A[k], pa);
            B[k] = (f & kOpFirst) ? pb : add4(B[k], pb);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if ((f & kOpLast) && !single) {
        const float sh = a.sh[j], gm = a.gm[j];
#pragma unroll
        for (int k = 0; k < kChunks; ++k) {
          w[k] = add4(w[k], add4(mul4(sh, h[k]), A[k]));
          h[k] = add4(mul4(gm, h[k]), B[k]);
          if constexpr (kBf) A[k] = B[k] = kNegZero4;  // the next commit's fold starts at -0
        }
        if constexpr (!kBf) {
          if (j == a.backup_after) {
#pragma unroll
            for (int k = 0; k < kChunks; ++k) {
              const int c = tid + k * kConsumers;
              if (c * 4 < cnt) {
                __stcs(reinterpret_cast<float4 *>(a.backup + e0) + c, w[k]);
                __stcs(reinterpret_cast<float4 *>(a.backup_h + e0) + c, h[k]);
              }
            }
          }
        }
      }
      if constexpr (kBf) {
        if (j == a.backup_after) {
#pragma unroll
          for (int k = 0; k < kChunks; ++k) {
            const int c = tid + k * kConsumers;
            if (c * 4 < cnt) {
              __stcs(reinterpret_cast<float4 *>(a.backup + e0) + c, w[k]);
              __stcs(reinterpret_cast<float4 *>(a.backup_h + e0) + c, h[k]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kChunks; ++k) {
      const int c = tid + k * kConsumers;
      if (c * 4 < cnt) {
        __stcs(reinterpret_cast<float4 *>(a.w + e0) + c, w[k]);
        __stcs(reinterpret_cast<float4 *>(a.h + e0) + c, h[k]);
      }
    }
  }
  // ragged tail (< 8 elements) on CTA 0
  const int64_t tail = a.n - n_bulk;
  if (blockIdx.x == 0 && tid < tail) {
    const int64_t e = n_bulk + tid;
    float wv = a.w[e], hv = a.h[e], Av = 0.f, Bv = 0.f;
    if (a.backup_after == -1) {
      a.backup[e] = wv;
      a.backup_h[e] = hv;
    }
    for (int j = 0; j < a.n_ops; ++j) {
      const uint8_t f = a.flag[j];
      const float g = (f & kOpBf16)
                          ? __uint_as_float(uint32_t(static_cast<const uint16_t *>(a.op[j])[a.src_off + e]) << 16)
                          : static_cast<const float *>(a.op[j])[a.src_off + e];
      const float u = -__fmul_rn(a.lr, g);
      const float pa = __fmul_rn(a.cA[j], u), pb = __fmul_rn(a.cB[j], u);
      Av = (f & kOpFirst) ? pa : __fadd_rn(Av, pa);
      Bv = (f & kOpFirst) ? pb : __fadd_rn(Bv, pb);
      if (f & kOpLast) {
        wv = __fadd_rn(wv, __fadd_rn(__fmul_rn(a.sh[j], hv), Av));
        hv = __fadd_rn(__fmul_rn(a.gm[j], hv), Bv);
        if (j == a.backup_after) {
          a.backup[e] = wv;
          a.backup_h[e] = hv;
        }
      }
    }
    a.w[e] = wv;
    a.h[e] = hv;
  }
}

// The momentum pass with static round-robin tiles and no tile-index hand-off: measured
// faster for long operand lists (config 2, tau 32: 104.5% of the HBM roofline vs 93.4% for
// the dynamic kernel above, whose longer loops cost the compute-heavier momentum consumers),
// slower for short ones (tau 4: 96.9% vs 104.3%).  launch_commit_momentum picks.
template <int kTile, int kStages, bool kBf>
__global__ void __launch_bounds__(kThreads, 1) fused_commit_momentum_rr(const __grid_constant__ MomentumArgs a) {
  constexpr int kStageBytes = kTile * 4;
  constexpr int kChunks = kTile / 4 / kConsumers;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)kStages * kStageBytes);
  uint64_t *empty = full + kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_bulk = a.n & ~int64_t(7);
  const int64_t n_tiles = (n_bulk + kTile - 1) / kTile;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kConsumerWarps) {
    if (lane == 0) {
      uint32_t L = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int64_t e0 = t * kTile;
        const uint32_t cnt = (uint32_t)(n_bulk - e0 < kTile ? n_bulk - e0 : kTile);
        for (int j = -2; j < a.n_ops; ++j, ++L) {
          const uint32_t s = L % kStages;
          if (L >= (uint32_t)kStages) {
            mbar_wait(&empty[s], ((L / kStages) & 1) ^ 1);
            fence_proxy_async_smem();
          }
          const void *src;
          uint32_t bytes = cnt * 4;
          if (j == -2) {
            src = a.w + e0;
          } else if (j == -1) {
            src = a.h + e0;
          } else if (a.flag[j] & kOpBf16) {
            src = static_cast<const uint16_t *>(a.op[j]) + a.src_off + e0;
            bytes = cnt * 2;
          } else {
            src = static_cast<const float *>(a.op[j]) + a.src_off + e0;
          }
          mbar_expect_tx(&full[s], bytes);
          bulk_g2s(smem + (size_t)s * kStageBytes, src, bytes, &full[s]);
        }
      }
    }
    return;
  }
  const int tid = threadIdx.x;
  uint32_t L = 0;
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const int64_t e0 = t * kTile;
    const int cnt = (int)(n_bulk - e0 < kTile ? n_bulk - e0 : kTile);
    float4 w[kChunks], h[kChunks], A[kChunks], B[kChunks];
    const bool full_tile = cnt == kTile;
    if constexpr (kBf) {
#pragma unroll
      for (int k = 0; k < kChunks; ++k) A[k] = B[k] = kNegZero4;
    }
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      const uint32_t s = L % kStages;
      mbar_wait(&full[s], (L / kStages) & 1);
      const float4 *sp = reinterpret_cast<const float4 *>(smem + (size_t)s * kStageBytes);
#pragma unroll
      for (int k = 0; k < kChunks; ++k) {
        const int c = tid + k * kConsumers;
        if (c * 4 < cnt) (which == 0 ? w[k] : h[k]) = sp[c];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      ++L;
    }
    if (a.backup_after == -1) {
#pragma unroll
      for (int k = 0; k < kChunks; ++k) {
        const int c = tid + k * kConsumers;
        if (c * 4 < cnt) {
          __stcs(reinterpret_cast<float4 *>(a.backup + e0) + c, w[k]);
          __stcs(reinterpret_cast<float4 *>(a.backup_h + e0) + c, h[k]);
        }
      }
    }
    for (int j = 0; j < a.n_ops; ++j, ++L) {
      const uint32_t s = L % kStages;
      const uint8_t f = a.flag[j];
      const float ca = a.cA[j], cb = a.cB[j];
      mbar_wait(&full[s], (L / kStages) & 1);
      const uint8_t *st = smem + (size_t)s * kStageBytes;
      // the one-member fast path only in the all-bf16 (consumer-bound) instantiation: in the
      // generic one its extra code measured 13% slower at config 2 fp32 tau 32 (profiles/r02)
      const bool single = kBf && (f & kOpSingle);
      if (single) {
        if (full_tile) mom_single<true, kChunks, kConsumers>(st, true, tid, cnt, a.lr, a.gm[j], w, h);
        else mom_single<false, kChunks, kConsumers>(st, true, tid, cnt, a.lr, a.gm[j], w, h);
      } else if constexpr (kBf) {
        if (full_tile) mom_fold_bf16<true, kChunks>(st, tid, cnt, a.lr, ca, cb, A, B);
        else mom_fold_bf16<false, kChunks>(st, tid, cnt, a.lr, ca, cb, A, B);
      } else {
#pragma unroll
        for (int k = 0; k < kChunks; ++k) {
          const int c = tid + k * kConsumers;
          if (c * 4 < cnt) {
            const float4 g = (f & kOpBf16) ? widen_bf16x4(reinterpret_cast<const uint2 *>(st)[c])
                                           : reinterpret_cast<const float4 *>(st)[c];
            const float4 u = neg4(mul4(a.lr, g));
            const float4 pa = mul4(ca, u), pb = mul4(cb, u);
            A[k] = (f & kOpFirst) ? pa : add4(A[k], pa);
            B[k] = (f & kOpFirst) ? pb : add4(B[k], pb);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if ((f & kOpLast) && !single) {
        const float sh = a.sh[j], gm = a.gm[j];
#pragma unroll
        for (int k = 0; k < kChunks; ++k) {
          w[k] = add4(w[k], add4(mul4(sh, h[k]), A[k]));
          h[k] = add4(mul4(gm, h[k]), B[k]);
          if constexpr (kBf) A[k] = B[k] = kNegZero4;  // the next commit's fold starts at -0
        }
        if constexpr (!kBf) {
          if (j == a.backup_after) {
#pragma unroll
            for (int k = 0; k < kChunks; ++k) {
              const int c = tid + k * kConsumers;
              if (c * 4 < cnt) {
                __stcs(reinterpret_cast<float4 *>(a.backup + e0) + c, w[k]);
                __stcs(reinterpret_cast<float4 *>(a.backup_h + e0) + c, h[k]);
              }
            }
          }
        }
      }
      if constexpr (kBf) {
        if (j == a.backup_after) {
#pragma unroll
          for (int k = 0; k < kChunks; ++k) {
            const int c = tid + k * kConsumers;
            if (c * 4 < cnt) {
              __stcs(reinterpret_cast<float4 *>(a.backup + e0) + c, w[k]);
              __stcs(reinterpret_cast<float4 *>(a.backup_h + e0) + c, h[k]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kChunks; ++k) {
      const int c = tid + k * kConsumers;
      if (c * 4 < cnt) {
        __stcs(reinterpret_cast<float4 *>(a.w + e0) + c, w[k]);
        __stcs(reinterpret_cast<float4 *>(a.h + e0) + c, h[k]);
      }
    }
  }
  // ragged tail (< 8 elements) on CTA 0
  const int64_t tail = a.n - n_bulk;
  if (blockIdx.x == 0 && tid < tail) {
    const int64_t e = n_bulk + tid;
    float wv = a.w[e], hv = a.h[e], Av = 0.f, Bv = 0.f;
    if (a.backup_after == -1) {
      a.backup[e] = wv;
      a.backup_h[e] = hv;
    }
    for (int j = 0; j < a.n_ops; ++j) {
      const uint8_t f = a.flag[j];
      const float g = (f & kOpBf16)
                          ? __uint_as_float(uint32_t(static_cast<const uint16_t *>(a.op[j])[a.src_off + e]) << 16)
                          : static_cast<const float *>(a.op[j])[a.src_off + e];
      const float u = -__fmul_rn(a.lr, g);
      const float pa = __fmul_rn(a.cA[j], u), pb = __fmul_rn(a.cB[j], u);
      Av = (f & kOpFirst) ? pa : __fadd_rn(Av, pa);
      Bv = (f & kOpFirst) ? pb : __fadd_rn(Bv, pb);
      if (f & kOpLast) {
        wv = __fadd_rn(wv, __fadd_rn(__fmul_rn(a.sh[j], hv), Av));
        hv = __fadd_rn(__fmul_rn(a.gm[j], hv), Bv);
        if (j == a.backup_after) {
          a.backup[e] = wv;
          a.backup_h[e] = hv;
        }
      }
    }
    a.w[e] = wv;
    a.h[e] = hv;
  }
}

// ---------------------------------------------------------------------------------------
// bf16 momentum, wide: the all-bf16 momentum pass with kCW consumer warps (16: twice the
// warps of the kernels above) and 16 KB bf16 stages.  ncu on fused_commit_momentum_rr<4096,12,
// true> (config 2 bf16, gamma 0.9, tau 32; profiles/r02) shows the consumers latency-bound: 2.25
// warps per scheduler, 0.82 eligible, issue slots 57% busy, DRAM 63%.  Here a tile is kTile =
// 8192 elements: each bf16 operand tile fills one 16 KB stage (all 12 stages carry 16 KB), the
// fp32 w and h tiles span two stages each, and every consumer thread still folds 16 elements
// per stage (kTile / kCW / 32), so the per-stage hand-off cost per element is unchanged while
// the warps available to hide latency double.  Each CTA owns one contiguous range of
// n / grid elements (multiples of 8) walked in tiles, so every CTA moves the same bytes (no
// last-wave imbalance of round-robin 8192-element tiles: 3125 tiles over 148 CTAs = 21.1).
// Same arithmetic, order and roundings as fused_commit_momentum_rr<., ., true>.
template <bool kFull, int kChunks, int kCons>
__device__ __forceinline__ void mom_fold_bf16_w(const uint8_t *st, int tid, int cnt, float lr, float ca, float cb,
                                                float4 *A, float4 *B) {
  const float2 nlr = make_float2(-lr, -lr), ca2 = make_float2(ca, ca), cb2 = make_float2(cb, cb);
#pragma unroll
  for (int k = 0; k < kChunks; ++k) {
    const int c = tid + k * kCons;
    if (kFull || c * 4 < cnt) {
      const float4 g = widen_bf16x4(reinterpret_cast<const uint2 *>(st)[c]);
      const float2 u0 = mul2(nlr, lo2(g)), u1 = mul2(nlr, hi2(g));
      A[k] = add4(A[k], cat2(mul2(ca2, u0), mul2(ca2, u1)));
      B[k] = add4(B[k], cat2(mul2(cb2, u0), mul2(cb2, u1)));
    }
  }
}

template <int kTile, int kStages, int kCW>
__global__ void __launch_bounds__(kCW * 32 + 32, kCW <= 8 ? 2 : 1) fused_commit_momentum_bh(const __grid_constant__ MomentumArgs a) {
  constexpr int kCons = kCW * 32;
  constexpr int kStageBytes = kTile * 2;            // one bf16 operand tile
  constexpr int kHalf = kTile / 2;                  // fp32 elements per stage
  constexpr int kChunks = kTile / 4 / kCons;        // float4 chunks per consumer thread per tile
  constexpr int kHalfChunks = kChunks / 2;          // ... of them in the first fp32 half-stage
  static_assert(kChunks % 2 == 0 && kTile % (8 * kCons) == 0, "tile must split evenly");
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)kStages * kStageBytes);
  uint64_t *empty = full + kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_bulk = a.n & ~int64_t(7);
  const int64_t n8 = n_bulk / 8;
  const int64_t r_begin = n8 * blockIdx.x / gridDim.x * 8, r_end = n8 * (blockIdx.x + 1) / gridDim.x * 8;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kCW) {
    if (lane == 0) {
      uint32_t L = 0;
      for (int64_t e0 = r_begin; e0 < r_end; e0 += kTile) {
        const uint32_t cnt = (uint32_t)(r_end - e0 < kTile ? r_end - e0 : kTile);
        for (int j = -4; j < a.n_ops; ++j, ++L) {   // -4, -3: the halves of w; -2, -1: of h
          const uint32_t s = L % kStages;
          if (L >= (uint32_t)kStages) {
            mbar_wait(&empty[s], ((L / kStages) & 1) ^ 1);
            fence_proxy_async_smem();
          }
          const void *src;
          uint32_t bytes;
          if (j < 0) {
            const uint32_t h0 = (j & 1) ? (uint32_t)kHalf : 0u;        // -3, -1: second half
            const uint32_t h = cnt > h0 ? (cnt - h0 < (uint32_t)kHalf ? cnt - h0 : (uint32_t)kHalf) : 0u;
            src = (j < -2 ? a.w : a.h) + e0 + h0;
            bytes = h * 4;
          } else {
            src = static_cast<const uint16_t *>(a.op[j]) + a.src_off + e0;
            bytes = cnt * 2;
          }
          mbar_expect_tx(&full[s], bytes);
          if (bytes) bulk_g2s(smem + (size_t)s * kStageBytes, src, bytes, &full[s]);
        }
      }
    }
    return;
  }
  const int tid = threadIdx.x;
  // ring position kept incrementally (stage index and phase parity), no division per stage
  uint32_t s = 0, ph = 0;
  auto advance = [&]() {
    if (++s == (uint32_t)kStages) {
      s = 0;
      ph ^= 1u;
    }
  };
  for (int64_t e0 = r_begin; e0 < r_end; e0 += kTile) {
    const int cnt = (int)(r_end - e0 < kTile ? r_end - e0 : kTile);
    const bool full_tile = cnt == kTile;
    float4 w[kChunks], h[kChunks], A[kChunks], B[kChunks];
#pragma unroll
    for (int k = 0; k < kChunks; ++k) A[k] = B[k] = kNegZero4;
    // w and h: two half-stages each; chunk k lives in the first half iff k < kHalfChunks
#pragma unroll
    for (int which = 0; which < 4; ++which) {
      mbar_wait(&full[s], ph);
      const float4 *sp = reinterpret_cast<const float4 *>(smem + (size_t)s * kStageBytes);
      const int k0 = (which & 1) ? kHalfChunks : 0;
#pragma unroll
      for (int kk = 0; kk < kHalfChunks; ++kk) {
        const int k = k0 + kk;
        const int c = tid + k * kCons;
        if (c * 4 < cnt) (which < 2 ? w[k] : h[k]) = sp[c - ((which & 1) ? kHalf / 4 : 0)];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      advance();
    }
    if (a.backup_after == -1) {
#pragma unroll
      for (int k = 0; k < kChunks; ++k) {
        const int c = tid + k * kCons;
        if (c * 4 < cnt) {
          __stcs(reinterpret_cast<float4 *>(a.backup + e0) + c, w[k]);
          __stcs(reinterpret_cast<float4 *>(a.backup_h + e0) + c, h[k]);
        }
      }
    }
    for (int j = 0; j < a.n_ops; ++j) {
      const uint8_t f = a.flag[j];
      mbar_wait(&full[s], ph);
      const uint8_t *st = smem + (size_t)s * kStageBytes;
      const bool single = f & kOpSingle;
      if (single) {
        if (full_tile) mom_single<true, kChunks, kCons>(st, true, tid, cnt, a.lr, a.gm[j], w, h);
        else mom_single<false, kChunks, kCons>(st, true, tid, cnt, a.lr, a.gm[j], w, h);
      } else if (full_tile) {
        mom_fold_bf16_w<true, kChunks, kCons>(st, tid, cnt, a.lr, a.cA[j], a.cB[j], A, B);
      } else {
        mom_fold_bf16_w<false, kChunks, kCons>(st, tid, cnt, a.lr, a.cA[j], a.cB[j], A, B);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      advance();
      if ((f & kOpLast) && !single) {
        const float sh = a.sh[j], gm = a.gm[j];
#pragma unroll
        for (int k = 0; k < kChunks; ++k) {
          w[k] = add4(w[k], add4(mul4(sh, h[k]), A[k]));
          h[k] = add4(mul4(gm, h[k]), B[k]);
          A[k] = B[k] = kNegZero4;                    // the next commit's fold starts at -0
        }
      }
      if (j == a.backup_after) {
#pragma unroll
        for (int k = 0; k < kChunks; ++k) {
          const int c = tid + k * kCons;
          if (c * 4 < cnt) {
            __stcs(reinterpret_cast<float4 *>(a.backup + e0) + c, w[k]);
            __stcs(reinterpret_cast<float4 *>(a.backup_h + e0) + c, h[k]);
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kChunks; ++k) {
      const int c = tid + k * kCons;
      if (c * 4 < cnt) {
        __stcs(reinterpret_cast<float4 *>(a.w + e0) + c, w[k]);
        __stcs(reinterpret_cast<float4 *>(a.h + e0) + c, h[k]);
      }
    }
  }
  // ragged tail (< 8 elements) on CTA 0
  const int64_t tail = a.n - n_bulk;
  if (blockIdx.x == 0 && tid < tail) {
    const int64_t e = n_bulk + tid;
    float wv = a.w[e], hv = a.h[e], Av = 0.f, Bv = 0.f;
    if (a.backup_after == -1) {
      a.backup[e] = wv;
      a.backup_h[e] = hv;
    }
    for (int j = 0; j < a.n_ops; ++j) {
      const uint8_t f = a.flag[j];
      const float g = __uint_as_float(uint32_t(static_cast<const uint16_t *>(a.op[j])[a.src_off + e]) << 16);
      const float u = -__fmul_rn(a.lr, g);
      const float pa = __fmul_rn(a.cA[j], u), pb = __fmul_rn(a.cB[j], u);
      Av = (f & kOpFirst) ? pa : __fadd_rn(Av, pa);
      Bv = (f & kOpFirst) ? pb : __fadd_rn(Bv, pb);
      if (f & kOpLast) {
        wv = __fadd_rn(wv, __fadd_rn(__fmul_rn(a.sh[j], hv), Av));
        hv = __fadd_rn(__fmul_rn(a.gm[j], hv), Bv);
        if (j == a.backup_after) {
          a.backup[e] = wv;
          a.backup_h[e] = hv;
        }
      }
    }
    a.w[e] = wv;
    a.h[e] = hv;
  }
}

// ---------------------------------------------------------------------------------------
// The same commit for bf16 operands with 16 KB bulk copies: a tile is kTile = 8192
// elements, so every bf16 operand tile fills one 16 KB stage and the fp32 w tile spans two.
// With the fp32 layout (4096-element tiles) bf16 copies are 8 KB and the per-stage hand-off
// costs show (config 2, tau 32: 86% of the HBM roofline).  Same fold order and roundings.
template <int kTile, int kStages>
__global__ void __launch_bounds__(kThreads, 1) fused_commit_bulk_h(const __grid_constant__ CommitArgs a) {
  constexpr int kStageBytes = kTile * 2;
  constexpr int kHalf = kTile / 2;                  // fp32 elements per stage
  constexpr int kChunks = kTile / 4 / kConsumers;   // float4 chunks per consumer thread per tile
  static_assert(kChunks % 2 == 0 && kTile % (8 * kConsumers) == 0, "tile must split evenly");
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)kStages * kStageBytes);
  uint64_t *empty = full + kStages;
  int64_t *tile_of = reinterpret_cast<int64_t *>(empty + kStages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_bulk = a.n & ~int64_t(7);
  const int64_t n_tiles = (n_bulk + kTile - 1) / kTile;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    if (lane == 0) {
      uint32_t L = 0;
      int64_t t = a.sched ? (int64_t)atomicAdd(&a.sched[0], 1ull) : (int64_t)blockIdx.x;
      for (;;) {
        const int64_t e0 = t * kTile;
        const uint32_t cnt = t < n_tiles ? (uint32_t)(n_bulk - e0 < kTile ? n_bulk - e0 : kTile) : 0u;
        // fetch the next tile now: the atomic's latency hides behind this tile's issues
        int64_t t_next = 0;
        if (t < n_tiles) t_next = a.sched ? (int64_t)atomicAdd(&a.sched[0], 1ull) : t + gridDim.x;
        for (int j = -2; j < a.n_ops; ++j, ++L) {       // j = -2, -1: the two halves of w
          const uint32_t s = L % kStages;
          if (L >= (uint32_t)kStages) {
            mbar_wait(&empty[s], ((L / kStages) & 1) ^ 1);
            fence_proxy_async_smem();
          }
          if (j == -2) {
            tile_of[s] = t < n_tiles ? t : -1;       // the first w stage carries the tile index
            if (t >= n_tiles) {
              mbar_arrive(&full[s]);
              break;
            }
          }
          const void *src;
          uint32_t bytes;
          if (j < 0) {
            const uint32_t h0 = j == -2 ? 0u : (uint32_t)kHalf;
            const uint32_t h = cnt > h0 ? (cnt - h0 < (uint32_t)kHalf ? cnt - h0 : (uint32_t)kHalf) : 0u;
            src = a.w + e0 + h0;
            bytes = h * 4;
          } else {
            src = static_cast<const uint16_t *>(a.op[j]) + a.src_off + e0;
            bytes = cnt * 2;
          }
          mbar_expect_tx(&full[s], bytes);
          if (bytes) bulk_g2s(smem + (size_t)s * kStageBytes, src, bytes, &full[s]);
        }
        if (t >= n_tiles) break;
        t = t_next;
      }
      if (a.sched) {                                  // the last CTA resets the counters
        __threadfence();
        if (atomicAdd(&a.sched[1], 1ull) == gridDim.x - 1) {
          a.sched[0] = 0;
          a.sched[1] = 0;
          __threadfence();
        }
      }
    }
  } else {
    const int tid = threadIdx.x;
    uint32_t L = 0;
    for (;;) {
      mbar_wait(&full[L % kStages], (L / kStages) & 1);
      const int64_t t = tile_of[L % kStages];
      if (t < 0) break;
      const int64_t e0 = t * kTile;
      const int cnt = (int)(n_bulk - e0 < kTile ? n_bulk - e0 : kTile);
      float4 w[kChunks], x[kChunks];
      for (int half = 0; half < 2; ++half, ++L) {       // chunks [half*kChunks/2, ...) of w
        const uint32_t s = L % kStages;
        mbar_wait(&full[s], (L / kStages) & 1);
        const float4 *sw = reinterpret_cast<const float4 *>(smem + (size_t)s * kStageBytes);
#pragma unroll
        for (int k = 0; k < kChunks / 2; ++k) {
          const int kk = half * (kChunks / 2) + k;
          const int c = tid + kk * kConsumers;
          if (c * 4 < cnt) w[kk] = sw[c - half * (kHalf / 4)];
          x[kk] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      if (a.backup_after == -1) {
#pragma unroll
        for (int k = 0; k < kChunks; ++k) {
          const int c = tid + k * kConsumers;
          if (c * 4 < cnt) __stcs(reinterpret_cast<float4 *>(a.backup + e0) + c, w[k]);
        }
      }
      for (int j = 0; j < a.n_ops; ++j, ++L) {
        const uint32_t s = L % kStages;
        const uint8_t f = a.flag[j];
        mbar_wait(&full[s], (L / kStages) & 1);
        const uint2 *st = reinterpret_cast<const uint2 *>(smem + (size_t)s * kStageBytes);
#pragma unroll
        for (int k = 0; k < kChunks; ++k) {
          const int c = tid + k * kConsumers;
          if (c * 4 < cnt) {
            const float4 u = widen_bf16x4(st[c]);
            x[k] = (f & kOpFirst) ? u : add4(x[k], u);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (f & kOpLast) {
#pragma unroll
          for (int k = 0; k < kChunks; ++k) w[k] = apply4(w[k], a.lr, x[k]);
          if (j == a.backup_after) {
#pragma unroll
            for (int k = 0; k < kChunks; ++k) {
              const int c = tid + k * kConsumers;
              if (c * 4 < cnt) __stcs(reinterpret_cast<float4 *>(a.backup + e0) + c, w[k]);
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kChunks; ++k) {
        const int c = tid + k * kConsumers;
        if (c * 4 < cnt) __stcs(reinterpret_cast<float4 *>(a.w + e0) + c, w[k]);
      }
      for (int b = 0; b < a.n_bcast; ++b) {
#pragma unroll
        for (int k = 0; k < kChunks; ++k) {
          const int c = tid + k * kConsumers;
          if (c * 4 < cnt) store_get(a.bcast[b] + e0 + 4 * c, w[k], a.bcast_mc != 0);
        }
      }
    }
    const int64_t tail = a.n - n_bulk;                // ragged tail (< 8 elements) on CTA 0
    if (blockIdx.x == 0 && tid < tail) {
      const int64_t e = n_bulk + tid;
      float wv = a.w[e];
      if (a.backup_after == -1) a.backup[e] = wv;
      float xv = 0.f;
      for (int j = 0; j < a.n_ops; ++j) {
        const uint8_t f = a.flag[j];
        const float u = __uint_as_float(uint32_t(static_cast<const uint16_t *>(a.op[j])[a.src_off + e]) << 16);
        xv = (f & kOpFirst) ? u : __fadd_rn(xv, u);
        if (f & kOpLast) {
          wv = __fsub_rn(wv, __fmul_rn(a.lr, xv));
          if (j == a.backup_after) a.backup[e] = wv;
        }
      }
      a.w[e] = wv;
      for (int b = 0; b < a.n_bcast; ++b) store_get1(a.bcast[b] + e, wv, a.bcast_mc != 0);
    }
    if (a.bcast_mc) __threadfence_system();        // multimem stores visible system-wide at exit
  }
}

// ---------------------------------------------------------------------------------------
// Tree reduce: the fp32 aggregate of a group on its
// aggregator's GPU, acc = ((x1 + x2) + x3) + ... in O(U) order, bf16 widened exactly.
// The same TMA ring as the commit, without w: the producer streams every member's tile,
// the consumers fold it from shared memory and store the aggregate tile.
template <int kTile, int kStages>
__global__ void __launch_bounds__(kThreads, 1) tree_reduce_bulk(const __grid_constant__ ReduceArgs a) {
  constexpr int kStageBytes = kTile * 4;
  constexpr int kChunks = kTile / 4 / kConsumers;
  static_assert(kChunks >= 1 && kTile % (4 * kConsumers) == 0, "tile must be a multiple of 4 * consumers");
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)kStages * kStageBytes);
  uint64_t *empty = full + kStages;
  int64_t *tile_of = reinterpret_cast<int64_t *>(empty + kStages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_bulk = a.n & ~int64_t(7);
  const int64_t n_tiles = (n_bulk + kTile - 1) / kTile;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    if (lane == 0) {
      uint32_t L = 0;
      int64_t t = a.sched ? (int64_t)atomicAdd(&a.sched[0], 1ull) : (int64_t)blockIdx.x;
      for (;;) {
        const int64_t e0 = t * kTile;
        const uint32_t cnt = t < n_tiles ? (uint32_t)(n_bulk - e0 < kTile ? n_bulk - e0 : kTile) : 0u;
        int64_t t_next = 0;
        if (t < n_tiles) t_next = a.sched ? (int64_t)atomicAdd(&a.sched[0], 1ull) : t + gridDim.x;
        for (int j = 0; j < a.n_ops; ++j, ++L) {
          const uint32_t s = L % kStages;
          if (L >= (uint32_t)kStages) {
            mbar_wait(&empty[s], ((L / kStages) & 1) ^ 1);
            fence_proxy_async_smem();
          }
          if (j == 0) {
            tile_of[s] = t < n_tiles ? t : -1;        // the first member's stage carries the tile index
            if (t >= n_tiles) {
              mbar_arrive(&full[s]);
              break;
            }
          }
          const bool bf = a.flag[j] & kOpBf16;
          const void *src = bf ? (const void *)(static_cast<const uint16_t *>(a.op[j]) + a.src_off + e0)
                               : (const void *)(static_cast<const float *>(a.op[j]) + a.src_off + e0);
          const uint32_t bytes = cnt * (bf ? 2 : 4);
          mbar_expect_tx(&full[s], bytes);
          bulk_g2s(smem + (size_t)s * kStageBytes, src, bytes, &full[s]);
        }
        if (t >= n_tiles) break;
        t = t_next;
      }
      if (a.sched) {                                  // the last CTA resets the counters
        __threadfence();
        if (atomicAdd(&a.sched[1], 1ull) == gridDim.x - 1) {
          a.sched[0] = 0;
          a.sched[1] = 0;
          __threadfence();
        }
      }
    }
  } else {
    const int tid = threadIdx.x;
    uint32_t L = 0;
    for (;;) {
      mbar_wait(&full[L % kStages], (L / kStages) & 1);
      const int64_t t = tile_of[L % kStages];
      if (t < 0) break;
      const int64_t e0 = t * kTile;
      const int cnt = (int)(n_bulk - e0 < kTile ? n_bulk - e0 : kTile);
      float4 x[kChunks];
      for (int j = 0; j < a.n_ops; ++j, ++L) {
        const uint32_t s = L % kStages;
        const bool bf = a.flag[j] & kOpBf16;
        mbar_wait(&full[s], (L / kStages) & 1);
        const uint8_t *st = smem + (size_t)s * kStageBytes;
#pragma unroll
        for (int k = 0; k < kChunks; ++k) {
          const int c = tid + k * kConsumers;
          if (c * 4 < cnt) {
            const float4 u = bf ? widen_bf16x4(reinterpret_cast<const uint2 *>(st)[c])
                                : reinterpret_cast<const float4 *>(st)[c];
            x[k] = j == 0 ? u : add4(x[k], u);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
#pragma unroll
      for (int k = 0; k < kChunks; ++k) {
        const int c = tid + k * kConsumers;
        if (c * 4 < cnt) __stcs(reinterpret_cast<float4 *>(a.out + e0) + c, x[k]);
      }
    }
    const int64_t tail = a.n - n_bulk;                // ragged tail (< 8 elements) on CTA 0
    if (blockIdx.x == 0 && tid < tail) {
      const int64_t e = n_bulk + tid;
      float xv = 0.f;
      for (int j = 0; j < a.n_ops; ++j) {
        const float u = (a.flag[j] & kOpBf16)
                            ? __uint_as_float(uint32_t(static_cast<const uint16_t *>(a.op[j])[a.src_off + e]) << 16)
                            : static_cast<const float *>(a.op[j])[a.src_off + e];
        xv = j == 0 ? u : __fadd_rn(xv, u);
      }
      a.out[e] = xv;
    }
  }
}

}  // namespace bulk

cudaError_t launch_reduce_bulk(const ReduceArgs &a, cudaStream_t s, int sm_count) {
  constexpr int kTile = 4096, kStages = 12;
  constexpr size_t smem = bulk::smem_bytes(kTile, kStages);
  static std::atomic<uint64_t> init{0};
  if (cudaError_t e = ensure_smem(bulk::tree_reduce_bulk<kTile, kStages>, smem, init); e != cudaSuccess)
    return e;
  if (a.n_ops < 1 || a.n < 1) return cudaSuccess;
  const int64_t n_tiles = ((a.n & ~int64_t(7)) + kTile - 1) / kTile;
  int grid = (int)(n_tiles < sm_count ? (n_tiles > 0 ? n_tiles : 1) : sm_count);
  int64_t tile_bytes = 0;                          // dynamic tiles only when a tile loads >= 64 KB
  for (int j = 0; j < a.n_ops; ++j) tile_bytes += (int64_t)kTile * ((a.flag[j] & kOpBf16) ? 2 : 4);
  if (a.sched && tile_bytes < (64 << 10)) {
    ReduceArgs b = a;
    b.sched = nullptr;
    bulk::tree_reduce_bulk<kTile, kStages><<<grid, bulk::kThreads, smem, s>>>(b);
  } else {
    bulk::tree_reduce_bulk<kTile, kStages><<<grid, bulk::kThreads, smem, s>>>(a);
  }
  return cudaGetLastError();
}

template <bool kBf>
static cudaError_t launch_momentum_t(const MomentumArgs &a, cudaStream_t s, int sm_count) {
  constexpr int kTile = 4096, kStages = 12;
  constexpr size_t smem = bulk::smem_bytes(kTile, kStages);
  static std::atomic<uint64_t> init{0};
  if (cudaError_t e = ensure_smem(bulk::fused_commit_momentum<kTile, kStages, kBf>, smem, init); e != cudaSuccess)
    return e;
  const int64_t n_tiles = ((a.n & ~int64_t(7)) + kTile - 1) / kTile;
  int grid = (int)(n_tiles < sm_count ? (n_tiles > 0 ? n_tiles : 1) : sm_count);
  // dynamic tiles for short fp32 lists; bf16 lists measured faster round-robin at every
  // length (config 2 bf16, tau 4: 86.3% vs 80.2%; tau 8: 71.4% vs 65.9%)
  if (!kBf && a.sched && a.n_ops <= 8) {
    bulk::fused_commit_momentum<kTile, kStages, kBf><<<grid, bulk::kThreads, smem, s>>>(a);
  } else {
    static std::atomic<uint64_t> init_rr{0};
    if (cudaError_t e = ensure_smem(bulk::fused_commit_momentum_rr<kTile, kStages, kBf>, smem, init_rr); e != cudaSuccess)
      return e;
    bulk::fused_commit_momentum_rr<kTile, kStages, kBf><<<grid, bulk::kThreads, smem, s>>>(a);
  }
  return cudaGetLastError();
}

// all-bf16 operand lists take the branch-free fold (config 2 bf16, gamma 0.9, tau 32: 60% ->
// 73% of the HBM roofline); fp32 keeps the generic one, which measured faster there
cudaError_t launch_commit_momentum(const MomentumArgs &a, cudaStream_t s, int sm_count) {
  bool all_bf16 = a.n_ops > 0;
  for (int j = 0; j < a.n_ops && all_bf16; ++j) all_bf16 = (a.flag[j] & kOpBf16) != 0;
  // the 16-warp kernel for all-bf16 lists of >= MLF_MOM_WIDE operands (0: never): config 2
  // tau 8 / 16 / 32 92.1 / 93.5 / 95.0% vs 89.8 / 80.7 / 78.0% for the 8-warp kernel; at tau 4
  // (4 operands, a third of the stages are w and h) the 8-warp kernel wins, 97.8% vs 92.7%
  const char *wide = getenv("MLF_MOM_WIDE");
  const int wide_min = wide ? atoi(wide) : 6;
  // MLF_MOM_BH2=1 (A/B knob): two CTAs per SM, each 8 consumer warps over a 12-stage ring of
  // 8 KB bf16 stages (the same warps per SM, more registers per thread, two producers)
  const char *bh2 = getenv("MLF_MOM_BH2");
  if (all_bf16 && wide_min > 0 && a.n_ops >= wide_min && bh2 && atoi(bh2) == 1) {
    constexpr int kT = 4096, kS = 12, kCW = 8;
    constexpr size_t smem = (size_t)kS * kT * 2 + 2 * kS * sizeof(uint64_t);
    static std::atomic<uint64_t> init{0};
    if (cudaError_t e = ensure_smem(bulk::fused_commit_momentum_bh<kT, kS, kCW>, smem, init); e != cudaSuccess)
      return e;
    const int64_t n_tiles = ((a.n & ~int64_t(7)) + kT - 1) / kT;
    const int ctas = 2 * (sm_count > 0 ? sm_count : 148);
    const int grid = (int)(n_tiles < ctas ? (n_tiles > 0 ? n_tiles : 1) : ctas);
    bulk::fused_commit_momentum_bh<kT, kS, kCW><<<grid, kCW * 32 + 32, smem, s>>>(a);
    return cudaGetLastError();
  }
  if (all_bf16 && wide_min > 0 && a.n_ops >= wide_min) {
    constexpr int kT = 8192, kS = 12, kCW = 16;
    constexpr size_t smem = (size_t)kS * kT * 2 + 2 * kS * sizeof(uint64_t);
    static std::atomic<uint64_t> init{0};
    if (cudaError_t e = ensure_smem(bulk::fused_commit_momentum_bh<kT, kS, kCW>, smem, init); e != cudaSuccess)
      return e;
    const int64_t n_tiles = ((a.n & ~int64_t(7)) + kT - 1) / kT;
    const int sms = sm_count > 0 ? sm_count : 148;
    const int grid = (int)(n_tiles < sms ? (n_tiles > 0 ? n_tiles : 1) : sms);
    bulk::fused_commit_momentum_bh<kT, kS, kCW><<<grid, kCW * 32 + 32, smem, s>>>(a);
    return cudaGetLastError();
  }
  return all_bf16 ? launch_momentum_t<true>(a, s, sm_count) : launch_momentum_t<false>(a, s, sm_count);
}

template <int kTile, int kStages, bool kHint>
static cudaError_t launch_tile_h(const CommitArgs &a, cudaStream_t s, int sm_count) {
  constexpr size_t smem = bulk::smem_bytes(kTile, kStages);
  static std::atomic<uint64_t> init{0};
  if (cudaError_t e = ensure_smem(bulk::fused_commit_bulk<kTile, kStages, kHint>, smem, init); e != cudaSuccess)
    return e;
  const int64_t n_tiles = ((a.n & ~int64_t(7)) + kTile - 1) / kTile;
  int grid = (int)(n_tiles < sm_count ? (n_tiles > 0 ? n_tiles : 1) : sm_count);
  // Dynamic tiles pay one global atomic per tile; below ~64 KB of loads per tile its latency
  // under 148-way contention outlasts the tile (config 2 bf16, tau 4: 85.8% dynamic vs 98.9%
  // static; fp32 tau 4, 80 KB per tile: 104% vs 98%), so short tiles stay round-robin.
  int64_t tile_bytes = (int64_t)kTile * 4;
  for (int j = 0; j < a.n_ops; ++j) tile_bytes += (int64_t)kTile * ((a.flag[j] & kOpBf16) ? 2 : 4);
  if (a.sched && tile_bytes < (64 << 10)) {
    CommitArgs b = a;
    b.sched = nullptr;
    bulk::fused_commit_bulk<kTile, kStages, kHint><<<grid, bulk::kThreads, smem, s>>>(b);
  } else {
    bulk::fused_commit_bulk<kTile, kStages, kHint><<<grid, bulk::kThreads, smem, s>>>(a);
  }
  return cudaGetLastError();
}
// The evict-first hint pays only where every copy is >= 16 KB: the hinted copy costs the
// producer more issue time, and with 8 KB copies that outweighs the L2 gain (config 2, tau 4:
// fp32 16 KB copies +3.5% static / +3% dynamic; bf16 8 KB copies -3.3%; fp32 2048-element
// tiles -2%)
template <int kTile, int kStages>
static cudaError_t launch_tile(const CommitArgs &a, cudaStream_t s, int sm_count) {
  bool hint = a.l2_hint && kTile * 4 >= (16 << 10);
  for (int j = 0; j < a.n_ops && hint; ++j) hint = kTile * ((a.flag[j] & kOpBf16) ? 2 : 4) >= (16 << 10);
  return hint ? launch_tile_h<kTile, kStages, true>(a, s, sm_count)
              : launch_tile_h<kTile, kStages, false>(a, s, sm_count);
}

// Tile size (elements) per bulk copy: MLF_BULK_TILE in {1024, 2048, 4096, 8192}; the ring is
// always 192 KB.  Default 4096 (16 KB per copy): measured best on one B200 (99.7% of the
// HBM copy roofline at config 2, tau 4, vs 93.5% at 2048 and 8192); NVLink-bound runs
// are insensitive to the tile size.
cudaError_t launch_commit_bulk(const CommitArgs &a, cudaStream_t s, int sm_count) {
  const char *env = getenv("MLF_BULK_TILE");           // read per launch (tests switch it)
  const int forced = env ? atoi(env) : 0;
  // adaptive tile: the largest of 4096 / 2048 / 1024 elements that still deals >= 32 tiles to
  // every persistent CTA, so the last wave's imbalance stays small (a shard of 6.4M elements,
  // config 4 at 4 GPUs: 76.8% of the NVLink roofline at 2048 vs 70.8% at 4096)
  int tile = forced;
  const int sms = sm_count > 0 ? sm_count : 148;
  if (tile == 0) {
    // all operands bf16 (one context's update dtype; tree-mode aggregates are fp32) and enough
    // of them that the stage hand-offs matter: 16 KB bf16 copies through the 8192-element
    // layout while it still deals >= 16 tiles per CTA (config 2 bf16: tau 32 98.3% vs 86.5%;
    // at tau 4 the 4096 layout's finer tiles win, 103.9% vs 96.2%)
    bool all_bf16 = a.n_ops >= 8;
    for (int j = 0; j < a.n_ops && all_bf16; ++j) all_bf16 = (a.flag[j] & kOpBf16) != 0;
    const char *hb = getenv("MLF_BULK_BF16");
    if (all_bf16 && !(hb && atoi(hb) == 0) && (a.n / 8192) / sms >= 16) {
      constexpr int kT = 8192, kS = 12;
      constexpr size_t smem = (size_t)kS * kT * 2 + 3 * kS * sizeof(uint64_t);
      static std::atomic<uint64_t> init{0};
      if (cudaError_t e = ensure_smem(bulk::fused_commit_bulk_h<kT, kS>, smem, init); e != cudaSuccess)
        return e;
      const int64_t n_tiles = ((a.n & ~int64_t(7)) + kT - 1) / kT;
      const int grid = (int)(n_tiles < sms ? (n_tiles > 0 ? n_tiles : 1) : sms);
      bulk::fused_commit_bulk_h<kT, kS><<<grid, bulk::kThreads, smem, s>>>(a);
      return cudaGetLastError();
    }
    const int64_t per_cta = (a.n / 4096) / sms;
    // contiguous ranges balance the bytes per CTA by construction: keep 16 KB copies
    tile = (per_cta >= 32 || (a.contig && !a.sched)) ? 4096 : ((a.n / 2048) / sms >= 32 ? 2048 : 1024);
  }
  if (tile == 8192) return launch_tile<8192, 6>(a, s, sm_count);
  if (tile == 2048) return launch_tile<2048, 24>(a, s, sm_count);
  if (tile == 1024) return launch_tile<1024, 48>(a, s, sm_count);
  return launch_tile<4096, 12>(a, s, sm_count);
}

}  // namespace mlf
