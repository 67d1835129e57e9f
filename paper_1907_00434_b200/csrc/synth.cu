// synth.cu — test-infrastructure kernels: the counter-based input generator and
// a plain device copy (HBM / NVLink denominators).  Not on the hot path.
//
// The generator is splitmix64 used as a counter-based stream:
//   key          = sm64(sm64(sm64(seed ^ kind) ^ a) ^ b),  sm64(x) = mix64(x + GOLDEN)
//   word(key, i) = mix64(key + (i + 1) * GOLDEN)
// with the value maps documented in synthgen/__init__.py (an independent
// NumPy implementation of the same definition; tests compare them bit for bit).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace mlf {

static constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t sm64(uint64_t x) { return mix64(x + kGolden); }

uint64_t synth_stream_key(uint64_t seed, uint64_t kind, uint64_t a, uint64_t b) {
  uint64_t k = sm64(seed ^ kind);
  k = sm64(k ^ a);
  return sm64(k ^ b);
}

// kind 1 = update, 2 = w0; variant 0 normal, 1 exact; dtype 0 f32, 1 bf16
__global__ void synth_fill_kernel(void *dst, int64_t n, int64_t off, int dtype, uint64_t key, int kind,
                                  int variant) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t w = mix64(key + (uint64_t)(off + i + 1) * kGolden);
    float v;
    if (kind == 2) {
      v = variant == 0 ? (float)((int64_t)(w >> 40) - (1ll << 23)) * 0x1p-24f
                       : (float)((int64_t)(w >> 42) - (1ll << 21)) * 0x1p-24f;
    } else if (dtype == 0) {
      v = variant == 0 ? (float)((int64_t)(w >> 40) - (1ll << 23)) * 0x1p-31f
                       : (float)((int64_t)(w >> 53) - 1024) * 0x1p-20f;
    } else {
      v = (float)((int64_t)(w >> 56) - 128) * (variant == 0 ? 0x1p-14f : 0x1p-17f);
    }
    if (dtype == 1 && kind != 2)
      static_cast<uint16_t *>(dst)[i] = (uint16_t)(__float_as_uint(v) >> 16);
    else
      static_cast<float *>(dst)[i] = v;
  }
}

cudaError_t launch_synth(void *dst, int64_t n, int64_t elem_offset, int dtype, uint64_t key, int kind, int variant,
                         cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  synth_fill_kernel<<<(int)blocks, 256, 0, s>>>(dst, n, elem_offset, dtype, key, kind, variant);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) copy_kernel(float4 *__restrict__ dst, const float4 *__restrict__ src, int64_t nv) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < nv; i += 4 * stride) {
    float4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride),
           d = __ldcs(src + i + 3 * stride);
    __stcs(dst + i, a);
    __stcs(dst + i + stride, b);
    __stcs(dst + i + 2 * stride, c);
    __stcs(dst + i + 3 * stride, d);
  }
  for (; i < nv; i += stride) __stcs(dst + i, __ldcs(src + i));
}

// get of the whole model: every shard (local or peer) copied in ONE launch, so the reads
// from all peers are in flight together instead of one peer per launch
__global__ void __launch_bounds__(256) gather_kernel(const __grid_constant__ GatherArgs a) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int j = 0;
  for (; i < a.total_v; i += stride) {
    while (j + 1 < a.n && i >= a.vstart[j + 1]) ++j;
    while (j > 0 && i < a.vstart[j]) --j;
    const int64_t v = i - a.vstart[j];
    __stcs(reinterpret_cast<float4 *>(a.dst[j]) + v, __ldcs(reinterpret_cast<const float4 *>(a.src[j]) + v));
  }
}

// Copy with TMA bulk copies only (denominator probe): one elected thread per CTA moves 16 KB
// chunks global -> shared (cp.async.bulk ... mbarrier::complete_tx) -> global (bulk store),
// kStages chunks in flight per SM.  Used to measure what TMA-driven peer reads can reach.
namespace bulkcopy {
constexpr int kChunk = kBulkChunk, kStages = 12;
__device__ __forceinline__ uint32_t saddr(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
}  // namespace bulkcopy

__global__ void __launch_bounds__(32, 1) bulk_copy_kernel(const __grid_constant__ BulkSegs a) {
  using namespace bulkcopy;
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)kStages * kChunk);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  // round i of this CTA works on segment i % n, chunk (i / n) * gridDim.x + blockIdx.x of it:
  // every CTA interleaves the segments (a gather's local shard and its NVLink shards are read
  // at the same time instead of one after the other)
  int64_t kmax = 0;
  for (int j = 0; j < a.n; ++j) kmax = max(kmax, a.cstart[j + 1] - a.cstart[j]);
  const int64_t rounds = (int64_t)a.n * ((kmax + gridDim.x - 1) / gridDim.x);
  auto next = [&](int64_t i) -> int64_t {          // first round >= i with a chunk for this CTA
    for (; i < rounds; ++i) {
      const int j = (int)(i % a.n);
      if ((i / a.n) * gridDim.x + blockIdx.x < a.cstart[j + 1] - a.cstart[j]) return i;
    }
    return rounds;
  };
  auto locate = [&](int64_t i, int &j, int64_t &off, uint32_t &len) {
    j = (int)(i % a.n);
    off = ((i / a.n) * gridDim.x + blockIdx.x) * kChunk;
    const int64_t rest = a.bytes[j] - off;
    len = (uint32_t)(rest < kChunk ? rest : kChunk);
  };
  // issue loads for up to kStages chunks, then per chunk: wait load, store it; the stage of the
  // store issued kLag chunks earlier is refilled once that store has read it (wait_group.read
  // kLag), so kLag stores and kStages - kLag loads stay in flight
  constexpr uint32_t kLag = 4;
  int64_t i_load = next(0), i_store = i_load;
  uint32_t L = 0, S = 0;
  auto issue_load = [&](int64_t i, uint32_t stage) {
    int j;
    int64_t off;
    uint32_t len;
    locate(i, j, off, len);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&full[stage])), "r"(len)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     saddr(sm + (size_t)stage * kChunk)),
                 "l"(a.src[j] + off), "r"(len), "r"(saddr(&full[stage]))
                 : "memory");
  };
  for (; L < (uint32_t)kStages && i_load < rounds; ++L, i_load = next(i_load + 1)) issue_load(i_load, L);
  for (; i_store < rounds; i_store = next(i_store + 1), ++S) {
    const uint32_t stage = S % kStages, parity = (S / kStages) & 1;
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
            saddr(&full[stage])),
        "r"(parity)
        : "memory");
    int j;
    int64_t off;
    uint32_t len;
    locate(i_store, j, off, len);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a.dst[j] + off),
                 "r"(saddr(sm + (size_t)stage * kChunk)), "r"(len)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (S >= kLag && i_load < rounds) {
      // at most kLag store groups still reading: the store of chunk S - kLag has read its stage
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kLag) : "memory");
      issue_load(i_load, L % kStages);           // L % kStages == (S - kLag) % kStages
      i_load = next(i_load + 1);
      ++L;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Read-only roofline probe: every CTA streams its 16 KB chunks of src into a ring of shared-memory
// stages with TMA bulk copies and waits for each to land; nothing is written back.  The read end of
// the mixed read/write HBM ceiling bench.py reports (bench.py roofline_extras).
__global__ void __launch_bounds__(32, 1) bulk_read_kernel(const char *src, int64_t n_chunks, int64_t bytes) {
  using namespace bulkcopy;
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)kStages * kChunk);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t L = 0, S = 0;
  int64_t i_load = blockIdx.x, i_wait = blockIdx.x;
  auto issue = [&](int64_t i, uint32_t stage) {
    const int64_t off = i * kChunk;
    const uint32_t len = (uint32_t)(bytes - off < kChunk ? bytes - off : kChunk);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&full[stage])), "r"(len)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     saddr(sm + (size_t)stage * kChunk)),
                 "l"(src + off), "r"(len), "r"(saddr(&full[stage]))
                 : "memory");
  };
  for (; L < (uint32_t)kStages && i_load < n_chunks; ++L, i_load += gridDim.x) issue(i_load, L);
  for (; i_wait < n_chunks; i_wait += gridDim.x, ++S) {
    const uint32_t stage = S % kStages, parity = (S / kStages) & 1;
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
            saddr(&full[stage])),
        "r"(parity)
        : "memory");
    if (i_load < n_chunks) {                       // the stage was consumed on arrival: refill it
      issue(i_load, stage);
      i_load += gridDim.x;
    }
  }
}

cudaError_t launch_bulk_read(const void *src, int64_t bytes, cudaStream_t s, int sm_count) {
  using namespace bulkcopy;
  if (bytes <= 0) return cudaSuccess;
  const size_t smem = (size_t)kStages * kChunk + kStages * sizeof(uint64_t);
  static std::atomic<uint64_t> init{0};
  if (cudaError_t e = ensure_smem(bulk_read_kernel, smem, init); e != cudaSuccess) return e;
  bulk_read_kernel<<<sm_count, 32, smem, s>>>(static_cast<const char *>(src), (bytes + kChunk - 1) / kChunk, bytes);
  return cudaGetLastError();
}

cudaError_t launch_bulk_segs(const BulkSegs &a, cudaStream_t s, int sm_count) {
  using namespace bulkcopy;
  if (a.n <= 0 || a.cstart[a.n] <= 0) return cudaSuccess;
  const size_t smem = (size_t)kStages * kChunk + kStages * sizeof(uint64_t);
  static std::atomic<uint64_t> init{0};
  if (cudaError_t e = ensure_smem(bulk_copy_kernel, smem, init); e != cudaSuccess)
    return e;
  bulk_copy_kernel<<<sm_count, 32, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_bulk_copy(void *dst, const void *src, int64_t bytes, cudaStream_t s, int sm_count) {
  BulkSegs a{};
  if (bytes <= 0) return cudaSuccess;
  a.n = 1;
  a.dst[0] = static_cast<char *>(dst);
  a.src[0] = static_cast<const char *>(src);
  a.bytes[0] = bytes;
  a.cstart[0] = 0;
  a.cstart[1] = (bytes + bulkcopy::kChunk - 1) / bulkcopy::kChunk;
  return launch_bulk_segs(a, s, sm_count);
}

cudaError_t launch_gather(const GatherArgs &a, cudaStream_t s, int sm_count) {
  if (a.total_v <= 0) return cudaSuccess;
  gather_kernel<<<sm_count * 8, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_copy(void *dst, const void *src, int64_t bytes, cudaStream_t s, int sm_count) {
  int64_t nv = bytes / 16;
  if (nv <= 0) return cudaSuccess;
  copy_kernel<<<sm_count * 8, 256, 0, s>>>(static_cast<float4 *>(dst), static_cast<const float4 *>(src), nv);
  return cudaGetLastError();
}

}  // namespace mlf
