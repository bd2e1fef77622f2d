// Shared helpers for the sm_100a codec kernels and the C-ABI layer.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>

#include "bbcodec.h"

namespace bb {

void set_error(const char* fmt, ...);
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

constexpr int kNumSMs = 148;  // B200

#define BB_CUDA_TRY(expr)                                                                   \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      bb::set_error("CUDA error %s at %s:%d", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return BB_CUDA_ERROR;                                                                 \
    }                                                                                       \
  } while (0)

bool debug_sync();  // BB_DEBUG_SYNC=1: synchronize + log after every launch

#define BB_LAUNCH_CHECK()                                                                       \
  do {                                                                                          \
    bb::count_launch();                                                                         \
    if (bb::debug_sync()) {                                                                     \
      fprintf(stderr, "[bb] launch %s:%d\n", __FILE__, __LINE__);                              \
      cudaDeviceSynchronize();                                                                  \
      fprintf(stderr, "[bb]   done %s:%d\n", __FILE__, __LINE__);                              \
    }                                                                                           \
    cudaError_t e_ = cudaGetLastError();                                                        \
    if (e_ != cudaSuccess) {                                                                    \
      bb::set_error("CUDA launch error %s at %s:%d", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return BB_CUDA_ERROR;                                                                     \
    }                                                                                           \
  } while (0)

// Optional per-stage CUDA-event timing (enabled by bb_stage_timing(1)); the time
// between consecutive marks is charged to the earlier mark's stage name.
extern std::atomic<int> g_stage_timing;
struct StageTimer {
  cudaStream_t st;
  bool on;
  const char* names[32];
  cudaEvent_t ev[33];
  int n = 0;
  explicit StageTimer(cudaStream_t s) : st(s), on(g_stage_timing.load() != 0) {}
  void mark(const char* name) {
    if (!on || n >= 32) return;
    names[n] = name;
    cudaEventCreate(&ev[n]);
    cudaEventRecord(ev[n], st);
    n++;
  }
  void finish();  // call after the stream is synchronized
};

inline unsigned grid_for(size_t work_items, int threads, int per_sm = 8) {
  size_t blocks = (work_items + threads - 1) / threads;
  size_t cap = (size_t)kNumSMs * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  return (unsigned)blocks;
}

// ---------------------------------------------------------------------------
// Aligned-load gathers: 16 bytes at an arbitrary device address, read with at
// most two aligned 128-bit loads (the neighbours' loads hit L1).  A load never
// leaves the 16-byte block of a byte that is in bounds.
__device__ __forceinline__ uint4 ldg16(const uint8_t* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

__device__ __forceinline__ void gather16(const uint8_t* q, uint32_t out[4]) {
  uintptr_t a = reinterpret_cast<uintptr_t>(q);
  const uint8_t* A = reinterpret_cast<const uint8_t*>(a & ~uintptr_t(15));
  unsigned s = (unsigned)(a & 15);
  uint4 x = ldg16(A);
  if (s == 0) {
    out[0] = x.x, out[1] = x.y, out[2] = x.z, out[3] = x.w;
    return;
  }
  uint4 y = ldg16(A + 16);
  uint32_t w[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
  unsigned j = s >> 2, r = (s & 3) * 8;
  // shift the 8-word window left by j words with selects (no local memory)
#pragma unroll
  for (int i = 0; i < 4; i++) {
    uint32_t lo = j == 0 ? w[i] : j == 1 ? w[i + 1] : j == 2 ? w[i + 2] : w[i + 3];
    uint32_t hi = j == 0 ? w[i + 1] : j == 1 ? w[i + 2] : j == 2 ? w[i + 3] : w[i + 4];
    out[i] = __funnelshift_r(lo, hi, r);
  }
}

// 8 bytes at an arbitrary address (as two words)
__device__ __forceinline__ void gather8(const uint8_t* q, uint32_t out[2]) {
  uintptr_t a = reinterpret_cast<uintptr_t>(q);
  const uint8_t* A = reinterpret_cast<const uint8_t*>(a & ~uintptr_t(7));
  unsigned s = (unsigned)(a & 7);
  uint2 x = __ldg(reinterpret_cast<const uint2*>(A));
  if (s == 0) {
    out[0] = x.x, out[1] = x.y;
    return;
  }
  uint2 y = __ldg(reinterpret_cast<const uint2*>(A + 8));
  uint32_t w[4] = {x.x, x.y, y.x, y.y};
  unsigned j = s >> 2, r = (s & 3) * 8;
  out[0] = __funnelshift_r(j ? w[1] : w[0], j ? w[2] : w[1], r);
  out[1] = __funnelshift_r(j ? w[2] : w[1], j ? w[3] : w[2], r);
}

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, sm_90+): one elected thread moves a 16-byte
// aligned tile global -> shared through the copy engine, completion tracked by a
// shared-memory mbarrier (transaction bytes).  Used to stage tiles whose bytes
// are then expanded by the CTA (inflate's LZ77 resolution windows).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// arm the barrier for `bytes` and start the copy (one thread; sizes and addresses 16-byte aligned)
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

}  // namespace bb
