// K1 / K2: byte-lane split & merge, the identity BBC1 container, lane histograms.
//
// Reference semantics (/root/reference/proj):
//   byte_split   src/codec.cpp:86-99   high[k] = s[2k+1], low[k] = s[2k]
//   byte_merge   src/codec.cpp:101-111
//   identity backend + serialize_container  src/codec.cpp:42-51,127-140
//   entropy_bits_per_byte's histogram        src/codec.cpp:113-125
//
// All four are HBM-bound byte permutations.  Kernels are output-stationary:
// every thread owns one aligned 16-byte output word, gathers its source bytes
// with aligned 128-bit loads (neighbouring threads' overlapping loads hit L1,
// so DRAM sees each input byte once) and writes one STG.128.  Words that
// straddle a region boundary (container header / lane seam / buffer ends) take
// a byte-wise path.  Grids are capped at 8 CTAs per SM (148 SMs) and
// grid-stride so every launch is a whole number of waves.
#include "bb_common.cuh"
#include "bb_kernels.h"

namespace bb {

namespace {

__device__ __forceinline__ uint8_t header_byte(unsigned j, int backend, int split, uint64_t count,
                                               uint64_t hl, uint64_t ll) {
  if (j < 4) return (uint8_t)"BBC1"[j];
  if (j == 4) return 1;
  if (j == 5) return (uint8_t)backend;
  if (j == 6) return (uint8_t)(split ? 1 : 0);
  uint64_t v = j < 15 ? count : j < 23 ? hl : ll;
  unsigned k = (j - 7) & 7;
  return (uint8_t)(v >> (8 * k));
}

// byte j of serialize_container(identity compress(in, split))
__device__ __forceinline__ uint8_t container_byte(const uint8_t* in, uint64_t n, int split,
                                                  uint64_t j) {
  uint64_t N = n / 2;
  if (j < BB_CONTAINER_HEADER)
    return header_byte((unsigned)j, 0, split, N, split ? N : n, split ? N : 0);
  uint64_t b = j - BB_CONTAINER_HEADER;
  if (!split) return in[b];
  return b < N ? in[2 * b + 1] : in[2 * (b - N)];
}

__device__ __forceinline__ void odd_even16(const uint8_t* src, uint32_t hi[4], uint32_t lo[4]) {
  uint32_t a[4], b[4];
  gather16(src, a);
  gather16(src + 16, b);
  hi[0] = __byte_perm(a[0], a[1], 0x7531);
  hi[1] = __byte_perm(a[2], a[3], 0x7531);
  hi[2] = __byte_perm(b[0], b[1], 0x7531);
  hi[3] = __byte_perm(b[2], b[3], 0x7531);
  lo[0] = __byte_perm(a[0], a[1], 0x6420);
  lo[1] = __byte_perm(a[2], a[3], 0x6420);
  lo[2] = __byte_perm(b[0], b[1], 0x6420);
  lo[3] = __byte_perm(b[2], b[3], 0x6420);
}

__global__ void __launch_bounds__(256) k_identity_container(const uint8_t* __restrict__ in,
                                                            uint64_t n, int split,
                                                            uint8_t* __restrict__ out) {
  const uint64_t total = BB_CONTAINER_HEADER + n;
  const uint64_t N = n / 2;
  const uintptr_t o0 = reinterpret_cast<uintptr_t>(out);
  const uintptr_t first = o0 & ~uintptr_t(15);
  const uint64_t words = (o0 + total - first + 15) / 16;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words;
       w += (uint64_t)gridDim.x * blockDim.x) {
    uintptr_t A = first + 16 * w;
    int64_t j0 = (int64_t)(A - o0);  // container offset of this word's first byte
    bool full = j0 >= BB_CONTAINER_HEADER && (uint64_t)(j0 + 16) <= total;
    if (full && split && (uint64_t)(j0 + 16) <= BB_CONTAINER_HEADER + N) {
      uint32_t hi[4], lo[4];
      odd_even16(in + 2 * (j0 - BB_CONTAINER_HEADER), hi, lo);
      *reinterpret_cast<uint4*>(A) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    } else if (full && split && j0 >= (int64_t)(BB_CONTAINER_HEADER + N)) {
      uint32_t hi[4], lo[4];
      odd_even16(in + 2 * (j0 - BB_CONTAINER_HEADER - (int64_t)N), hi, lo);
      *reinterpret_cast<uint4*>(A) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    } else if (full && !split) {
      uint32_t v[4];
      gather16(in + (j0 - BB_CONTAINER_HEADER), v);
      *reinterpret_cast<uint4*>(A) = make_uint4(v[0], v[1], v[2], v[3]);
    } else {
      for (int k = 0; k < 16; k++) {
        int64_t j = j0 + k;
        if (j >= 0 && (uint64_t)j < total)
          out[j] = container_byte(in, n, split, (uint64_t)j);
      }
    }
  }
}

// split: one thread per 16 elements
__global__ void __launch_bounds__(256) k_split(const uint8_t* __restrict__ in, uint64_t count,
                                               uint8_t* __restrict__ hi_out,
                                               uint8_t* __restrict__ lo_out) {
  const uint64_t groups = (count + 15) / 16;
  const bool aligned = ((reinterpret_cast<uintptr_t>(hi_out) | reinterpret_cast<uintptr_t>(lo_out)) & 15) == 0;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
       g += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t e0 = 16 * g;
    if (e0 + 16 <= count) {
      uint32_t hi[4], lo[4];
      odd_even16(in + 2 * e0, hi, lo);
      if (aligned) {
        *reinterpret_cast<uint4*>(hi_out + e0) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(lo_out + e0) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      } else {
        for (int k = 0; k < 16; k++) {
          hi_out[e0 + k] = (uint8_t)(hi[k >> 2] >> (8 * (k & 3)));
          lo_out[e0 + k] = (uint8_t)(lo[k >> 2] >> (8 * (k & 3)));
        }
      }
    } else {
      for (uint64_t e = e0; e < count; e++) {
        lo_out[e] = in[2 * e];
        hi_out[e] = in[2 * e + 1];
      }
    }
  }
}

// merge: one thread per 8 elements (one 16-byte output word)
__global__ void __launch_bounds__(256) k_merge(const uint8_t* __restrict__ hi_in,
                                               const uint8_t* __restrict__ lo_in, uint64_t count,
                                               uint8_t* __restrict__ out) {
  const uint64_t groups = (count + 7) / 8;
  const bool aligned = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
       g += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t e0 = 8 * g;
    if (e0 + 8 <= count) {
      uint32_t h[2], l[2];
      gather8(hi_in + e0, h);
      gather8(lo_in + e0, l);
      uint4 v = make_uint4(__byte_perm(l[0], h[0], 0x5140), __byte_perm(l[0], h[0], 0x7362),
                           __byte_perm(l[1], h[1], 0x5140), __byte_perm(l[1], h[1], 0x7362));
      if (aligned) {
        *reinterpret_cast<uint4*>(out + 2 * e0) = v;
      } else {
        uint32_t w[4] = {v.x, v.y, v.z, v.w};
        for (int k = 0; k < 16; k++) out[2 * e0 + k] = (uint8_t)(w[k >> 2] >> (8 * (k & 3)));
      }
    } else {
      for (uint64_t e = e0; e < count; e++) {
        out[2 * e] = lo_in[e];
        out[2 * e + 1] = hi_in[e];
      }
    }
  }
}

// 256-bin histogram: per-warp shared-memory bins, one 64-bit atomic per bin per CTA
__global__ void __launch_bounds__(256) k_hist256(const uint8_t* __restrict__ in, uint64_t n,
                                                 unsigned long long* __restrict__ counts) {
  __shared__ uint32_t bins[8][256];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&bins[0][0])[i] = 0;
  __syncthreads();
  uintptr_t a0 = reinterpret_cast<uintptr_t>(in);
  uint64_t head = (16 - (a0 & 15)) & 15;
  if (head > n) head = n;
  uint64_t vecs = (n - head) / 16;
  const uint8_t* base = in + head;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < vecs;
       v += (uint64_t)gridDim.x * blockDim.x) {
    uint4 x = ldg16(base + 16 * v);
    uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; k++) {
      atomicAdd(&bins[warp][w[k] & 0xff], 1u);
      atomicAdd(&bins[warp][(w[k] >> 8) & 0xff], 1u);
      atomicAdd(&bins[warp][(w[k] >> 16) & 0xff], 1u);
      atomicAdd(&bins[warp][w[k] >> 24], 1u);
    }
  }
  if (blockIdx.x == 0) {
    for (uint64_t i = threadIdx.x; i < head; i += blockDim.x) atomicAdd(&bins[warp][in[i]], 1u);
    for (uint64_t i = head + 16 * vecs + threadIdx.x; i < n; i += blockDim.x)
      atomicAdd(&bins[warp][in[i]], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x) {
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < 8; w++) s += bins[w][b];
    if (s) atomicAdd(&counts[b], (unsigned long long)s);
  }
}

// a != b anywhere in [0, n): 16-byte loads where both sides share alignment, bytes otherwise
__global__ void __launch_bounds__(256) k_differ(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                                                uint64_t n, unsigned int* __restrict__ differ) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uintptr_t pa = reinterpret_cast<uintptr_t>(a), pb = reinterpret_cast<uintptr_t>(b);
  bool d = false;
  if (((pa ^ pb) & 15) == 0) {
    uint64_t head = (16 - (pa & 15)) & 15;
    if (head > n) head = n;
    const uint64_t vecs = (n - head) / 16;
    for (uint64_t v = tid; v < vecs; v += stride) {
      uint4 x = ldg16(a + head + 16 * v), y = ldg16(b + head + 16 * v);
      d |= (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
    }
    for (uint64_t i = tid; i < head; i += stride) d |= a[i] != b[i];
    for (uint64_t i = head + 16 * vecs + tid; i < n; i += stride) d |= a[i] != b[i];
  } else {
    for (uint64_t i = tid; i < n; i += stride) d |= a[i] != b[i];
  }
  if (__any_sync(0xffffffffu, d) && (threadIdx.x & 31) == 0) atomicOr(differ, 1u);
}

}  // namespace

int launch_differ(const uint8_t* a, const uint8_t* b, uint64_t n, unsigned int* differ, cudaStream_t st) {
  BB_CUDA_TRY(cudaMemsetAsync(differ, 0, sizeof(unsigned int), st));
  if (n == 0) return BB_OK;
  k_differ<<<grid_for(n / 16 + 1, 256, 8), 256, 0, st>>>(a, b, n, differ);
  BB_LAUNCH_CHECK();
  return BB_OK;
}

int launch_identity_container(const uint8_t* in, uint64_t n, int split, uint8_t* out,
                              cudaStream_t st) {
  uint64_t words = (BB_CONTAINER_HEADER + n) / 16 + 2;
  k_identity_container<<<grid_for(words, 256, 16), 256, 0, st>>>(in, n, split, out);
  BB_LAUNCH_CHECK();
  return BB_OK;
}

int launch_split(const uint8_t* in, uint64_t count, uint8_t* hi, uint8_t* lo, cudaStream_t st) {
  if (count == 0) return BB_OK;
  k_split<<<grid_for((count + 15) / 16, 256, 16), 256, 0, st>>>(in, count, hi, lo);
  BB_LAUNCH_CHECK();
  return BB_OK;
}

int launch_merge(const uint8_t* hi, const uint8_t* lo, uint64_t count, uint8_t* out, cudaStream_t st) {
  if (count == 0) return BB_OK;
  k_merge<<<grid_for((count + 7) / 8, 256, 16), 256, 0, st>>>(hi, lo, count, out);
  BB_LAUNCH_CHECK();
  return BB_OK;
}

int launch_hist256(const uint8_t* in, uint64_t n, unsigned long long* counts, cudaStream_t st) {
  BB_CUDA_TRY(cudaMemsetAsync(counts, 0, 256 * sizeof(unsigned long long), st));
  if (n == 0) return BB_OK;
  k_hist256<<<grid_for(n / 16 + 1, 256, 4), 256, 0, st>>>(in, n, counts);
  BB_LAUNCH_CHECK();
  return BB_OK;
}

}  // namespace bb
