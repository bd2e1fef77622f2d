// KV-cache offload chunks (BASELINE config 4): the producer
// side that turns a layer's KV cache into contiguous per-sequence chunks for the
// BBC1 codec before host / peer transfer.  The reference only models KV offload
// (cost_model.cpp:30-47: alpha, kv bytes = 2 * layers * ctx * d * 2 B); here the
// chunk is one (layer, K|V, sequence) = [ctx, d] fp16, as SURVEY §8 config 4
// defines it.
//
// A contiguous [B, T, D] cache needs no copy (a chunk is a view).  A paged cache
// (page pool [n_pages, page_bytes], one page table per sequence) is gathered here:
// one CTA per destination page, 16-byte vector copies when both sides allow it.
#include "bb_common.cuh"
#include "bb_kernels.h"

namespace bb {
namespace {

__global__ void k_gather_pages(const uint8_t* __restrict__ pool, uint64_t page_bytes,
                               const uint32_t* __restrict__ page_ids, uint32_t n_pages, uint64_t n_pool,
                               uint8_t* __restrict__ out, int* __restrict__ bad) {
  for (uint32_t p = blockIdx.x; p < n_pages; p += gridDim.x) {
    const uint32_t id = page_ids[p];
    if (id >= n_pool) {
      if (threadIdx.x == 0) atomicExch(bad, 1);
      continue;
    }
    const uint8_t* s = pool + (uint64_t)id * page_bytes;
    uint8_t* d = out + (uint64_t)p * page_bytes;
    if ((page_bytes & 15) == 0 && (((uintptr_t)s | (uintptr_t)d) & 15) == 0) {
      const uint4* s4 = reinterpret_cast<const uint4*>(s);
      uint4* d4 = reinterpret_cast<uint4*>(d);
      const uint64_t n4 = page_bytes / 16;
      for (uint64_t i = threadIdx.x; i < n4; i += blockDim.x) d4[i] = __ldcs(s4 + i);
    } else {
      for (uint64_t i = threadIdx.x; i < page_bytes; i += blockDim.x) d[i] = s[i];
    }
  }
}

}  // namespace
}  // namespace bb

using namespace bb;

extern "C" {

int bb_gather_pages(const uint8_t* d_pool, size_t n_pool_pages, size_t page_bytes, const uint32_t* d_page_ids,
                    uint32_t n_pages, uint8_t* d_out, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (n_pages == 0 || page_bytes == 0) return BB_OK;
  if (!d_pool || !d_page_ids || !d_out) {
    set_error("gather_pages: null argument");
    return BB_INVALID_ARG;
  }
  int* bad = nullptr;
  BB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&bad), sizeof(int), st));
  BB_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), st));
  const unsigned grid = n_pages < 8u * kNumSMs ? n_pages : 8u * kNumSMs;
  k_gather_pages<<<grid, 256, 0, st>>>(d_pool, page_bytes, d_page_ids, n_pages, n_pool_pages, d_out, bad);
  BB_LAUNCH_CHECK();
  int h_bad = 0;
  BB_CUDA_TRY(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  BB_CUDA_TRY(cudaFreeAsync(bad, st));
  BB_CUDA_TRY(cudaStreamSynchronize(st));
  if (h_bad) {
    set_error("gather_pages: page id out of range");
    return BB_INVALID_ARG;
  }
  return BB_OK;
}

}  // extern "C"
