// Speculative-decoding token-tree payloads: pack the retained
// hidden states of a batch of draft trees into the reference's PackedSd wire
// layout on the device, ready for the BBC1 codec and a PackedSd BBF1 frame.
//
// Reference (/root/reference/proj):
//   pack            src/specdec.cpp:153-165   padding-free [sum N', D] + prefix offsets
//   encode_packed   src/specdec.cpp:192-198   u32 count | u32 offsets[] | f32 payload (LE)
//   decode_packed   src/specdec.cpp:200-220   CorruptOffsets on truncation / length mismatch
//   unpack checks   src/specdec.cpp:167-180   offsets start at 0, non-decreasing
// Here the tree's states are one device tensor [rows, D] with a keep mask per
// row (the pruning result) and the request boundaries in rows; kept rows keep
// their order, as the reference's per-request vectors do.
#include <cub/device/device_scan.cuh>

#include <vector>

#include "bb_common.cuh"
#include "bb_kernels.h"

namespace bb {
namespace {

__global__ void k_keep_u32(const uint8_t* __restrict__ keep, uint64_t n, uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = keep[i] ? 1u : 0u;
}

// header: count | offsets (offset r = kept rows before request r's first row)
__global__ void k_packed_header(const uint32_t* __restrict__ rank, const uint32_t* __restrict__ req_rows,
                                uint32_t n_req, uint64_t n_rows, uint8_t* __restrict__ out) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r <= n_req; r += gridDim.x * blockDim.x) {
    const uint32_t v = req_rows[r] < n_rows ? rank[req_rows[r]] : rank[n_rows];
    uint8_t* p = out + 4 + 4ull * r;
    p[0] = (uint8_t)v, p[1] = (uint8_t)(v >> 8), p[2] = (uint8_t)(v >> 16), p[3] = (uint8_t)(v >> 24);
    if (r == 0) {
      const uint32_t c = n_req + 1;
      out[0] = (uint8_t)c, out[1] = (uint8_t)(c >> 8), out[2] = (uint8_t)(c >> 16), out[3] = (uint8_t)(c >> 24);
    }
  }
}

// one warp per row: kept rows are copied to payload row rank[i] (f32 LE = the
// device's native float layout)
__global__ void k_packed_gather(const float* __restrict__ rows, uint64_t n_rows, uint64_t dim,
                                const uint8_t* __restrict__ keep, const uint32_t* __restrict__ rank,
                                uint8_t* __restrict__ payload) {
  const uint64_t warps = (uint64_t)gridDim.x * blockDim.x / 32;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32; i < n_rows; i += warps) {
    if (!keep[i]) continue;
    const float* s = rows + i * dim;
    uint32_t* d = reinterpret_cast<uint32_t*>(payload) + (uint64_t)rank[i] * dim;  // payload is 4-byte aligned
    for (uint64_t k = threadIdx.x & 31; k < dim; k += 32) d[k] = __float_as_uint(s[k]);
  }
}

int fail(int status, const char* msg) {
  set_error("%s", msg);
  return status;
}

}  // namespace
}  // namespace bb

using namespace bb;

extern "C" {

size_t bb_packed_bound(size_t n_rows, size_t hidden_dim, uint32_t n_requests) {
  return 4 + 4ull * (n_requests + 1) + 4ull * n_rows * hidden_dim;
}

int bb_pack_sd(const float* d_rows, size_t n_rows, size_t hidden_dim, const uint8_t* d_keep,
               const uint32_t* h_request_rows, uint32_t n_requests, uint8_t* d_out, size_t out_cap,
               size_t* out_len, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!out_len || (n_rows && (!d_keep || (hidden_dim && !d_rows))) || !h_request_rows || !d_out)
    return fail(BB_INVALID_ARG, "pack_sd: null argument");
  for (uint32_t r = 0; r < n_requests; r++)
    if (h_request_rows[r + 1] < h_request_rows[r] || h_request_rows[r + 1] > n_rows)
      return fail(BB_INVALID_ARG, "pack_sd: request row ranges must be ordered and in range");
  if (h_request_rows[0] != 0) return fail(BB_INVALID_ARG, "pack_sd: request rows must start at 0");
  // the scratch below comes from the device's stream-ordered pool: keep freed
  // blocks in the pool (the default threshold 0 unmaps them at every synchronize,
  // so each call would map them again through the driver)
  static thread_local int pool_dev = -1;
  int dev = 0;
  BB_CUDA_TRY(cudaGetDevice(&dev));
  if (pool_dev != dev) {
    cudaMemPool_t pool;
    BB_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep_bytes = 64ull << 20;
    BB_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep_bytes));
    pool_dev = dev;
  }
  // kept-row ranks (exclusive scan of the keep mask, n_rows + 1 entries)
  uint32_t *rank = nullptr, *req = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  BB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&rank), 4 * (n_rows + 1), st));
  BB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&req), 4ull * (n_requests + 1), st));
  BB_CUDA_TRY(cudaMemsetAsync(rank, 0, 4 * (n_rows + 1), st));
  BB_CUDA_TRY(cudaMemcpyAsync(req, h_request_rows, 4ull * (n_requests + 1), cudaMemcpyHostToDevice, st));
  if (n_rows) {
    k_keep_u32<<<grid_for(n_rows, 256, 4), 256, 0, st>>>(d_keep, n_rows, rank);
    BB_LAUNCH_CHECK();
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, rank, rank, (int)(n_rows + 1), st);
    BB_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, st));
    BB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, rank, rank, (int)(n_rows + 1), st));
    count_launch(2);
  }
  uint32_t kept = 0;
  BB_CUDA_TRY(cudaMemcpyAsync(&kept, rank + n_rows, 4, cudaMemcpyDeviceToHost, st));
  BB_CUDA_TRY(cudaStreamSynchronize(st));
  const size_t hdr = 4 + 4ull * (n_requests + 1);
  const size_t len = hdr + 4ull * kept * hidden_dim;
  int rc = BB_OK;
  if (len > out_cap) {
    rc = fail(BB_INVALID_ARG, "pack_sd: output buffer too small");
  } else {
    k_packed_header<<<(n_requests + 256) / 256, 256, 0, st>>>(rank, req, n_requests, n_rows, d_out);
    BB_LAUNCH_CHECK();
    if (kept && hidden_dim) {
      k_packed_gather<<<grid_for(32 * n_rows, 256, 8), 256, 0, st>>>(d_rows, n_rows, hidden_dim, d_keep, rank,
                                                                     d_out + hdr);
      BB_LAUNCH_CHECK();
    }
    *out_len = len;
  }
  cudaFreeAsync(rank, st);
  cudaFreeAsync(req, st);
  if (tmp) cudaFreeAsync(tmp, st);
  BB_CUDA_TRY(cudaStreamSynchronize(st));
  return rc;
}

int bb_unpack_sd(const uint8_t* d_in, size_t n, size_t hidden_dim, uint32_t* h_offsets, size_t offsets_cap,
                 uint32_t* n_offsets, size_t* payload_offset, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (n < 4) return fail(BB_CORRUPT_OFFSETS, "packed batch: truncated offset count");
  uint8_t c4[4];
  BB_CUDA_TRY(cudaMemcpyAsync(c4, d_in, 4, cudaMemcpyDeviceToHost, st));
  BB_CUDA_TRY(cudaStreamSynchronize(st));
  const uint32_t count = c4[0] | (c4[1] << 8) | (c4[2] << 16) | ((uint32_t)c4[3] << 24);
  if (count < 1 || n < 4 + 4ull * count) return fail(BB_CORRUPT_OFFSETS, "packed batch: truncated offsets");
  std::vector<uint32_t> off(count);
  BB_CUDA_TRY(cudaMemcpyAsync(off.data(), d_in + 4, 4ull * count, cudaMemcpyDeviceToHost, st));
  BB_CUDA_TRY(cudaStreamSynchronize(st));
  const size_t payload_off = 4 + 4ull * count, payload_bytes = n - payload_off;
  if (payload_bytes % 4 != 0 || payload_bytes / 4 != (size_t)off.back() * hidden_dim)
    return fail(BB_CORRUPT_OFFSETS, "packed batch: payload length does not match offsets");
  if (off.front() != 0) return fail(BB_CORRUPT_OFFSETS, "unpack: offsets must start at 0");
  for (size_t i = 1; i < off.size(); i++)
    if (off[i] < off[i - 1]) return fail(BB_CORRUPT_OFFSETS, "unpack: offsets must be non-decreasing");
  *n_offsets = count;
  if (payload_offset) *payload_offset = payload_off;
  if (h_offsets) {
    if (offsets_cap < count) return fail(BB_INVALID_ARG, "unpack_sd: offsets buffer too small");
    for (uint32_t i = 0; i < count; i++) h_offsets[i] = off[i];
  }
  return BB_OK;
}

}  // extern "C"
