/* bbcodec.h -- C ABI of the B200-native BBC1 activation codec.
 *
 * The drop-in boundary for the reference's hot path (BloomBee `beeplan` codec):
 * plain pointers, sizes and a cudaStream_t passed as void*; no C++ or torch
 * types.  The C++ drop-in (include/beeplan/codec.hpp, same declarations as the
 * reference header) and the Python mirror (paper_2604_21072_b200/codec.py)
 * both sit on top of these symbols.
 *
 * Reference interfaces replaced (file:line in /root/reference/proj):
 *   bb_split / bb_split_host        byte_split              src/codec.cpp:86-99,   include/beeplan/codec.hpp:21
 *   bb_merge / bb_merge_host        byte_merge              src/codec.cpp:101-111, include/beeplan/codec.hpp:22
 *   bb_histogram256                 entropy_bits_per_byte's histogram  src/codec.cpp:113-125
 *   bb_backend_encode/_decode       CodecBackend::encode/decode (ids 0 identity, 1 deflate =
 *                                   zlib 1.3 compress2 level 6 / uncompress) src/codec.cpp:17-60
 *   bb_compress / bb_compress_host  serialize_container(compress(stream, backend, split))
 *                                   src/codec.cpp:127-140,163-179
 *   bb_decompress / _host           decompress(parse_container(bytes)) src/codec.cpp:142-161,181-192
 *   bb_compress_batch               the stage hand-off's per-micro-batch compress calls
 *                                   src/wire.cpp:406-411,496-501 (batched into one pipeline)
 *   bb_decompress_batch             the per-micro-batch decompress calls src/wire.cpp:484-491,581-585
 *   bb_pack_sd                      encode_packed(pack(per_request)) src/specdec.cpp:153-165,192-198,
 *                                   include/beeplan/specdec.hpp (PackedBatch)
 *   bb_unpack_sd                    decode_packed's checks src/specdec.cpp:167-180,200-220
 *   bb_gather_pages                 KV offload chunk producer (paged cache -> contiguous chunk);
 *                                   the reference only models it: src/cost_model.cpp:30-47
 *
 * Status codes map 1:1 onto the reference exception types (include/beeplan/errors.hpp:40-56).
 * All device entry points are stream-ordered; those returning a size on the host
 * synchronize the given stream before returning.  A context is not thread-safe;
 * use one per host thread (the C++ shim keeps a thread_local one).
 */
#ifndef BBCODEC_H
#define BBCODEC_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BB_OK = 0,
  BB_ODD_LENGTH = 1,        /* beeplan::OddLength */
  BB_LANE_MISMATCH = 2,     /* beeplan::LaneLengthMismatch */
  BB_BACKEND_UNKNOWN = 3,   /* beeplan::BackendUnknown */
  BB_CORRUPT_CONTAINER = 4, /* beeplan::CorruptContainer */
  BB_ERROR = 5,             /* beeplan::Error */
  BB_CUDA_ERROR = 6,        /* CUDA runtime failure (no reference equivalent) */
  BB_INVALID_ARG = 7,       /* caller error: null pointer / buffer too small */
  BB_CORRUPT_OFFSETS = 8,   /* beeplan::CorruptOffsets */
  BB_DIM_MISMATCH = 9       /* beeplan::DimMismatch */
} bb_status;

enum { BB_BACKEND_IDENTITY = 0, BB_BACKEND_DEFLATE = 1 };
#define BB_CONTAINER_HEADER 31

typedef struct bb_ctx bb_ctx;

#if defined(__GNUC__)
#define BB_API __attribute__((visibility("default")))
#else
#define BB_API
#endif

BB_API const char* bb_last_error(void);
BB_API const char* bb_version(void);

BB_API int bb_ctx_create(bb_ctx** out, int device);
BB_API void bb_ctx_destroy(bb_ctx* ctx);

/* ---- lanes (device) --------------------------------------------------- */
BB_API int bb_split(const uint8_t* d_stream, size_t n_bytes, uint8_t* d_high, uint8_t* d_low, void* stream);
BB_API int bb_merge(const uint8_t* d_high, const uint8_t* d_low, size_t count, uint8_t* d_stream, void* stream);
/* *equal = (d_a[0:n] == d_b[0:n]) on ctx's device (the sink's bit-exact reassembly check,
 * wire.cpp:555-560); synchronizes the stream. */
BB_API int bb_equal(bb_ctx* ctx, const uint8_t* d_a, const uint8_t* d_b, size_t n, int* equal, void* stream);
/* 256 u64 counts, overwritten */
BB_API int bb_histogram256(const uint8_t* d_data, size_t n, uint64_t* d_counts, void* stream);

/* ---- codec (device) ---------------------------------------------------- */
/* Upper bound on the serialized container size. */
BB_API size_t bb_compress_bound(size_t n_bytes, int backend, int split);
/* serialize_container(compress(d_in[0:n], backend, split)) into d_out. */
BB_API int bb_compress(bb_ctx* ctx, const uint8_t* d_in, size_t n, int backend, int split, uint8_t* d_out,
                size_t out_cap, size_t* out_len, void* stream);
/* decompress(parse_container(d_in[0:n])) into d_out; *out_len = decoded bytes.
 * With d_out == NULL only validates the header and reports the decoded size. */
BB_API int bb_decompress(bb_ctx* ctx, const uint8_t* d_in, size_t n, uint8_t* d_out, size_t out_cap,
                  size_t* out_len, void* stream);
/* Many tensors (e.g. the M micro-batches of one step) through one pipeline.
 * out_len[i] / status[i] per item; returns the first non-OK status. */
BB_API int bb_compress_batch(bb_ctx* ctx, int count, const uint8_t* const* d_in, const size_t* n, int backend,
                      int split, uint8_t* const* d_out, const size_t* out_cap, size_t* out_len,
                      int* status, void* stream);
BB_API int bb_decompress_batch(bb_ctx* ctx, int count, const uint8_t* const* d_in, const size_t* n,
                        uint8_t* const* d_out, const size_t* out_cap, size_t* out_len, int* status,
                        void* stream);

/* ---- backend level (one lane; CodecBackend::encode / decode) ----------- */
BB_API size_t bb_backend_bound(int backend, size_t n);
BB_API int bb_backend_encode(bb_ctx* ctx, int backend, const uint8_t* d_in, size_t n, uint8_t* d_out,
                      size_t out_cap, size_t* out_len, void* stream);
BB_API int bb_backend_decode(bb_ctx* ctx, int backend, const uint8_t* d_in, size_t n, size_t expected,
                      uint8_t* d_out, void* stream);

/* ---- host buffers (the reference-facing Bytes -> Bytes calls) ----------
 * H2D copy, the device pipeline, D2H copy; synchronous. */
BB_API int bb_compress_host(bb_ctx* ctx, const uint8_t* h_in, size_t n, int backend, int split,
                     uint8_t* h_out, size_t out_cap, size_t* out_len);
BB_API int bb_decompress_host(bb_ctx* ctx, const uint8_t* h_in, size_t n, uint8_t* h_out, size_t out_cap,
                       size_t* out_len);
BB_API int bb_backend_encode_host(bb_ctx* ctx, int backend, const uint8_t* h_in, size_t n, uint8_t* h_out,
                           size_t out_cap, size_t* out_len);
BB_API int bb_backend_decode_host(bb_ctx* ctx, int backend, const uint8_t* h_in, size_t n, size_t expected,
                           uint8_t* h_out);
BB_API int bb_split_host(bb_ctx* ctx, const uint8_t* h_stream, size_t n_bytes, uint8_t* h_high, uint8_t* h_low);
BB_API int bb_merge_host(bb_ctx* ctx, const uint8_t* h_high, const uint8_t* h_low, size_t count,
                  uint8_t* h_stream);
BB_API int bb_histogram256_host(bb_ctx* ctx, const uint8_t* h_data, size_t n, uint64_t* h_counts);

/* ---- speculative-decoding payloads (PackedSd frames) -------------------- */
/* Wire image: u32 count (= n_requests + 1) | u32 offsets[count] | f32 payload, LE. */
BB_API size_t bb_packed_bound(size_t n_rows, size_t hidden_dim, uint32_t n_requests);
/* d_rows: [n_rows, hidden_dim] f32 token-tree states; d_keep[n_rows] != 0 keeps a row;
 * h_request_rows[n_requests + 1]: request r owns rows [h_request_rows[r], h_request_rows[r+1]).
 * Writes encode_packed(pack(kept rows per request)) to d_out; synchronizes the stream. */
BB_API int bb_pack_sd(const float* d_rows, size_t n_rows, size_t hidden_dim, const uint8_t* d_keep,
                      const uint32_t* h_request_rows, uint32_t n_requests, uint8_t* d_out, size_t out_cap,
                      size_t* out_len, void* stream);
/* Validates a packed image in HBM (decode_packed's CorruptOffsets rules) and returns its
 * offsets (h_offsets may be NULL to query *n_offsets) and the payload's byte offset. */
BB_API int bb_unpack_sd(const uint8_t* d_in, size_t n, size_t hidden_dim, uint32_t* h_offsets,
                        size_t offsets_cap, uint32_t* n_offsets, size_t* payload_offset, void* stream);

/* ---- KV-cache offload chunks ------------------------------------------ */
/* out[p] = pool[page_ids[p]] for p < n_pages (page_bytes each; page_ids in device memory).
 * BB_INVALID_ARG when an id is >= n_pool_pages.  Synchronizes the stream. */
BB_API int bb_gather_pages(const uint8_t* d_pool, size_t n_pool_pages, size_t page_bytes,
                           const uint32_t* d_page_ids, uint32_t n_pages, uint8_t* d_out, void* stream);

/* ---- multi-GPU hand-off ------------------------------------------------ */
/* Lets kernels running on `device` read / write memory of `peer` over NVLink (the
 * codec then writes its containers straight into the next stage's HBM). */
BB_API int bb_enable_peer_access(int device, int peer);
/* CUDA IPC: export a device pointer as (64-byte handle of its allocation, offset); import it
 * into `device`'s context (the stage that writes into it); close with the returned base. */
BB_API int bb_ipc_export(const void* d_ptr, void* handle64, size_t* offset);
BB_API int bb_ipc_import(int device, const void* handle64, size_t offset, void** d_ptr, void** d_base);
BB_API int bb_ipc_close(void* d_base);
/* stream-ordered host -> device copy (e.g. frame headers into a peer's inbox) */
BB_API int bb_copy_h2d(void* d_dst, const void* h_src, size_t n, void* stream);

/* ---- instrumentation ---------------------------------------------------- */
/* Number of kernels this library launched (process-wide, monotonic). */
BB_API uint64_t bb_kernel_launches(void);
/* Per-stage CUDA-event timing of the codec pipelines (off by default). */
BB_API void bb_stage_timing(int enable);
/* JSON {"stage": {"ms": total, "count": calls}, ...}; reset != 0 clears. */
BB_API const char* bb_stage_report(int reset);

#ifdef __cplusplus
}
#endif
#endif
