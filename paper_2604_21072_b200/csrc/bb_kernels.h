// Internal (C++) interface between the C-ABI layer and the kernel files.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace bb {

// bb_lanes.cu
int launch_identity_container(const uint8_t* in, uint64_t n, int split, uint8_t* out, cudaStream_t st);
int launch_split(const uint8_t* in, uint64_t count, uint8_t* hi, uint8_t* lo, cudaStream_t st);
int launch_merge(const uint8_t* hi, const uint8_t* lo, uint64_t count, uint8_t* out, cudaStream_t st);
int launch_hist256(const uint8_t* in, uint64_t n, unsigned long long* counts, cudaStream_t st);
// Staged pageable <-> device copies of the host-buffer entry points (bb_hostio.cu):
// 4 MiB chunks through NB pinned buffers, host-side copies split across a worker pool.
struct HostStager {
  static constexpr int NB = 4;
  static constexpr size_t CHUNK = size_t(4) << 20;
  static constexpr size_t SMALL = size_t(1) << 20;  // below: one plain cudaMemcpyAsync
  uint8_t* buf[NB] = {};
  cudaEvent_t ev[NB] = {};
  ~HostStager();
  int ready();
  // stream-ordered: h_src may be reused on return (its bytes are in the pinned buffers or on the device)
  int h2d(uint8_t* d_dst, const uint8_t* h_src, size_t n, cudaStream_t st);
  // returns when h_dst holds the bytes
  int d2h(uint8_t* h_dst, const uint8_t* d_src, size_t n, cudaStream_t st);
};
int launch_differ(const uint8_t* a, const uint8_t* b, uint64_t n, unsigned int* differ, cudaStream_t st);

// Grow-only device scratch owned by a context.
struct Workspace {
  void* base = nullptr;
  size_t cap = 0;
  size_t used = 0;
  int reserve(size_t bytes);  // (re)allocates when too small; resets `used`
  template <class T>
  T* take(size_t count) {
    size_t off = (used + 255) & ~size_t(255);
    used = off + count * sizeof(T);
    return reinterpret_cast<T*>(static_cast<char*>(base) + off);
  }
  ~Workspace();
};

// One zlib stream to produce: input lane and where its blob lands.
struct LaneJob {
  const uint8_t* src;
  uint64_t n;
  int container;  // index into the container list
  int slot;       // 0 = high blob (first), 1 = low blob (second)
};

// One BBC1 container to assemble (header + one or two deflate blobs).
struct ContainerJob {
  uint8_t* dst;
  uint64_t cap;
  uint64_t element_count;
  int split;
};

struct DeflateEngine;
DeflateEngine* deflate_engine_create();
void deflate_engine_destroy(DeflateEngine* e);
// Encodes every lane with zlib-1.3-level-6-exact deflate and assembles the
// containers in place.  Synchronizes `st`; fills container_len (host) and
// container_status (BB_OK / BB_INVALID_ARG when cap is too small).
int deflate_containers(DeflateEngine* e, const std::vector<LaneJob>& lanes,
                       const std::vector<ContainerJob>& containers, cudaStream_t st,
                       uint64_t* container_len, int* container_status);

// One zlib stream to inflate into dst (exactly `expected` bytes on success).
struct InflateJob {
  const uint8_t* src;
  uint64_t n;
  uint8_t* dst;
  uint64_t expected;
  int btype0 = -1;  // BTYPE of the stream's first block when the caller read it (-1: unknown)
};
struct InflateEngine;
InflateEngine* inflate_engine_create();
void inflate_engine_destroy(InflateEngine* e);
// Synchronizes `st`; status[i] = BB_OK or BB_CORRUPT_CONTAINER (uncompress parity).
int inflate_lanes(InflateEngine* e, const std::vector<InflateJob>& jobs, cudaStream_t st, int* status);

// bb_inflate_par.cu: the parallel fast path (ok[i] = 1 when fully validated)
struct ParInflate;
ParInflate* par_inflate_create();
void par_inflate_destroy(ParInflate* p);
// find_dynamic = 0: only stored blocks are located (a fast first pass that fully
// decodes lanes made of stored blocks, e.g. incompressible mantissa planes)
int par_inflate(ParInflate* p, const std::vector<InflateJob>& jobs, cudaStream_t st, int* ok, int find_dynamic);

}  // namespace bb
