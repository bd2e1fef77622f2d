// C-ABI layer (include/bbcodec.h): argument checks, container header parsing,
// error mapping, workspace management and dispatch onto the sm_100a kernels.
//
// Container semantics follow the reference exactly (/root/reference/proj):
//   compress            src/codec.cpp:163-179 (backend lookup, then OddLength)
//   serialize_container src/codec.cpp:127-140
//   parse_container     src/codec.cpp:142-161 (truncated / magic / version / lengths)
//   decompress          src/codec.cpp:181-192 (split: decode(high,N), decode(low,N), merge;
//                                              raw: low blob must be empty, decode(high, 2N))
//   deflate decode guard src/codec.cpp:30-31 (expected > blob*1040 + 1024 -> CorruptContainer)
//   identity decode      src/codec.cpp:45-47 (size mismatch -> CorruptContainer)
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cuda.h>

#include <cstring>

#include "bb_common.cuh"
#include "bb_kernels.h"

namespace bb {

std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_stage_timing{0};

bool debug_sync() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BB_DEBUG_SYNC");
    v = (e && *e == '1') ? 1 : 0;
  }
  return v == 1;
}

namespace {
struct StageAcc {
  double ms = 0;
  uint64_t count = 0;
};
std::mutex g_stage_mu;
std::map<std::string, StageAcc> g_stage_acc;
std::string g_stage_report;
}  // namespace

void StageTimer::finish() {
  if (!on || n == 0) return;
  cudaEvent_t end;
  cudaEventCreate(&end);
  cudaEventRecord(end, st);
  cudaEventSynchronize(end);
  std::lock_guard<std::mutex> lk(g_stage_mu);
  for (int i = 0; i < n; i++) {
    float ms = 0;
    cudaEventElapsedTime(&ms, ev[i], i + 1 < n ? ev[i + 1] : end);
    StageAcc& a = g_stage_acc[names[i]];
    a.ms += ms;
    a.count += 1;
    cudaEventDestroy(ev[i]);
  }
  cudaEventDestroy(end);
  n = 0;
}
static thread_local std::string t_err;

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
}

int Workspace::reserve(size_t bytes) {
  used = 0;
  if (bytes <= cap) return BB_OK;
  if (base) cudaFree(base);
  base = nullptr;
  cap = 0;
  size_t want = bytes + bytes / 8 + (1u << 20);
  BB_CUDA_TRY(cudaMalloc(&base, want));
  cap = want;
  return BB_OK;
}

Workspace::~Workspace() {
  if (base) cudaFree(base);
}

static int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  return status;
}

}  // namespace bb

using namespace bb;

struct bb_ctx {
  int device = 0;
  cudaStream_t own = nullptr;  // stream for the host-buffer entry points
  Workspace ws;                // lanes / inflate scratch
  Workspace host_in, host_out; // device copies for the *_host calls
  DeflateEngine* deflate = nullptr;
  InflateEngine* inflate = nullptr;
  HostStager io;                   // pageable host buffers of the *_host entry points
  unsigned int* d_flag = nullptr;  // bb_equal's result word (device) and its pinned host copy
  unsigned int* h_flag = nullptr;
};

namespace {

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Selects a device for the duration of an entry point and restores the caller's
// current device on exit (a torchrun worker bound to GPU k must stay on GPU k).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};
#define BB_DEVICE_GUARD(dev)                                                                  \
  DeviceGuard bb_dg_(dev);                                                                    \
  if (bb_dg_.err != cudaSuccess)                                                              \
    return bb::fail(BB_CUDA_ERROR, "cudaSetDevice(%d): %s", (int)(dev), cudaGetErrorString(bb_dg_.err))

uint64_t rd_u64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; i++) v |= (uint64_t)p[i] << (8 * i);
  return v;
}

struct Header {
  int backend, split;
  uint64_t count, hl, ll;
};

// parse_container (codec.cpp:142-161) on a host copy of the 31-byte header
int parse_header(const uint8_t* h, uint64_t n, Header* c) {
  if (n < BB_CONTAINER_HEADER) return fail(BB_CORRUPT_CONTAINER, "container: truncated header");
  if (std::memcmp(h, "BBC1", 4) != 0) return fail(BB_CORRUPT_CONTAINER, "container: bad magic");
  if (h[4] != 1) return fail(BB_CORRUPT_CONTAINER, "container: unsupported version %u", h[4]);
  c->backend = h[5];
  c->split = h[6] & 1;
  c->count = rd_u64(h + 7);
  c->hl = rd_u64(h + 15);
  c->ll = rd_u64(h + 23);
  uint64_t avail = n - BB_CONTAINER_HEADER;
  if (c->hl > avail || c->ll > avail - c->hl || c->hl + c->ll != avail)
    return fail(BB_CORRUPT_CONTAINER, "container: blob lengths do not match the payload");
  return BB_OK;
}

// backend.decode(blob, expected) preconditions that need no decoding
int lane_precheck(int backend, uint64_t blob, uint64_t expected) {
  if (backend == BB_BACKEND_IDENTITY) {
    if (blob != expected)
      return fail(BB_CORRUPT_CONTAINER, "identity: blob length does not match the declared size");
    return BB_OK;
  }
  if (expected > blob * 1040 + 1024)
    return fail(BB_CORRUPT_CONTAINER, "deflate: declared size implausible for the blob");
  return BB_OK;
}

int check_backend(int backend) {
  if (backend != BB_BACKEND_IDENTITY && backend != BB_BACKEND_DEFLATE)
    return fail(BB_BACKEND_UNKNOWN, "codec backend id %d is not registered", backend);
  return BB_OK;
}

// Validates one container and returns its decoded size.
int plan_decode(const Header& c, uint64_t* decoded) {
  int rc = check_backend(c.backend);
  if (rc) return rc;
  if (c.split) {
    if ((rc = lane_precheck(c.backend, c.hl, c.count))) return rc;
    if ((rc = lane_precheck(c.backend, c.ll, c.count))) return rc;
    *decoded = 2 * c.count;
  } else {
    if (c.ll != 0) return fail(BB_CORRUPT_CONTAINER, "container: raw mode must have an empty low blob");
    uint64_t expected = c.count * 2;  // size_t arithmetic, as in the reference
    if ((rc = lane_precheck(c.backend, c.hl, expected))) return rc;
    *decoded = expected;
  }
  return BB_OK;
}

}  // namespace

extern "C" {

const char* bb_last_error(void) { return t_err.c_str(); }
const char* bb_version(void) { return "bbcodec-b200 0.1 (sm_100a)"; }
int bb_enable_peer_access(int device, int peer) {
  int cur = 0;
  BB_CUDA_TRY(cudaGetDevice(&cur));
  BB_CUDA_TRY(cudaSetDevice(device));
  int can = 0;
  cudaError_t e = cudaDeviceCanAccessPeer(&can, device, peer);
  if (e == cudaSuccess && can) {
    e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
      cudaGetLastError();
      e = cudaSuccess;
    }
  } else if (e == cudaSuccess) {
    e = cudaErrorPeerAccessUnsupported;
  }
  cudaSetDevice(cur);
  if (e != cudaSuccess) {
    bb::set_error("peer access %d -> %d: %s", device, peer, cudaGetErrorString(e));
    return BB_CUDA_ERROR;
  }
  return BB_OK;
}

// CUDA IPC for the direct hand-off: a device pointer (possibly inside a larger
// allocation of a caching allocator) is exported as (handle of its allocation,
// offset) and imported into the *caller's* device context, so kernels of this
// stage can write the next stage's HBM over NVLink.
int bb_ipc_export(const void* d_ptr, void* handle64, size_t* offset) {
  if (!d_ptr || !handle64 || !offset) {
    bb::set_error("ipc_export: null argument");
    return BB_INVALID_ARG;
  }
  // the driver's cuMemGetAddressRange, fetched through the runtime (no libcuda link
  // dependency, so the library still loads on machines without a driver)
  typedef CUresult (*GetRange)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    BB_CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) {
      bb::set_error("ipc_export: cuMemGetAddressRange unavailable");
      return BB_CUDA_ERROR;
    }
    get_range = reinterpret_cast<GetRange>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS) {
    bb::set_error("ipc_export: cuMemGetAddressRange failed");
    return BB_CUDA_ERROR;
  }
  BB_CUDA_TRY(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle64), reinterpret_cast<void*>(base)));
  *offset = reinterpret_cast<uintptr_t>(d_ptr) - (uintptr_t)base;
  return BB_OK;
}

int bb_ipc_import(int device, const void* handle64, size_t offset, void** d_ptr, void** d_base) {
  if (!handle64 || !d_ptr || !d_base) {
    bb::set_error("ipc_import: null argument");
    return BB_INVALID_ARG;
  }
  BB_DEVICE_GUARD(device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof h);
  void* base = nullptr;
  BB_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *d_base = base;
  *d_ptr = static_cast<char*>(base) + offset;
  return BB_OK;
}

int bb_ipc_close(void* d_base) {
  BB_CUDA_TRY(cudaIpcCloseMemHandle(d_base));
  return BB_OK;
}

int bb_copy_h2d(void* d_dst, const void* h_src, size_t n, void* stream) {
  BB_CUDA_TRY(cudaMemcpyAsync(d_dst, h_src, n, cudaMemcpyHostToDevice, reinterpret_cast<cudaStream_t>(stream)));
  return BB_OK;
}

uint64_t bb_kernel_launches(void) { return g_launches.load(); }

void bb_stage_timing(int enable) { g_stage_timing.store(enable); }

const char* bb_stage_report(int reset) {
  std::lock_guard<std::mutex> lk(g_stage_mu);
  std::string r = "{";
  bool first = true;
  for (const auto& [k, v] : g_stage_acc) {
    char buf[256];
    snprintf(buf, sizeof buf, "%s\"%s\": {\"ms\": %.6f, \"count\": %llu}", first ? "" : ", ", k.c_str(), v.ms,
             (unsigned long long)v.count);
    r += buf;
    first = false;
  }
  r += "}";
  g_stage_report = r;
  if (reset) g_stage_acc.clear();
  return g_stage_report.c_str();
}

int bb_ctx_create(bb_ctx** out, int device) {
  if (!out) return fail(BB_INVALID_ARG, "null ctx pointer");
  BB_DEVICE_GUARD(device);
  bb_ctx* c = new bb_ctx();
  c->device = device;
  cudaError_t e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return fail(BB_CUDA_ERROR, "cudaStreamCreate: %s", cudaGetErrorString(e));
  }
  c->deflate = deflate_engine_create();
  c->inflate = inflate_engine_create();
  *out = c;
  return BB_OK;
}

void bb_ctx_destroy(bb_ctx* c) {
  if (!c) return;
  DeviceGuard g(c->device);
  deflate_engine_destroy(c->deflate);
  inflate_engine_destroy(c->inflate);
  if (c->own) cudaStreamDestroy(c->own);
  if (c->d_flag) cudaFree(c->d_flag);
  if (c->h_flag) cudaFreeHost(c->h_flag);
  delete c;
}

int bb_split(const uint8_t* d_stream, size_t n, uint8_t* d_high, uint8_t* d_low, void* stream) {
  if (n % 2) return fail(BB_ODD_LENGTH, "byte_split: stream length must be even, got %zu", n);
  if (n && (!d_stream || !d_high || !d_low)) return fail(BB_INVALID_ARG, "null pointer");
  return launch_split(d_stream, n / 2, d_high, d_low, S(stream));
}

int bb_merge(const uint8_t* d_high, const uint8_t* d_low, size_t count, uint8_t* d_out, void* stream) {
  if (count && (!d_high || !d_low || !d_out)) return fail(BB_INVALID_ARG, "null pointer");
  return launch_merge(d_high, d_low, count, d_out, S(stream));
}

int bb_equal(bb_ctx* ctx, const uint8_t* d_a, const uint8_t* d_b, size_t n, int* equal, void* stream) {
  if (!ctx || !equal || (n && (!d_a || !d_b))) return fail(BB_INVALID_ARG, "null pointer");
  BB_DEVICE_GUARD(ctx->device);
  if (!ctx->h_flag)
    BB_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_flag), sizeof(unsigned int), cudaHostAllocDefault));
  if (!ctx->d_flag) BB_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&ctx->d_flag), sizeof(unsigned int)));
  int rc = launch_differ(d_a, d_b, n, ctx->d_flag, S(stream));
  if (rc) return rc;
  BB_CUDA_TRY(cudaMemcpyAsync(ctx->h_flag, ctx->d_flag, sizeof(unsigned int), cudaMemcpyDeviceToHost, S(stream)));
  BB_CUDA_TRY(cudaStreamSynchronize(S(stream)));
  *equal = *ctx->h_flag == 0;
  return BB_OK;
}

int bb_histogram256(const uint8_t* d, size_t n, uint64_t* d_counts, void* stream) {
  if (!d_counts || (n && !d)) return fail(BB_INVALID_ARG, "null pointer");
  return launch_hist256(d, n, reinterpret_cast<unsigned long long*>(d_counts), S(stream));
}

size_t bb_backend_bound(int backend, size_t n) {
  // zlib compressBound (compress.c) for deflate; identity is a copy
  return backend == BB_BACKEND_DEFLATE ? n + (n >> 12) + (n >> 14) + (n >> 25) + 13 : n;
}

size_t bb_compress_bound(size_t n, int backend, int split) {
  if (split) return BB_CONTAINER_HEADER + 2 * bb_backend_bound(backend, n / 2);
  return BB_CONTAINER_HEADER + bb_backend_bound(backend, n);
}

int bb_compress_batch(bb_ctx* ctx, int count, const uint8_t* const* d_in, const size_t* n, int backend,
                      int split, uint8_t* const* d_out, const size_t* out_cap, size_t* out_len,
                      int* status, void* stream) {
  if (!ctx || count < 0) return fail(BB_INVALID_ARG, "bad arguments");
  BB_DEVICE_GUARD(ctx->device);  // the stream and the engines belong to ctx->device
  cudaStream_t st = S(stream);
  int first = BB_OK;
  int rc = check_backend(backend);
  std::vector<int> st_local(count > 0 ? count : 1);
  int* stv = status ? status : st_local.data();
  for (int i = 0; i < count; i++) {
    stv[i] = rc;
    out_len[i] = 0;
  }
  if (rc) return rc;
  std::vector<LaneJob> lanes;
  std::vector<ContainerJob> cons;
  std::vector<int> con_item;
  size_t lane_bytes = 0;
  for (int i = 0; i < count; i++) {
    if (n[i] % 2) {
      stv[i] = fail(BB_ODD_LENGTH, "compress: FP16 stream length must be even");
      continue;
    }
    if (backend == BB_BACKEND_DEFLATE && split) lane_bytes += ((n[i] + 255) & ~size_t(255)) + 256;
  }
  if (lane_bytes) {
    int r = ctx->ws.reserve(lane_bytes + 4096);
    if (r) return r;
  }
  for (int i = 0; i < count; i++) {
    if (stv[i]) continue;
    if (backend == BB_BACKEND_IDENTITY) {
      if (out_cap[i] < BB_CONTAINER_HEADER + n[i]) {
        stv[i] = fail(BB_INVALID_ARG, "output buffer too small");
        continue;
      }
      int r = launch_identity_container(d_in[i], n[i], split, d_out[i], st);
      if (r) return r;
      out_len[i] = BB_CONTAINER_HEADER + n[i];
      continue;
    }
    int ci = (int)cons.size();
    cons.push_back(ContainerJob{d_out[i], out_cap[i], n[i] / 2, split});
    con_item.push_back(i);
    if (split) {
      uint64_t N = n[i] / 2;
      uint8_t* hi = ctx->ws.take<uint8_t>(N + 16);
      uint8_t* lo = ctx->ws.take<uint8_t>(N + 16);
      int r = launch_split(d_in[i], N, hi, lo, st);
      if (r) return r;
      lanes.push_back(LaneJob{hi, N, ci, 0});
      lanes.push_back(LaneJob{lo, N, ci, 1});
    } else {
      lanes.push_back(LaneJob{d_in[i], n[i], ci, 0});
    }
  }
  if (!cons.empty()) {
    std::vector<uint64_t> clen(cons.size());
    std::vector<int> cst(cons.size());
    int r = deflate_containers(ctx->deflate, lanes, cons, st, clen.data(), cst.data());
    if (r) return r;
    for (size_t k = 0; k < cons.size(); k++) {
      int i = con_item[k];
      stv[i] = cst[k];
      out_len[i] = clen[k];
      if (cst[k]) fail(cst[k], "output buffer too small for the compressed container");
    }
  }
  for (int i = 0; i < count; i++)
    if (stv[i] && !first) first = stv[i];
  return first;
}

int bb_compress(bb_ctx* ctx, const uint8_t* d_in, size_t n, int backend, int split, uint8_t* d_out,
                size_t out_cap, size_t* out_len, void* stream) {
  int status = 0;
  size_t len = 0;
  int rc = bb_compress_batch(ctx, 1, &d_in, &n, backend, split, &d_out, &out_cap, &len, &status, stream);
  if (out_len) *out_len = len;
  return rc;
}

int bb_decompress_batch(bb_ctx* ctx, int count, const uint8_t* const* d_in, const size_t* n,
                        uint8_t* const* d_out, const size_t* out_cap, size_t* out_len, int* status,
                        void* stream) {
  if (!ctx || count < 0) return fail(BB_INVALID_ARG, "bad arguments");
  BB_DEVICE_GUARD(ctx->device);  // the stream and the engines belong to ctx->device
  cudaStream_t st = S(stream);
  std::vector<int> st_local(count > 0 ? count : 1);
  int* stv = status ? status : st_local.data();
  // 1. headers to the host (parse_container runs host-side on 31 bytes), with the first bytes of the
  //    high blob: its first block's BTYPE routes dynamic lanes straight to the full candidate search
  constexpr size_t HB = BB_CONTAINER_HEADER + 3, HS = 40;  // bytes read / host stride per item
  std::vector<uint8_t> hdr((size_t)count * HS + 1);
  for (int i = 0; i < count; i++) {
    out_len[i] = 0;
    if (n[i] >= BB_CONTAINER_HEADER)
      BB_CUDA_TRY(cudaMemcpyAsync(hdr.data() + (size_t)i * HS, d_in[i], std::min<size_t>(n[i], HB),
                                  cudaMemcpyDeviceToHost, st));
  }
  BB_CUDA_TRY(cudaStreamSynchronize(st));
  std::vector<Header> H(count > 0 ? count : 1);
  std::vector<uint64_t> dec(count > 0 ? count : 1, 0);
  size_t scratch = 0;
  for (int i = 0; i < count; i++) {
    stv[i] = parse_header(hdr.data() + (size_t)i * HS, n[i], &H[i]);
    if (!stv[i]) stv[i] = plan_decode(H[i], &dec[i]);
    if (!stv[i]) {
      out_len[i] = dec[i];
      if (d_out && d_out[i] && out_cap[i] < dec[i]) stv[i] = fail(BB_INVALID_ARG, "output buffer too small");
      if (!stv[i] && H[i].backend == BB_BACKEND_DEFLATE && H[i].split)
        scratch += 2 * (((H[i].count + 255) & ~uint64_t(255)) + 256);
    }
  }
  if (!d_out) {
    int first = BB_OK;
    for (int i = 0; i < count; i++)
      if (stv[i] && !first) first = stv[i];
    return first;
  }
  if (scratch) {
    int r = ctx->ws.reserve(scratch + 4096);
    if (r) return r;
  }
  // 2. decode
  std::vector<InflateJob> jobs;
  std::vector<int> job_item;
  struct MergeTask {
    int item;
    uint8_t *hi, *lo;
  };
  std::vector<MergeTask> merges;
  for (int i = 0; i < count; i++) {
    if (stv[i]) continue;
    const Header& c = H[i];
    const uint8_t* hb = d_in[i] + BB_CONTAINER_HEADER;
    const uint8_t* lb = hb + c.hl;
    if (c.backend == BB_BACKEND_IDENTITY) {
      if (c.split) {
        int r = launch_merge(hb, lb, c.count, d_out[i], st);
        if (r) return r;
      } else if (dec[i]) {
        BB_CUDA_TRY(cudaMemcpyAsync(d_out[i], hb, dec[i], cudaMemcpyDeviceToDevice, st));
      }
      continue;
    }
    if (c.split) {
      uint8_t* hi = ctx->ws.take<uint8_t>(c.count + 16);
      uint8_t* lo = ctx->ws.take<uint8_t>(c.count + 16);
      const uint8_t* h3 = hdr.data() + (size_t)i * HS + BB_CONTAINER_HEADER;  // zlib CMF, FLG, first block
      const int bt = (c.hl >= 3 && n[i] >= HB) ? (h3[2] >> 1) & 3 : -1;
      jobs.push_back(InflateJob{hb, c.hl, hi, c.count, bt});
      job_item.push_back(i);
      jobs.push_back(InflateJob{lb, c.ll, lo, c.count});
      job_item.push_back(i);
      merges.push_back(MergeTask{i, hi, lo});
    } else {
      jobs.push_back(InflateJob{hb, c.hl, d_out[i], dec[i]});
      job_item.push_back(i);
    }
  }
  if (!jobs.empty()) {
    std::vector<int> js(jobs.size());
    int r = inflate_lanes(ctx->inflate, jobs, st, js.data());
    if (r) return r;
    for (size_t k = 0; k < jobs.size(); k++)
      if (js[k] && !stv[job_item[k]])
        stv[job_item[k]] = fail(js[k], "deflate: blob does not inflate to the declared size");
    for (const MergeTask& m : merges) {
      if (stv[m.item]) continue;
      int r2 = launch_merge(m.hi, m.lo, H[m.item].count, d_out[m.item], st);
      if (r2) return r2;
    }
  }
  int first = BB_OK;
  for (int i = 0; i < count; i++) {
    if (stv[i]) out_len[i] = 0;
    if (stv[i] && !first) first = stv[i];
  }
  return first;
}

int bb_decompress(bb_ctx* ctx, const uint8_t* d_in, size_t n, uint8_t* d_out, size_t out_cap,
                  size_t* out_len, void* stream) {
  int status = 0;
  size_t len = 0;
  uint8_t* outs[1] = {d_out};
  int rc = bb_decompress_batch(ctx, 1, &d_in, &n, d_out ? outs : nullptr, &out_cap, &len, &status, stream);
  if (out_len) *out_len = len;
  return rc;
}

int bb_backend_encode(bb_ctx* ctx, int backend, const uint8_t* d_in, size_t n, uint8_t* d_out,
                      size_t out_cap, size_t* out_len, void* stream) {
  int rc = check_backend(backend);
  if (rc) return rc;
  if (!ctx) return fail(BB_INVALID_ARG, "null ctx");
  BB_DEVICE_GUARD(ctx->device);  // the stream and the engines belong to ctx->device
  cudaStream_t st = S(stream);
  if (backend == BB_BACKEND_IDENTITY) {
    if (out_cap < n) return fail(BB_INVALID_ARG, "output buffer too small");
    if (n) BB_CUDA_TRY(cudaMemcpyAsync(d_out, d_in, n, cudaMemcpyDeviceToDevice, st));
    *out_len = n;
    return BB_OK;
  }
  // a "container" with no header: the blob goes straight to d_out
  std::vector<LaneJob> lanes{LaneJob{d_in, n, 0, 0}};
  std::vector<ContainerJob> cons{ContainerJob{d_out, out_cap, n, -1}};
  uint64_t len = 0;
  int cst = 0;
  rc = deflate_containers(ctx->deflate, lanes, cons, st, &len, &cst);
  if (rc) return rc;
  if (cst) return fail(cst, "output buffer too small");
  *out_len = len;
  return BB_OK;
}

int bb_backend_decode(bb_ctx* ctx, int backend, const uint8_t* d_in, size_t n, size_t expected,
                      uint8_t* d_out, void* stream) {
  int rc = check_backend(backend);
  if (rc) return rc;
  if ((rc = lane_precheck(backend, n, expected))) return rc;
  if (!ctx) return fail(BB_INVALID_ARG, "null ctx");
  BB_DEVICE_GUARD(ctx->device);
  cudaStream_t st = S(stream);
  if (backend == BB_BACKEND_IDENTITY) {
    if (n) BB_CUDA_TRY(cudaMemcpyAsync(d_out, d_in, n, cudaMemcpyDeviceToDevice, st));
    return BB_OK;
  }
  std::vector<InflateJob> jobs{InflateJob{d_in, n, d_out, expected}};
  int js = 0;
  rc = inflate_lanes(ctx->inflate, jobs, st, &js);
  if (rc) return rc;
  if (js) return fail(js, "deflate: blob does not inflate to the declared size");
  return BB_OK;
}

// ---- host-buffer entry points --------------------------------------------

static int to_device(bb_ctx* c, Workspace& w, const uint8_t* h, size_t n, uint8_t** d) {
  int r = w.reserve(n + 64);
  if (r) return r;
  *d = static_cast<uint8_t*>(w.base);
  return c->io.h2d(*d, h, n, c->own);
}

int bb_compress_host(bb_ctx* c, const uint8_t* h_in, size_t n, int backend, int split, uint8_t* h_out,
                     size_t out_cap, size_t* out_len) {
  if (!c) return fail(BB_INVALID_ARG, "null ctx");
  BB_DEVICE_GUARD(c->device);
  uint8_t *din, *dout;
  int rc = to_device(c, c->host_in, h_in, n, &din);
  if (rc) return rc;
  size_t bound = bb_compress_bound(n, backend, split);
  if ((rc = c->host_out.reserve(bound + 64))) return rc;
  dout = static_cast<uint8_t*>(c->host_out.base);
  size_t len = 0;
  rc = bb_compress(c, din, n, backend, split, dout, bound, &len, c->own);
  if (rc) return rc;
  if (len > out_cap) return fail(BB_INVALID_ARG, "output buffer too small");
  if (len && (rc = c->io.d2h(h_out, dout, len, c->own))) return rc;
  BB_CUDA_TRY(cudaStreamSynchronize(c->own));
  *out_len = len;
  return BB_OK;
}

int bb_decompress_host(bb_ctx* c, const uint8_t* h_in, size_t n, uint8_t* h_out, size_t out_cap,
                       size_t* out_len) {
  if (!c) return fail(BB_INVALID_ARG, "null ctx");
  if (!h_in && n) return fail(BB_INVALID_ARG, "null input");
  // parse_container + the decode plan run on the host copy: a size query uploads nothing
  Header hd;
  uint64_t need = 0;
  int rc = parse_header(h_in, n, &hd);
  if (!rc) rc = plan_decode(hd, &need);
  if (rc) return rc;
  if (!h_out) {
    *out_len = need;
    return BB_OK;
  }
  BB_DEVICE_GUARD(c->device);
  uint8_t* din;
  if ((rc = to_device(c, c->host_in, h_in, n, &din))) return rc;
  if (need > out_cap) return fail(BB_INVALID_ARG, "output buffer too small");
  if ((rc = c->host_out.reserve(need + 64))) return rc;
  uint8_t* dout = static_cast<uint8_t*>(c->host_out.base);
  size_t len = 0;
  rc = bb_decompress(c, din, n, dout, need, &len, c->own);
  if (rc) return rc;
  if (len && (rc = c->io.d2h(h_out, dout, len, c->own))) return rc;
  BB_CUDA_TRY(cudaStreamSynchronize(c->own));
  *out_len = len;
  return BB_OK;
}

int bb_backend_encode_host(bb_ctx* c, int backend, const uint8_t* h_in, size_t n, uint8_t* h_out,
                           size_t out_cap, size_t* out_len) {
  if (!c) return fail(BB_INVALID_ARG, "null ctx");
  int rc = check_backend(backend);
  if (rc) return rc;
  BB_DEVICE_GUARD(c->device);
  uint8_t* din;
  if ((rc = to_device(c, c->host_in, h_in, n, &din))) return rc;
  size_t bound = bb_backend_bound(backend, n);
  if ((rc = c->host_out.reserve(bound + 64))) return rc;
  uint8_t* dout = static_cast<uint8_t*>(c->host_out.base);
  size_t len = 0;
  if ((rc = bb_backend_encode(c, backend, din, n, dout, bound, &len, c->own))) return rc;
  if (len > out_cap) return fail(BB_INVALID_ARG, "output buffer too small");
  if (len && (rc = c->io.d2h(h_out, dout, len, c->own))) return rc;
  BB_CUDA_TRY(cudaStreamSynchronize(c->own));
  *out_len = len;
  return BB_OK;
}

int bb_backend_decode_host(bb_ctx* c, int backend, const uint8_t* h_in, size_t n, size_t expected,
                           uint8_t* h_out) {
  if (!c) return fail(BB_INVALID_ARG, "null ctx");
  int rc = check_backend(backend);
  if (rc) return rc;
  if ((rc = lane_precheck(backend, n, expected))) return rc;
  BB_DEVICE_GUARD(c->device);
  uint8_t* din;
  if ((rc = to_device(c, c->host_in, h_in, n, &din))) return rc;
  if ((rc = c->host_out.reserve(expected + 64))) return rc;
  uint8_t* dout = static_cast<uint8_t*>(c->host_out.base);
  if ((rc = bb_backend_decode(c, backend, din, n, expected, dout, c->own))) return rc;
  if (expected && (rc = c->io.d2h(h_out, dout, expected, c->own))) return rc;
  BB_CUDA_TRY(cudaStreamSynchronize(c->own));
  return BB_OK;
}

int bb_split_host(bb_ctx* c, const uint8_t* h_stream, size_t n, uint8_t* h_high, uint8_t* h_low) {
  if (!c) return fail(BB_INVALID_ARG, "null ctx");
  if (n % 2) return fail(BB_ODD_LENGTH, "byte_split: stream length must be even, got %zu", n);
  BB_DEVICE_GUARD(c->device);
  uint8_t* din;
  int rc = to_device(c, c->host_in, h_stream, n, &din);
  if (rc) return rc;
  if ((rc = c->host_out.reserve(n + 64))) return rc;
  uint8_t* hi = static_cast<uint8_t*>(c->host_out.base);
  uint8_t* lo = hi + ((n / 2 + 15) & ~size_t(15));
  if ((rc = launch_split(din, n / 2, hi, lo, c->own))) return rc;
  if (n) {
    BB_CUDA_TRY(cudaMemcpyAsync(h_high, hi, n / 2, cudaMemcpyDeviceToHost, c->own));
    BB_CUDA_TRY(cudaMemcpyAsync(h_low, lo, n / 2, cudaMemcpyDeviceToHost, c->own));
  }
  BB_CUDA_TRY(cudaStreamSynchronize(c->own));
  return BB_OK;
}

int bb_merge_host(bb_ctx* c, const uint8_t* h_high, const uint8_t* h_low, size_t count, uint8_t* h_out) {
  if (!c) return fail(BB_INVALID_ARG, "null ctx");
  BB_DEVICE_GUARD(c->device);
  int rc = c->host_in.reserve(2 * count + 64);
  if (rc) return rc;
  uint8_t* hi = static_cast<uint8_t*>(c->host_in.base);
  uint8_t* lo = hi + ((count + 15) & ~size_t(15));
  if (count) {
    BB_CUDA_TRY(cudaMemcpyAsync(hi, h_high, count, cudaMemcpyHostToDevice, c->own));
    BB_CUDA_TRY(cudaMemcpyAsync(lo, h_low, count, cudaMemcpyHostToDevice, c->own));
  }
  if ((rc = c->host_out.reserve(2 * count + 64))) return rc;
  uint8_t* dout = static_cast<uint8_t*>(c->host_out.base);
  if ((rc = launch_merge(hi, lo, count, dout, c->own))) return rc;
  if (count && (rc = c->io.d2h(h_out, dout, 2 * count, c->own))) return rc;
  BB_CUDA_TRY(cudaStreamSynchronize(c->own));
  return BB_OK;
}

int bb_histogram256_host(bb_ctx* c, const uint8_t* h_data, size_t n, uint64_t* h_counts) {
  if (!c) return fail(BB_INVALID_ARG, "null ctx");
  BB_DEVICE_GUARD(c->device);
  uint8_t* din;
  int rc = to_device(c, c->host_in, h_data, n, &din);
  if (rc) return rc;
  if ((rc = c->host_out.reserve(256 * 8 + 64))) return rc;
  unsigned long long* cnt = static_cast<unsigned long long*>(c->host_out.base);
  if ((rc = launch_hist256(din, n, cnt, c->own))) return rc;
  BB_CUDA_TRY(cudaMemcpyAsync(h_counts, cnt, 256 * 8, cudaMemcpyDeviceToHost, c->own));
  BB_CUDA_TRY(cudaStreamSynchronize(c->own));
  return BB_OK;
}

}  // extern "C"
