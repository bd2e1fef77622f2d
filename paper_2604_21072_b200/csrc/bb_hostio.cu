// Host <-> device copies of the host-buffer entry points (bb_*_host): the reference's
// plugin calls take and return pageable std::vector memory (codec.hpp `Bytes`).
//
// A pageable cudaMemcpy is staged by the driver through small pinned buffers by one
// thread (~8 GB/s measured on the box).  Here the copy is cut into 4 MiB chunks that
// rotate through NB pinned buffers owned by the context: the host-side copy of a
// chunk (pageable <-> pinned) is split across a process-wide pool of worker threads
// and overlaps the DMA of the neighbouring chunks on the context's stream.  Pointers
// that are already page-locked go straight to the DMA engine.
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "bb_common.cuh"
#include "bb_kernels.h"

namespace bb {

namespace {

// fixed pool of memcpy workers; run(k, fn) executes fn(0..k-1) and returns when all are done
class CopyPool {
 public:
  CopyPool() {
    unsigned hw = std::thread::hardware_concurrency();
    int n = (int)std::min(8u, std::max(1u, hw / 2));
    if (const char* env = getenv("BB_COPY_THREADS")) n = std::max(1, atoi(env));
    for (int i = 0; i < n - 1; i++) workers_.emplace_back([this] { loop(); });
    size_ = n;
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  int size() const { return size_; }
  void run(int k, const std::function<void(int)>& fn) {
    std::unique_lock<std::mutex> call(call_mu_);  // one parallel copy at a time per process
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      next_ = 0;
      total_ = k;
      done_ = 0;
      gen_++;
    }
    cv_.notify_all();
    work();  // the caller takes tasks too
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ == total_; });
    fn_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      int i;
      const std::function<void(int)>* f;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (!fn_ || next_ >= total_) return;
        i = next_++;
        f = fn_;
      }
      (*f)(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (++done_ == total_) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && fn_ && next_ < total_); });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> workers_;
  int size_ = 1;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int next_ = 0, total_ = 0, done_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

CopyPool& pool() {
  static CopyPool p;
  return p;
}

void par_memcpy(uint8_t* dst, const uint8_t* src, size_t n) {
  const size_t kSlice = 1 << 20;
  const int k = (int)std::min<size_t>((n + kSlice - 1) / kSlice, (size_t)pool().size());
  if (k <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
  const size_t per = (n + k - 1) / k;
  pool().run(k, [&](int i) {
    const size_t o = (size_t)i * per;
    if (o < n) std::memcpy(dst + o, src + o, std::min(per, n - o));
  });
}

// BB_HOSTIO_REGISTER=1: page-lock large pageable buffers for the duration of the copy
// (cudaHostRegister, direct DMA, unregister) instead of staging them.  Measured on the B200 box:
// registering costs ~0.1 s per 64 MiB there, so the staged path is the default.
constexpr size_t kRegisterMin = size_t(8) << 20;
bool try_register(const void* p, size_t n) {
  static const bool reg = getenv("BB_HOSTIO_REGISTER") != nullptr;
  if (!reg || n < kRegisterMin) return false;
  if (cudaHostRegister(const_cast<void*>(p), n, cudaHostRegisterDefault) != cudaSuccess) {
    cudaGetLastError();  // e.g. overlaps an already registered range: use the staged path
    return false;
  }
  return true;
}

// BB_HOSTIO_DIRECT=1: plain cudaMemcpyAsync from / to pageable memory (the driver's own staging)
bool direct_only() {
  static const bool d = getenv("BB_HOSTIO_DIRECT") != nullptr;
  return d;
}

bool page_locked(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

}  // namespace

HostStager::~HostStager() {
  for (int b = 0; b < NB; b++) {
    if (ev[b]) cudaEventDestroy(ev[b]);
    if (buf[b]) cudaFreeHost(buf[b]);
  }
}

int HostStager::ready() {
  if (buf[0]) return BB_OK;
  for (int b = 0; b < NB; b++) {
    BB_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&buf[b]), CHUNK, cudaHostAllocDefault));
    BB_CUDA_TRY(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
  }
  return BB_OK;
}

int HostStager::h2d(uint8_t* d_dst, const uint8_t* h_src, size_t n, cudaStream_t st) {
  if (!n) return BB_OK;
  if (n < SMALL || direct_only() || page_locked(h_src)) {
    BB_CUDA_TRY(cudaMemcpyAsync(d_dst, h_src, n, cudaMemcpyHostToDevice, st));
    return BB_OK;
  }
  if (try_register(h_src, n)) {
    cudaError_t e = cudaMemcpyAsync(d_dst, h_src, n, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaHostUnregister(const_cast<uint8_t*>(h_src));
    BB_CUDA_TRY(e);
    return BB_OK;
  }
  int rc = ready();
  if (rc) return rc;
  for (size_t off = 0, c = 0; off < n; off += CHUNK, c++) {
    const int b = (int)(c % NB);
    const size_t len = std::min(CHUNK, n - off);
    BB_CUDA_TRY(cudaEventSynchronize(ev[b]));  // its previous DMA (this call or the last) is done
    par_memcpy(buf[b], h_src + off, len);
    BB_CUDA_TRY(cudaMemcpyAsync(d_dst + off, buf[b], len, cudaMemcpyHostToDevice, st));
    BB_CUDA_TRY(cudaEventRecord(ev[b], st));
  }
  return BB_OK;
}

int HostStager::d2h(uint8_t* h_dst, const uint8_t* d_src, size_t n, cudaStream_t st) {
  if (!n) return BB_OK;
  if (n < SMALL || direct_only() || page_locked(h_dst)) {
    BB_CUDA_TRY(cudaMemcpyAsync(h_dst, d_src, n, cudaMemcpyDeviceToHost, st));
    return BB_OK;
  }
  if (try_register(h_dst, n)) {
    cudaError_t e = cudaMemcpyAsync(h_dst, d_src, n, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaHostUnregister(h_dst);
    BB_CUDA_TRY(e);
    return BB_OK;
  }
  int rc = ready();
  if (rc) return rc;
  const size_t chunks = (n + CHUNK - 1) / CHUNK;
  for (int b = 0; b < NB; b++) BB_CUDA_TRY(cudaEventSynchronize(ev[b]));  // an earlier h2d's DMAs
  auto issue = [&](size_t c) -> int {
    const int b = (int)(c % NB);
    const size_t off = c * CHUNK;
    BB_CUDA_TRY(cudaMemcpyAsync(buf[b], d_src + off, std::min(CHUNK, n - off), cudaMemcpyDeviceToHost, st));
    BB_CUDA_TRY(cudaEventRecord(ev[b], st));
    return BB_OK;
  };
  for (size_t c = 0; c < std::min<size_t>(chunks, NB); c++)
    if ((rc = issue(c))) return rc;
  for (size_t c = 0; c < chunks; c++) {
    const int b = (int)(c % NB);
    const size_t off = c * CHUNK;
    BB_CUDA_TRY(cudaEventSynchronize(ev[b]));
    par_memcpy(h_dst + off, buf[b], std::min(CHUNK, n - off));
    if (c + NB < chunks && (rc = issue(c + NB))) return rc;
  }
  return BB_OK;
}

}  // namespace bb
