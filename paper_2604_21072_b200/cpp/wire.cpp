// SPDX-License-Identifier: Apache-2.0
// Stage API drop-in (reference proj/include/beeplan/wire.hpp, proj/src/wire.cpp).
//
//   encode_frame / decode_frame         BBF1 framing                   wire.cpp:342-370
//   Pacer                               ShapedWriter token bucket      wire.cpp:201-248
//   run_wire_source / stage / sink      TCP roles, codec on the B200   wire.cpp:388-602
//   run_wire_local                      multi-GPU runner               wire.cpp:604-684
//   join_hop_metrics, *_to_json         metrics                        wire.cpp:372-386,686-724
//
// run_wire_local is the B200 design: every role (source, relay stages, sink) owns one
// GPU, frames stay in HBM, and a hop is a ShapedWriter-paced copy of the frame's bytes
// into an inbox slot that lives in the receiving GPU's memory (peer copies over NVLink,
// 64 KiB chunks admitted by the token bucket).  A stage keeps the reference's three
// workers (recv / compute / send) and its two bounded queues, so micro-batches overlap:
// frame k+1 lands while frame k is decoded and frame k-1 is on the outbound link.  The
// codec calls are the device entry points of include/bbcodec.h on the role's own
// stream.  Inbox slots and the per-stage buffer pools are the back-pressure: a sender
// blocks for a free slot as it would on a full socket buffer.  A failing role closes
// both of its hops, so upstream senders and downstream receivers unblock with
// ConnectionLost, and run_wire_local rethrows the first failure (wire.cpp:441-450).
//
// The TCP roles are the cross-host deployment (the paper's WAN nodes): host frames over
// sockets, every codec call through the C++ drop-in (cpp/codec.cpp -> the B200).
#include "beeplan/wire.hpp"

#include <arpa/inet.h>
#include <cuda_runtime.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <sys/socket.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <thread>
#include <utility>

#include <nlohmann/json.hpp>

#include "bbcodec.h"
#include "beeplan/errors.hpp"
#include "beeplan/synth.hpp"
#include "beeplan/wire_b200.hpp"

namespace beeplan {

namespace {

using Clock = std::chrono::steady_clock;

constexpr std::size_t kChunk = 64 * 1024;        // pacing granularity (wire.cpp:30)
constexpr std::uint64_t kMaxPayload = 1ull << 30;  // read_frame's cap (wire.cpp:31,260)
constexpr int kIoTimeoutSec = 30;

double ms_since_epoch(Clock::time_point t) {
  return std::chrono::duration<double, std::milli>(t.time_since_epoch()).count();
}

// ---------------------------------------------------------------------------
// BBF1 header

void put_le(std::uint8_t* p, std::uint64_t v, int n) {
  for (int i = 0; i < n; ++i) p[i] = static_cast<std::uint8_t>(v >> (8 * i));
}

std::uint64_t get_le(const std::uint8_t* p, int n) {
  std::uint64_t v = 0;
  for (int i = 0; i < n; ++i) v |= static_cast<std::uint64_t>(p[i]) << (8 * i);
  return v;
}

struct Head {
  WireFrame::Type type = WireFrame::Type::Activations;
  std::uint64_t batch = 0;
  std::uint16_t micro = 0;
  std::uint8_t flags = 0;
  std::uint64_t payload_len = 0;
};

void write_head(std::uint8_t* h, WireFrame::Type type, std::uint64_t batch, std::uint16_t micro,
                std::uint8_t flags, std::uint64_t payload_len) {
  std::memcpy(h, "BBF1", 4);
  h[4] = static_cast<std::uint8_t>(type);
  put_le(h + 5, batch, 8);
  put_le(h + 13, micro, 2);
  h[15] = flags;
  put_le(h + 16, payload_len, 4);
}

// decode_frame's header checks (magic, msg_type)
Head read_head(const std::uint8_t* h) {
  if (std::memcmp(h, "BBF1", 4) != 0) throw FrameCorrupt("frame: bad magic");
  if (h[4] > 3) throw FrameCorrupt("frame: unknown msg_type " + std::to_string(h[4]));
  Head d;
  d.type = static_cast<WireFrame::Type>(h[4]);
  d.batch = get_le(h + 5, 8);
  d.micro = static_cast<std::uint16_t>(get_le(h + 13, 2));
  d.flags = h[15];
  d.payload_len = get_le(h + 16, 4);
  return d;
}

// ---------------------------------------------------------------------------
// ShapedWriter's pacing, independent of the transport: the virtual wire clock
// advances by chunk / rate per 64 KiB chunk and every chunk is admitted at
// wire_free + latency; rate <= 0 delays the whole frame by the latency once.

class Pacer {
 public:
  explicit Pacer(LinkShape shape) : shape_(shape) {}

  // emit(offset, bytes) moves one admitted chunk of a frame of `total` bytes
  template <class Emit>
  void run(std::size_t total, Emit&& emit) {
    const auto latency = std::chrono::duration_cast<Clock::duration>(
        std::chrono::duration<double>(shape_.latency_ms / 1e3));
    if (shape_.rate_bps <= 0.0) {
      if (shape_.latency_ms > 0.0) std::this_thread::sleep_until(Clock::now() + latency);
      if (total) emit(std::size_t{0}, total);
      return;
    }
    const double bytes_per_s = shape_.rate_bps / 8.0;
    for (std::size_t off = 0; off < total;) {
      const std::size_t n = std::min(kChunk, total - off);
      const auto now = Clock::now();
      if (wire_free_ < now) wire_free_ = now;
      wire_free_ += std::chrono::duration_cast<Clock::duration>(
          std::chrono::duration<double>(static_cast<double>(n) / bytes_per_s));
      std::this_thread::sleep_until(wire_free_ + latency);
      emit(off, n);
      off += n;
    }
  }

 private:
  LinkShape shape_;
  Clock::time_point wire_free_{};
};

// ---------------------------------------------------------------------------
// Bounded FIFO with close(): pushes after close are dropped, pops drain and then
// report "closed" (the caller turns that into a Shutdown), wire.cpp:269-313.

template <class T>
class Bounded {
 public:
  explicit Bounded(std::size_t cap) : cap_(std::max<std::size_t>(1, cap)) {}
  void push(T v) {
    std::unique_lock<std::mutex> lk(mu_);
    not_full_.wait(lk, [&] { return closed_ || q_.size() < cap_; });
    if (closed_) return;
    q_.push_back(std::move(v));
    not_empty_.notify_one();
  }
  std::optional<T> pop() {
    std::unique_lock<std::mutex> lk(mu_);
    not_empty_.wait(lk, [&] { return closed_ || !q_.empty(); });
    if (q_.empty()) return std::nullopt;
    T v = std::move(q_.front());
    q_.pop_front();
    not_full_.notify_one();
    return v;
  }
  void close() {
    std::lock_guard<std::mutex> lk(mu_);
    closed_ = true;
    not_full_.notify_all();
    not_empty_.notify_all();
  }

 private:
  std::mutex mu_;
  std::condition_variable not_full_, not_empty_;
  std::deque<T> q_;
  std::size_t cap_;
  bool closed_ = false;
};

// first failure of a group of workers; later ones are consequences
class FirstFailure {
 public:
  void record(std::exception_ptr e) {
    std::lock_guard<std::mutex> lk(mu_);
    if (!first_) first_ = e;
  }
  void rethrow() {
    if (first_) std::rethrow_exception(first_);
  }

 private:
  std::mutex mu_;
  std::exception_ptr first_;
};

// every role's device context is created and its codec warmed up before the source's first
// offer (the clock of end_to_end_ms): module loading and workspace growth are setup, not transfer
class Latch {
 public:
  explicit Latch(int n) : n_(n) {}
  void arrive() {
    std::lock_guard<std::mutex> lk(mu_);
    if (--n_ <= 0) cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return n_ <= 0; });
  }

 private:
  std::mutex mu_;
  std::condition_variable cv_;
  int n_;
};

// arrives at the latch once: when the role is ready, or when it unwinds before that
class Arrival {
 public:
  explicit Arrival(Latch& l) : l_(l) {}
  ~Arrival() { now(); }
  void now() {
    if (!done_) l_.arrive();
    done_ = true;
  }

 private:
  Latch& l_;
  bool done_ = false;
};

// Role threads keep their device contexts until every role thread is done: tearing a context down
// (bb_ctx_destroy's cudaFree / cudaFreeHost) while other roles still run stalled their next codec
// call by 0.1-0.4 s (measured on the 1-GPU acceptance-#9 shape).  hold() at the end of a thread's
// normal path arrives and waits; a thread that unwinds with an error only arrives, so a failing
// role never blocks the others' shutdown.
class Linger {
 public:
  explicit Linger(Latch& l) : l_(l) {}
  ~Linger() {
    if (!done_) l_.arrive();
  }
  void hold() {
    done_ = true;
    l_.arrive();
    l_.wait();
  }

 private:
  Latch& l_;
  bool done_ = false;
};

// make_step_slices' spans (wire.cpp:321-336): elements split into M spans, the
// first `rem` spans one element longer
std::vector<std::pair<std::size_t, std::size_t>> step_spans(std::size_t payload_bytes, int micro) {
  if (payload_bytes % 2 != 0) throw ValidationError("payload_bytes: must be even (FP16)");
  if (micro < 1) throw ValidationError("micro_batches: must be >= 1");
  const std::size_t elements = payload_bytes / 2;
  const std::size_t base = elements / static_cast<std::size_t>(micro);
  const std::size_t rem = elements % static_cast<std::size_t>(micro);
  std::vector<std::pair<std::size_t, std::size_t>> spans;
  std::size_t at = 0;
  for (int k = 0; k < micro; ++k) {
    const std::size_t e = base + (static_cast<std::size_t>(k) < rem ? 1 : 0);
    spans.emplace_back(2 * at, 2 * e);
    at += e;
  }
  return spans;
}

Bytes step_stream(std::size_t payload_bytes, std::uint64_t seed, std::uint64_t step) {
  return synth_gaussian_fp16(payload_bytes / 2, seed + step);
}

// ---------------------------------------------------------------------------
// TCP transport (cross-host roles)

struct Endpoint {
  sockaddr_in sin{};
};

Endpoint parse_endpoint(const std::string& ep) {
  const auto colon = ep.rfind(':');
  if (colon == std::string::npos) throw ValidationError("endpoint '" + ep + "': expected host:port");
  Endpoint e;
  e.sin.sin_family = AF_INET;
  const std::string host = ep.substr(0, colon);
  int port = 0;
  try {
    port = std::stoi(ep.substr(colon + 1));
  } catch (const std::exception&) {
    throw ValidationError("endpoint '" + ep + "': bad port");
  }
  e.sin.sin_port = htons(static_cast<std::uint16_t>(port));
  if (::inet_pton(AF_INET, host.c_str(), &e.sin.sin_addr) != 1)
    throw ValidationError("endpoint host '" + host + "': expected an IPv4 address");
  return e;
}

class Fd {
 public:
  Fd() = default;
  explicit Fd(int fd) : fd_(fd) {}
  Fd(Fd&& o) noexcept : fd_(std::exchange(o.fd_, -1)) {}
  Fd& operator=(Fd&& o) noexcept {
    if (this != &o) {
      reset();
      fd_ = std::exchange(o.fd_, -1);
    }
    return *this;
  }
  Fd(const Fd&) = delete;
  Fd& operator=(const Fd&) = delete;
  ~Fd() { reset(); }
  int get() const { return fd_; }
  void reset() {
    if (fd_ >= 0) ::close(fd_);
    fd_ = -1;
  }

 private:
  int fd_ = -1;
};

std::string errno_text() { return std::strerror(errno); }

void tune(int fd) {
  timeval tv{kIoTimeoutSec, 0};
  ::setsockopt(fd, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof tv);
  ::setsockopt(fd, SOL_SOCKET, SO_SNDTIMEO, &tv, sizeof tv);
  int one = 1;
  ::setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof one);
}

Fd listen_on(const std::string& ep) {
  Endpoint e = parse_endpoint(ep);
  Fd s(::socket(AF_INET, SOCK_STREAM, 0));
  if (s.get() < 0) throw ConnectionLost("socket(): " + errno_text());
  int one = 1;
  ::setsockopt(s.get(), SOL_SOCKET, SO_REUSEADDR, &one, sizeof one);
  if (::bind(s.get(), reinterpret_cast<sockaddr*>(&e.sin), sizeof e.sin) != 0)
    throw ConnectionLost("bind(" + ep + "): " + errno_text());
  if (::listen(s.get(), 4) != 0) throw ConnectionLost("listen(" + ep + "): " + errno_text());
  return s;
}

Fd accept_from(int listen_fd) {
  timeval tv{kIoTimeoutSec, 0};
  ::setsockopt(listen_fd, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof tv);
  const int fd = ::accept(listen_fd, nullptr, nullptr);
  if (fd < 0) throw ConnectionLost("accept(): " + errno_text());
  tune(fd);
  return Fd(fd);
}

Fd dial(const std::string& ep) {
  Endpoint e = parse_endpoint(ep);
  const auto give_up = Clock::now() + std::chrono::seconds(10);
  for (;;) {
    Fd s(::socket(AF_INET, SOCK_STREAM, 0));
    if (s.get() < 0) throw ConnectionLost("socket(): " + errno_text());
    if (::connect(s.get(), reinterpret_cast<sockaddr*>(&e.sin), sizeof e.sin) == 0) {
      tune(s.get());
      return s;
    }
    if (Clock::now() >= give_up) throw ConnectionLost("connect(" + ep + "): " + errno_text());
    std::this_thread::sleep_for(std::chrono::milliseconds(20));
  }
}

void send_all(int fd, const std::uint8_t* p, std::size_t n) {
  while (n > 0) {
    const ssize_t k = ::send(fd, p, n, MSG_NOSIGNAL);
    if (k <= 0) throw ConnectionLost("send(): " + errno_text());
    p += k;
    n -= static_cast<std::size_t>(k);
  }
}

// false on a clean EOF before the first byte (when allowed)
bool recv_all(int fd, std::uint8_t* p, std::size_t n, bool eof_ok) {
  std::size_t got = 0;
  while (got < n) {
    const ssize_t k = ::recv(fd, p + got, n - got, 0);
    if (k == 0) {
      if (got == 0 && eof_ok) return false;
      throw ConnectionLost("recv(): peer closed mid-frame");
    }
    if (k < 0) throw ConnectionLost("recv(): " + errno_text());
    got += static_cast<std::size_t>(k);
  }
  return true;
}

// read_frame (wire.cpp:250-267): header checks, 1 GiB cap, then the payload
std::optional<WireFrame> read_socket_frame(int fd, double* t_recv) {
  std::uint8_t h[kFrameHeaderSize];
  if (!recv_all(fd, h, sizeof h, true)) return std::nullopt;
  const Head d = read_head(h);
  if (d.payload_len > kMaxPayload) throw FrameCorrupt("frame: implausible payload length");
  WireFrame f;
  f.msg_type = d.type;
  f.batch_id = d.batch;
  f.micro_index = d.micro;
  f.flags = d.flags;
  f.payload.resize(d.payload_len);
  if (d.payload_len) recv_all(fd, f.payload.data(), d.payload_len, false);
  if (t_recv) *t_recv = wire_now_ms();
  return f;
}

FrameSendRecord socket_send(Pacer& pacer, int fd, const Bytes& frame, std::uint64_t batch, std::uint16_t micro) {
  FrameSendRecord r;
  r.batch_id = batch;
  r.micro_index = micro;
  r.bytes = frame.size();
  r.t_offer_ms = wire_now_ms();
  pacer.run(frame.size(), [&](std::size_t off, std::size_t n) { send_all(fd, frame.data() + off, n); });
  r.t_sent_ms = wire_now_ms();
  return r;
}

WireFrame shutdown_frame() {
  WireFrame f;
  f.msg_type = WireFrame::Type::Shutdown;
  return f;
}

// ---------------------------------------------------------------------------
// GPU transport (run_wire_local)

[[noreturn]] void cuda_fail(cudaError_t e, const char* what) {
  throw Error(std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}
#define WIRE_CUDA(expr)                          \
  do {                                           \
    cudaError_t wire_e_ = (expr);                \
    if (wire_e_ != cudaSuccess) cuda_fail(wire_e_, #expr); \
  } while (0)

[[noreturn]] void codec_fail(int rc) {
  const std::string msg = bb_last_error();
  switch (rc) {
    case BB_ODD_LENGTH: throw OddLength(msg);
    case BB_LANE_MISMATCH: throw LaneLengthMismatch(msg);
    case BB_BACKEND_UNKNOWN: throw BackendUnknown(msg);
    case BB_CORRUPT_CONTAINER: throw CorruptContainer(msg);
    default: throw Error(msg.empty() ? "bbcodec failure" : msg);
  }
}
void codec_ok(int rc) {
  if (rc != BB_OK) codec_fail(rc);
}

// growable device buffer on one GPU
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void ensure(int dev, std::size_t n) {
    if (p_ && cap_ >= n) return;
    release();
    int prev = 0;
    cudaGetDevice(&prev);
    WIRE_CUDA(cudaSetDevice(dev));
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, std::max<std::size_t>(n, 256));
    cudaSetDevice(prev);
    if (e != cudaSuccess) cuda_fail(e, "cudaMalloc");
    p_ = static_cast<std::uint8_t*>(p);
    cap_ = std::max<std::size_t>(n, 256);
    dev_ = dev;
  }
  std::uint8_t* get() const { return p_; }
  std::size_t cap() const { return cap_; }

 private:
  void release() {
    if (!p_) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dev_);
    cudaFree(p_);
    cudaSetDevice(prev);
    p_ = nullptr;
    cap_ = 0;
  }
  std::uint8_t* p_ = nullptr;
  std::size_t cap_ = 0;
  int dev_ = 0;
};

// per-thread device context of one role: current device, codec context, stream,
// pinned header staging
class RoleDevice {
 public:
  explicit RoleDevice(int dev) : dev_(dev) {
    WIRE_CUDA(cudaSetDevice(dev));
    codec_ok(bb_ctx_create(&ctx_, dev));
    WIRE_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    WIRE_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&pinned_), 64, cudaHostAllocDefault));
    WIRE_CUDA(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
  }
  ~RoleDevice() {
    cudaSetDevice(dev_);
    if (st_) cudaStreamSynchronize(st_);
    if (done_) cudaEventDestroy(done_);
    if (pinned_) cudaFreeHost(pinned_);
    if (st_) cudaStreamDestroy(st_);
    bb_ctx_destroy(ctx_);
  }
  RoleDevice(const RoleDevice&) = delete;
  RoleDevice& operator=(const RoleDevice&) = delete;
  int dev() const { return dev_; }
  bb_ctx* ctx() const { return ctx_; }
  cudaStream_t stream() const { return st_; }
  std::uint8_t* pinned() const { return pinned_; }
  // waits of the pacing threads poll briefly, then sleep between polls instead of spinning: a box
  // runs three threads per role, and spinning waiters delay the token buckets' wake-ups (link
  // jitter).  (A cudaEventBlockingSync wait measured ~25 ms of wake-up latency per frame.)
  void sync() {
    WIRE_CUDA(cudaEventRecord(done_, st_));
    const auto t0 = Clock::now();
    for (;;) {
      const cudaError_t e = cudaEventQuery(done_);
      if (e == cudaSuccess) return;
      if (e != cudaErrorNotReady) cuda_fail(e, "cudaEventQuery");
      if (Clock::now() - t0 < std::chrono::microseconds(100)) std::this_thread::yield();
      else std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  }

 private:
  int dev_;
  bb_ctx* ctx_ = nullptr;
  cudaStream_t st_ = nullptr;
  cudaEvent_t done_ = nullptr;
  std::uint8_t* pinned_ = nullptr;
};

// The receiving side of one hop: frame slots in the receiver's HBM.  A sender
// acquires a free slot (blocking: back-pressure), writes the frame into it with
// paced peer copies and publishes it; the receiver pops landed frames in order
// and releases a slot once the frame's bytes are no longer needed.
class Inbox {
 public:
  // every slot is allocated up front at the run's largest frame: no cudaMalloc / cudaFree (which
  // synchronizes the whole device) happens once frames flow
  Inbox(int dev, int slots, std::size_t slot_bytes) : dev_(dev), bufs_(static_cast<std::size_t>(slots)) {
    for (int i = 0; i < slots; ++i) {
      bufs_[static_cast<std::size_t>(i)].ensure(dev, slot_bytes);
      free_.push_back(i);
    }
  }
  int dev() const { return dev_; }
  int acquire(std::size_t bytes) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return closed_ || !free_.empty(); });
    if (closed_) throw ConnectionLost("send(): downstream closed");
    const int s = free_.front();
    free_.pop_front();
    lk.unlock();
    bufs_[static_cast<std::size_t>(s)].ensure(dev_, bytes);
    return s;
  }
  std::uint8_t* slot(int s) const { return bufs_[static_cast<std::size_t>(s)].get(); }
  void publish(int s, std::size_t bytes, double t_land) {
    std::lock_guard<std::mutex> lk(mu_);
    if (closed_) throw ConnectionLost("send(): downstream closed");
    landed_.push_back({s, bytes, t_land});
    cv_.notify_all();
  }
  struct Landed {
    int slot;
    std::size_t bytes;
    double t_land;
  };
  std::optional<Landed> pop() {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return closed_ || !landed_.empty(); });
    if (landed_.empty()) return std::nullopt;
    Landed l = landed_.front();
    landed_.pop_front();
    return l;
  }
  void release(int s) {
    std::lock_guard<std::mutex> lk(mu_);
    free_.push_back(s);
    cv_.notify_all();
  }
  void close() {
    std::lock_guard<std::mutex> lk(mu_);
    closed_ = true;
    cv_.notify_all();
  }

 private:
  int dev_;
  std::vector<DevBuf> bufs_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<int> free_;
  std::deque<Landed> landed_;
  bool closed_ = false;
};

// pool of reusable device buffers of one role (decoded payloads, outbound frames)
class BufPool {
 public:
  BufPool(int dev, int n, std::size_t bytes) : dev_(dev), bufs_(static_cast<std::size_t>(n)) {
    for (int i = 0; i < n; ++i) {
      bufs_[static_cast<std::size_t>(i)].ensure(dev, bytes);
      free_.push_back(i);
    }
  }
  int take(std::size_t bytes) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return closed_ || !free_.empty(); });
    if (closed_) throw ConnectionLost("stage: shutting down");
    const int b = free_.front();
    free_.pop_front();
    lk.unlock();
    bufs_[static_cast<std::size_t>(b)].ensure(dev_, bytes);
    return b;
  }
  std::uint8_t* get(int b) const { return bufs_[static_cast<std::size_t>(b)].get(); }
  void give(int b) {
    std::lock_guard<std::mutex> lk(mu_);
    free_.push_back(b);
    cv_.notify_all();
  }
  void close() {
    std::lock_guard<std::mutex> lk(mu_);
    closed_ = true;
    cv_.notify_all();
  }

 private:
  int dev_;
  std::vector<DevBuf> bufs_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<int> free_;
  bool closed_ = false;
};

// a frame in HBM: header fields on the host, payload bytes on the device; the
// payload is owned by an inbox slot or a pool buffer until it is sent / consumed
struct DevFrame {
  Head head;
  const std::uint8_t* payload = nullptr;
  std::size_t len = 0;
  int inbox_slot = -1;
  int pool_buf = -1;
};

using b200::WireFault;

// the sending side of one hop
class HopSender {
 public:
  HopSender(Inbox& to, LinkShape shape, const WireFault* fault)
      : to_(to), pacer_(shape), fault_(fault) {}

  FrameSendRecord send(RoleDevice& rd, const DevFrame& f) {
    FrameSendRecord r;
    r.batch_id = f.head.batch;
    r.micro_index = f.head.micro;
    const std::size_t total = kFrameHeaderSize + f.len;
    r.bytes = total;
    r.t_offer_ms = wire_now_ms();
    const std::uint64_t index = offered_++;
    if (fault_ && fault_->kind == WireFault::Kind::DropLink && index == static_cast<std::uint64_t>(fault_->frame)) {
      to_.close();  // the peer vanishes mid-stream
      throw ConnectionLost("send(): link dropped (injected)");
    }
    std::uint8_t* h = rd.pinned();
    write_head(h, f.head.type, f.head.batch, f.head.micro, f.head.flags, f.len);
    if (fault_ && fault_->kind == WireFault::Kind::CorruptMagic && index == static_cast<std::uint64_t>(fault_->frame))
      h[0] = 'X';
    const int s = to_.acquire(total);
    std::uint8_t* dst = to_.slot(s);
    try {
      pacer_.run(total, [&](std::size_t off, std::size_t n) {
        // [0, 20) comes from the pinned header, [20, total) from the payload in HBM
        if (off < kFrameHeaderSize) {
          const std::size_t k = std::min(n, kFrameHeaderSize - off);
          WIRE_CUDA(cudaMemcpyAsync(dst + off, h + off, k, cudaMemcpyHostToDevice, rd.stream()));
          off += k;
          n -= k;
        }
        if (n) {
          const std::size_t p = off - kFrameHeaderSize;
          if (to_.dev() == rd.dev())
            WIRE_CUDA(cudaMemcpyAsync(dst + off, f.payload + p, n, cudaMemcpyDeviceToDevice, rd.stream()));
          else
            WIRE_CUDA(cudaMemcpyPeerAsync(dst + off, to_.dev(), f.payload + p, rd.dev(), n, rd.stream()));
        }
      });
      rd.sync();
    } catch (...) {
      to_.release(s);
      throw;
    }
    r.t_sent_ms = wire_now_ms();
    to_.publish(s, total, r.t_sent_ms);
    bytes_ += total;
    return r;
  }
  std::uint64_t bytes() const { return bytes_; }

  // one small copy into the receiver's HBM before the clock starts: the first peer copy between
  // two GPUs of a process sets up the mapping (measured: up to ~150 ms), which is not transfer time
  void warm(RoleDevice& rd) {
    DevBuf scratch;
    scratch.ensure(rd.dev(), 256);
    const int s = to_.acquire(256);  // slots are pre-sized: no reallocation
    cudaError_t e = to_.dev() == rd.dev()
                        ? cudaMemcpyAsync(to_.slot(s), scratch.get(), 256, cudaMemcpyDeviceToDevice, rd.stream())
                        : cudaMemcpyPeerAsync(to_.slot(s), to_.dev(), scratch.get(), rd.dev(), 256, rd.stream());
    if (e == cudaSuccess) e = cudaStreamSynchronize(rd.stream());
    to_.release(s);
    if (e != cudaSuccess) cuda_fail(e, "hop warm-up copy");
  }

 private:
  Inbox& to_;
  Pacer pacer_;
  const WireFault* fault_;
  std::uint64_t offered_ = 0;
  std::uint64_t bytes_ = 0;
};

// the receiving side: pop a landed frame, read its header back from HBM and
// validate it as read_frame does
std::optional<DevFrame> hop_recv(RoleDevice& rd, Inbox& in, double* t_recv) {
  std::optional<Inbox::Landed> l = in.pop();
  if (!l) return std::nullopt;
  *t_recv = wire_now_ms();
  DevFrame f;
  f.inbox_slot = l->slot;
  std::uint8_t* h = rd.pinned() + 32;
  try {
    WIRE_CUDA(cudaMemcpyAsync(h, in.slot(l->slot), kFrameHeaderSize, cudaMemcpyDeviceToHost, rd.stream()));
    rd.sync();
    f.head = read_head(h);
    if (f.head.payload_len > kMaxPayload) throw FrameCorrupt("frame: implausible payload length");
    if (l->bytes != kFrameHeaderSize + f.head.payload_len)
      throw FrameCorrupt("frame: payload length does not match the header");
  } catch (...) {
    in.release(l->slot);
    throw;
  }
  f.payload = in.slot(l->slot) + kFrameHeaderSize;
  f.len = f.head.payload_len;
  return f;
}

// the decoded size of a BBC1 container in HBM (parse_container + plan, no decoding)
std::size_t container_decoded_size(RoleDevice& rd, const std::uint8_t* c, std::size_t n) {
  std::size_t need = 0;
  codec_ok(bb_decompress(rd.ctx(), c, n, nullptr, 0, &need, rd.stream()));
  return need;
}

// one compress + decompress of a micro-batch of the run's own data on the role's context: loads the
// codec's kernels on this device and grows the context's workspaces to what the run's frames need
// (a workspace that grows while frames flow costs a device-synchronising cudaFree)
void warm_codec(RoleDevice& rd, const Bytes& sample, std::uint8_t backend) {
  std::size_t bytes = sample.size() & ~std::size_t(1);
  if (bytes < 2) return;
  DevBuf in, out, back;
  const std::size_t cap = bb_compress_bound(bytes, backend, 1);
  in.ensure(rd.dev(), bytes);
  out.ensure(rd.dev(), cap);
  back.ensure(rd.dev(), bytes);
  WIRE_CUDA(cudaMemcpyAsync(in.get(), sample.data(), bytes, cudaMemcpyHostToDevice, rd.stream()));
  std::size_t len = 0, got = 0;
  codec_ok(bb_compress(rd.ctx(), in.get(), bytes, backend, 1, out.get(), cap, &len, rd.stream()));
  codec_ok(bb_decompress(rd.ctx(), out.get(), len, back.get(), bytes, &got, rd.stream()));
  rd.sync();
}

std::vector<int> wire_devices(const std::vector<int>& asked) {
  if (!asked.empty()) return asked;
  std::vector<int> devs;
  if (const char* env = std::getenv("BEEPLAN_WIRE_DEVICES")) {
    std::string s(env);
    std::size_t at = 0;
    while (at < s.size()) {
      std::size_t comma = s.find(',', at);
      if (comma == std::string::npos) comma = s.size();
      if (comma > at) devs.push_back(std::atoi(s.substr(at, comma - at).c_str()));
      at = comma + 1;
    }
  }
  if (devs.empty()) {
    int n = 0;
    WIRE_CUDA(cudaGetDeviceCount(&n));
    if (n < 1) throw Error("run_wire_local: no CUDA device");
    for (int d = 0; d < n; ++d) devs.push_back(d);
  }
  return devs;
}

}  // namespace

// ---------------------------------------------------------------------------

double wire_now_ms() { return ms_since_epoch(Clock::now()); }

// BEEPLAN_WIRE_TRACE=1: per-frame timings of the GPU runner's stage workers on stderr
bool wire_trace() {
  static const bool on = std::getenv("BEEPLAN_WIRE_TRACE") != nullptr;
  return on;
}

Bytes encode_frame(const WireFrame& frame) {
  Bytes out(kFrameHeaderSize + frame.payload.size());
  write_head(out.data(), frame.msg_type, frame.batch_id, frame.micro_index, frame.flags, frame.payload.size());
  if (!frame.payload.empty()) std::memcpy(out.data() + kFrameHeaderSize, frame.payload.data(), frame.payload.size());
  return out;
}

WireFrame decode_frame(const Bytes& data) {
  if (data.size() < kFrameHeaderSize) throw FrameCorrupt("frame: truncated header");
  const Head d = read_head(data.data());
  if (data.size() != kFrameHeaderSize + d.payload_len)
    throw FrameCorrupt("frame: payload length does not match the header");
  WireFrame f;
  f.msg_type = d.type;
  f.batch_id = d.batch;
  f.micro_index = d.micro;
  f.flags = d.flags;
  f.payload.assign(data.begin() + kFrameHeaderSize, data.end());
  return f;
}

HopMetrics join_hop_metrics(const WireRoleReport& sender, const WireRoleReport& receiver) {
  // first receive record per (batch, micro), as the reference's linear search finds it
  std::map<std::pair<std::uint64_t, std::uint16_t>, double> first_recv;
  for (const FrameRecvRecord& r : receiver.received) first_recv.emplace(std::make_pair(r.batch_id, r.micro_index), r.t_recv_ms);
  HopMetrics hop;
  for (const FrameSendRecord& s : sender.sent) {
    auto it = first_recv.find({s.batch_id, s.micro_index});
    if (it == first_recv.end()) continue;
    hop.transfer_ms_total += it->second - s.t_offer_ms;
    ++hop.frames;
  }
  hop.transfer_ms_mean = hop.frames > 0 ? hop.transfer_ms_total / hop.frames : 0.0;
  hop.compression_ms_total = sender.codec_ms_total;
  return hop;
}

// ---------------------------------------------------------------------------
// TCP roles

WireRoleReport run_wire_source(const WireSourceConfig& cfg) {
  WireRoleReport rep;
  const auto spans = step_spans(cfg.payload_bytes, cfg.micro_batches);
  Fd sock = dial(cfg.connect);
  Pacer pacer(cfg.shape);
  double first_offer = 0.0, last_sent = 0.0;
  for (int step = 0; step < cfg.steps; ++step) {
    const Bytes stream = step_stream(cfg.payload_bytes, cfg.seed, static_cast<std::uint64_t>(step));
    for (int m = 0; m < cfg.micro_batches; ++m) {
      const auto [off, bytes] = spans[static_cast<std::size_t>(m)];
      WireFrame f;
      f.batch_id = static_cast<std::uint64_t>(step);
      f.micro_index = static_cast<std::uint16_t>(m);
      Bytes slice(stream.begin() + static_cast<std::ptrdiff_t>(off),
                  stream.begin() + static_cast<std::ptrdiff_t>(off + bytes));
      if (cfg.compress) {
        const double t0 = wire_now_ms();
        f.payload = serialize_container(compress(slice, cfg.backend, true));
        rep.codec_ms_total += wire_now_ms() - t0;
        f.flags = WireFrame::kFlagCompressed | WireFrame::kFlagByteSplit;
      } else {
        f.payload = std::move(slice);
      }
      FrameSendRecord r = socket_send(pacer, sock.get(), encode_frame(f), f.batch_id, f.micro_index);
      if (rep.sent.empty()) first_offer = r.t_offer_ms;
      last_sent = r.t_sent_ms;
      rep.sent.push_back(r);
      ++rep.frames_seen;
    }
  }
  socket_send(pacer, sock.get(), encode_frame(shutdown_frame()), 0, 0);
  rep.metrics.completion_ms = last_sent - first_offer;
  rep.metrics.step_ms = cfg.steps > 0 ? rep.metrics.completion_ms / cfg.steps : 0.0;
  return rep;
}

WireRoleReport run_wire_stage(const WireStageConfig& cfg) {
  WireRoleReport rep;
  Fd own_listener = cfg.listen_fd >= 0 ? Fd() : listen_on(cfg.listen);
  const int lfd = cfg.listen_fd >= 0 ? cfg.listen_fd : own_listener.get();
  Fd down = dial(cfg.connect);
  Fd up = accept_from(lfd);

  Bounded<WireFrame> inbound(static_cast<std::size_t>(cfg.queue_slots));
  Bounded<WireFrame> outbound(static_cast<std::size_t>(cfg.queue_slots));
  FirstFailure failure;
  auto fail_all = [&] {
    failure.record(std::current_exception());
    inbound.close();
    outbound.close();
  };
  std::vector<FrameRecvRecord> received;
  double dec_ms = 0.0, enc_ms = 0.0, busy_ms = 0.0;

  std::thread rx([&] {
    try {
      for (;;) {
        double t = 0.0;
        std::optional<WireFrame> f = read_socket_frame(up.get(), &t);
        if (!f) throw ConnectionLost("stage: upstream closed before shutdown");
        const bool last = f->msg_type == WireFrame::Type::Shutdown;
        if (!last) received.push_back({f->batch_id, f->micro_index, t, kFrameHeaderSize + f->payload.size()});
        inbound.push(std::move(*f));
        if (last) break;
      }
    } catch (...) {
      fail_all();
    }
  });
  std::thread work([&] {
    try {
      for (;;) {
        WireFrame f = inbound.pop().value_or(shutdown_frame());
        if (f.msg_type == WireFrame::Type::Shutdown) {
          outbound.push(std::move(f));
          break;
        }
        if (f.flags & WireFrame::kFlagCompressed) {
          const double t0 = wire_now_ms();
          f.payload = decompress(parse_container(f.payload));
          dec_ms += wire_now_ms() - t0;
          f.flags &= static_cast<std::uint8_t>(~(WireFrame::kFlagCompressed | WireFrame::kFlagByteSplit));
        }
        if (cfg.compute_ms > 0.0) {
          std::this_thread::sleep_for(std::chrono::duration<double, std::milli>(cfg.compute_ms));
          busy_ms += cfg.compute_ms;
        }
        if (cfg.compress_out) {
          const double t0 = wire_now_ms();
          f.payload = serialize_container(compress(f.payload, cfg.backend, true));
          enc_ms += wire_now_ms() - t0;
          f.flags |= WireFrame::kFlagCompressed | WireFrame::kFlagByteSplit;
        }
        outbound.push(std::move(f));
      }
    } catch (...) {
      fail_all();
    }
  });
  std::thread tx([&] {
    try {
      Pacer pacer(cfg.shape);
      for (;;) {
        WireFrame f = outbound.pop().value_or(shutdown_frame());
        const bool last = f.msg_type == WireFrame::Type::Shutdown;
        FrameSendRecord r = socket_send(pacer, down.get(), encode_frame(f), f.batch_id, f.micro_index);
        if (last) break;
        rep.sent.push_back(r);
      }
    } catch (...) {
      fail_all();
    }
  });
  rx.join();
  work.join();
  tx.join();
  failure.rethrow();

  rep.received = std::move(received);
  rep.codec_ms_total = dec_ms + enc_ms;
  rep.frames_seen = rep.received.size();
  if (!rep.received.empty() && !rep.sent.empty())
    rep.metrics.completion_ms = rep.sent.back().t_sent_ms - rep.received.front().t_recv_ms;
  rep.metrics.stages.push_back({busy_ms, rep.metrics.completion_ms - busy_ms});
  return rep;
}

WireRoleReport run_wire_sink(const WireSinkConfig& cfg) {
  WireRoleReport rep;
  Fd own_listener = cfg.listen_fd >= 0 ? Fd() : listen_on(cfg.listen);
  const int lfd = cfg.listen_fd >= 0 ? cfg.listen_fd : own_listener.get();
  Fd up = accept_from(lfd);
  const auto spans = step_spans(cfg.payload_bytes, cfg.micro_batches);

  std::uint64_t step = ~0ull;
  Bytes expected, assembled;
  auto close_step = [&] {
    if (step != ~0ull && cfg.verify && assembled != expected) rep.payload_ok = false;
  };
  for (;;) {
    double t = 0.0;
    std::optional<WireFrame> f = read_socket_frame(up.get(), &t);
    if (!f) throw ConnectionLost("sink: upstream closed before shutdown");
    if (f->msg_type == WireFrame::Type::Shutdown) break;
    rep.received.push_back({f->batch_id, f->micro_index, t, kFrameHeaderSize + f->payload.size()});
    ++rep.frames_seen;
    if (f->msg_type != WireFrame::Type::Activations) continue;
    if (f->batch_id != step) {
      close_step();
      step = f->batch_id;
      expected = step_stream(cfg.payload_bytes, cfg.seed, step);
      assembled.assign(expected.size(), 0);
    }
    if (f->micro_index >= spans.size())
      throw FrameCorrupt("sink: micro_index " + std::to_string(f->micro_index) +
                         " outside the configured micro-batch count");
    Bytes payload = std::move(f->payload);
    if (f->flags & WireFrame::kFlagCompressed) {
      const double t0 = wire_now_ms();
      payload = decompress(parse_container(payload));
      rep.codec_ms_total += wire_now_ms() - t0;
    }
    const auto [off, bytes] = spans[f->micro_index];
    if (payload.size() != bytes)
      rep.payload_ok = false;
    else
      std::copy(payload.begin(), payload.end(), assembled.begin() + static_cast<std::ptrdiff_t>(off));
  }
  close_step();
  if (!rep.received.empty())
    rep.metrics.completion_ms = rep.received.back().t_recv_ms - rep.received.front().t_recv_ms;
  return rep;
}

// ---------------------------------------------------------------------------
// multi-GPU runner

namespace b200 {

WireLocalResult run_wire_local(const WireLocalConfig& cfg, const WireLocalOptions& opt,
                               WireLocalPlacement* placement) {
  if (cfg.stage_count < 0) throw ValidationError("stage_count: must be >= 0");
  const auto spans = step_spans(cfg.payload_bytes, cfg.micro_batches);
  const std::vector<int> devs = wire_devices(opt.devices);
  const int roles = cfg.stage_count + 2;
  std::vector<int> role_dev(static_cast<std::size_t>(roles));
  for (int r = 0; r < roles; ++r) role_dev[static_cast<std::size_t>(r)] = devs[static_cast<std::size_t>(r) % devs.size()];
  for (int r = 0; r + 1 < roles; ++r)
    if (role_dev[r] != role_dev[r + 1]) bb_enable_peer_access(role_dev[r], role_dev[r + 1]);  // else staged copies

  // The step streams are the source's activations, generated before the clock starts (on a
  // GPU node they come out of the model's compute, not out of a host RNG); the sink verifies
  // against the same reference generator's bytes (make_step_slices, wire.cpp:315-336).
  const int steps = std::max(0, cfg.steps);
  std::vector<Bytes> host_streams(static_cast<std::size_t>(steps));
  {
    const int nt = std::max(1, std::min<int>(steps, (int)std::max(1u, std::thread::hardware_concurrency())));
    std::atomic<int> next{0};
    std::vector<std::thread> gen;
    for (int k = 0; k < nt; ++k)
      gen.emplace_back([&] {
        for (int s; (s = next.fetch_add(1)) < steps;)
          host_streams[static_cast<std::size_t>(s)] = step_stream(cfg.payload_bytes, cfg.seed, s);
      });
    for (auto& t : gen) t.join();
  }
  const int src_dev = role_dev.front(), sink_dev = role_dev.back();
  std::vector<DevBuf> src_streams(static_cast<std::size_t>(steps)), want_streams(static_cast<std::size_t>(steps));
  for (int s = 0; s < steps; ++s) {
    const Bytes& h = host_streams[static_cast<std::size_t>(s)];
    src_streams[static_cast<std::size_t>(s)].ensure(src_dev, h.size());
    want_streams[static_cast<std::size_t>(s)].ensure(sink_dev, h.size());
    WIRE_CUDA(cudaMemcpy(src_streams[static_cast<std::size_t>(s)].get(), h.data(), h.size(), cudaMemcpyHostToDevice));
    WIRE_CUDA(cudaMemcpy(want_streams[static_cast<std::size_t>(s)].get(), h.data(), h.size(), cudaMemcpyHostToDevice));
  }
  // the warm-up sample: the largest micro-batch of the first step
  Bytes warm_sample;
  if (steps > 0) {
    std::size_t off = 0, len = 0;
    for (const auto& sp : spans)
      if (sp.second > len) off = sp.first, len = sp.second;
    warm_sample.assign(host_streams[0].begin() + static_cast<std::ptrdiff_t>(off),
                       host_streams[0].begin() + static_cast<std::ptrdiff_t>(off + len));
  }
  host_streams.clear();

  const std::size_t frame_cap = [&] {
    std::size_t mx = 0;
    for (const auto& sp : spans) mx = std::max(mx, sp.second);
    return std::max(mx, static_cast<std::size_t>(bb_compress_bound(mx, cfg.backend, 1)));
  }();
  const int slots = std::max(1, opt.queue_slots);
  // inbox[i] receives hop i (i = 0: source -> first receiver); its slots cover what the receiver
  // may hold at once: its queues, the frame in compute and the frame on the outbound link
  std::vector<std::unique_ptr<Inbox>> inbox;
  for (int r = 1; r < roles; ++r)
    inbox.push_back(std::make_unique<Inbox>(role_dev[static_cast<std::size_t>(r)], 2 * slots + 3,
                                            kFrameHeaderSize + frame_cap + 16));
  const WireFault* fault = opt.fault.kind == WireFault::Kind::None ? nullptr : &opt.fault;
  auto fault_for = [&](int hop) { return fault && fault->hop == hop ? fault : nullptr; };
  std::vector<std::unique_ptr<HopSender>> hop;
  for (int h = 0; h + 1 < roles; ++h)
    hop.push_back(std::make_unique<HopSender>(*inbox[static_cast<std::size_t>(h)], cfg.shape, fault_for(h)));

  WireLocalResult result;
  result.stages.resize(static_cast<std::size_t>(cfg.stage_count));
  FirstFailure failure;
  std::vector<std::unique_ptr<BufPool>> pools;
  for (int i = 0; i < cfg.stage_count; ++i)
    pools.push_back(std::make_unique<BufPool>(role_dev[static_cast<std::size_t>(i) + 1], slots + 4, frame_cap + 16));
  // a failing role unblocks both neighbours: its inbox (upstream sender) and its outbound hop
  auto close_role = [&](int r) {
    if (r >= 1) inbox[static_cast<std::size_t>(r) - 1]->close();
    if (r + 1 < roles) inbox[static_cast<std::size_t>(r)]->close();
    if (r >= 1 && r <= cfg.stage_count) pools[static_cast<std::size_t>(r) - 1]->close();
  };
  auto role_failed = [&](int r) {
    failure.record(std::current_exception());
    close_role(r);
  };
  // source, sink, and per stage its compute and send workers warm up (codec, first peer copy)
  Latch ready(2 + 2 * cfg.stage_count);
  // threads owning a RoleDevice: sink, source, and per stage its recv / compute / send workers
  Latch teardown(2 + 3 * cfg.stage_count);

  std::vector<std::thread> threads;
  // sink (wire.cpp:543-602): reassemble every step in HBM and compare with the expected stream
  threads.emplace_back([&] {
    const int r = roles - 1;
    try {
      Arrival arrival(ready);
      RoleDevice rd(sink_dev);
      Linger linger(teardown);
      if (cfg.compress) warm_codec(rd, warm_sample, cfg.backend);
      arrival.now();
      Inbox& in = *inbox.back();
      WireRoleReport& rep = result.sink;
      DevBuf assembled;
      assembled.ensure(sink_dev, cfg.payload_bytes + 16);
      std::uint64_t step = ~0ull;
      auto close_step = [&] {
        if (step == ~0ull) return;
        int eq = 0;
        const DevBuf* want = step < want_streams.size() ? &want_streams[step] : nullptr;
        if (!want) {
          rep.payload_ok = false;
          return;
        }
        codec_ok(bb_equal(rd.ctx(), assembled.get(), want->get(), cfg.payload_bytes, &eq, rd.stream()));
        if (!eq) rep.payload_ok = false;
      };
      for (;;) {
        double t = 0.0;
        std::optional<DevFrame> f = hop_recv(rd, in, &t);
        if (!f) throw ConnectionLost("sink: upstream closed before shutdown");
        if (f->head.type == WireFrame::Type::Shutdown) {
          in.release(f->inbox_slot);
          break;
        }
        rep.received.push_back({f->head.batch, f->head.micro, t, kFrameHeaderSize + f->len});
        ++rep.frames_seen;
        if (f->head.type != WireFrame::Type::Activations) {
          in.release(f->inbox_slot);
          continue;
        }
        if (f->head.batch != step) {
          close_step();
          step = f->head.batch;
          WIRE_CUDA(cudaMemsetAsync(assembled.get(), 0, cfg.payload_bytes, rd.stream()));
        }
        if (f->head.micro >= spans.size()) {
          in.release(f->inbox_slot);
          throw FrameCorrupt("sink: micro_index " + std::to_string(f->head.micro) +
                             " outside the configured micro-batch count");
        }
        const auto [off, bytes] = spans[f->head.micro];
        try {
          if (f->head.flags & WireFrame::kFlagCompressed) {
            const double t0 = wire_now_ms();
            const std::size_t need = container_decoded_size(rd, f->payload, f->len);
            if (need != bytes) {
              rep.payload_ok = false;
            } else {
              std::size_t got = 0;
              codec_ok(bb_decompress(rd.ctx(), f->payload, f->len, assembled.get() + off, bytes, &got, rd.stream()));
              rd.sync();
            }
            rep.codec_ms_total += wire_now_ms() - t0;
          } else if (f->len != bytes) {
            rep.payload_ok = false;
          } else {
            WIRE_CUDA(cudaMemcpyAsync(assembled.get() + off, f->payload, bytes, cudaMemcpyDeviceToDevice, rd.stream()));
            rd.sync();
          }
        } catch (...) {
          in.release(f->inbox_slot);
          throw;
        }
        in.release(f->inbox_slot);
      }
      close_step();
      if (!rep.received.empty())
        rep.metrics.completion_ms = rep.received.back().t_recv_ms - rep.received.front().t_recv_ms;
      linger.hold();
    } catch (...) {
      role_failed(r);
    }
  });

  // relay stages (wire.cpp:431-541): recv / compute / send workers, bounded queues
  for (int i = 0; i < cfg.stage_count; ++i) {
    threads.emplace_back([&, i] {
      const int r = i + 1;
      const int dev = role_dev[static_cast<std::size_t>(r)];
      Inbox& in = *inbox[static_cast<std::size_t>(i)];
      HopSender& out = *hop[static_cast<std::size_t>(r)];
      BufPool& pool = *pools[static_cast<std::size_t>(i)];
      WireRoleReport& rep = result.stages[static_cast<std::size_t>(i)];
      Bounded<DevFrame> inbound(static_cast<std::size_t>(slots)), outbound(static_cast<std::size_t>(slots));
      std::atomic<bool> failed{false};
      auto fail_stage = [&] {  // the root cause is recorded before any neighbour unblocks
        failure.record(std::current_exception());
        failed = true;
        inbound.close();
        outbound.close();
        close_role(r);
      };
      auto drop = [&](const DevFrame& f) {
        if (f.inbox_slot >= 0) in.release(f.inbox_slot);
        if (f.pool_buf >= 0) pool.give(f.pool_buf);
      };
      auto shutdown = [] {
        DevFrame f;
        f.head.type = WireFrame::Type::Shutdown;
        return f;
      };
      std::vector<FrameRecvRecord> received;
      double dec_ms = 0.0, enc_ms = 0.0, busy_ms = 0.0;
      std::thread rx([&] {
        try {
          RoleDevice rd(dev);
          Linger linger(teardown);
          for (;;) {
            double t = 0.0;
            std::optional<DevFrame> f = hop_recv(rd, in, &t);
            if (!f) throw ConnectionLost("stage: upstream closed before shutdown");
            const bool last = f->head.type == WireFrame::Type::Shutdown;
            if (!last) received.push_back({f->head.batch, f->head.micro, t, kFrameHeaderSize + f->len});
            inbound.push(*f);
            if (last) break;
          }
          linger.hold();
        } catch (...) {
          fail_stage();
        }
      });
      std::thread work([&] {
        try {
          Arrival arrival(ready);
          RoleDevice rd(dev);
          Linger linger(teardown);
          if (cfg.compress) warm_codec(rd, warm_sample, cfg.backend);
          arrival.now();
          for (;;) {
            DevFrame f = inbound.pop().value_or(shutdown());
            if (f.head.type == WireFrame::Type::Shutdown) {
              drop(f);
              f.inbox_slot = f.pool_buf = -1;
              f.len = 0;
              outbound.push(f);
              break;
            }
            if (f.head.flags & WireFrame::kFlagCompressed) {
              const double t0 = wire_now_ms();
              const std::size_t need = container_decoded_size(rd, f.payload, f.len);
              const double t1 = wire_now_ms();
              const int b = pool.take(need + 16);
              const double t2 = wire_now_ms();
              std::size_t got = 0;
              try {
                codec_ok(bb_decompress(rd.ctx(), f.payload, f.len, pool.get(b), need, &got, rd.stream()));
              } catch (...) {
                pool.give(b);
                throw;
              }
              const double t3 = wire_now_ms();
              rd.sync();
              dec_ms += wire_now_ms() - t0;
              if (wire_trace())
                std::fprintf(stderr, "[wire] stage %d dec b%llu m%u: size %.3f take %.3f call %.3f sync %.3f ms\n", r,
                             (unsigned long long)f.head.batch, f.head.micro, t1 - t0, t2 - t1, t3 - t2, wire_now_ms() - t3);
              drop(f);
              f.inbox_slot = -1;
              f.pool_buf = b;
              f.payload = pool.get(b);
              f.len = got;
              f.head.flags &= static_cast<std::uint8_t>(~(WireFrame::kFlagCompressed | WireFrame::kFlagByteSplit));
            }
            if (cfg.compute_ms > 0.0) {
              std::this_thread::sleep_for(std::chrono::duration<double, std::milli>(cfg.compute_ms));
              busy_ms += cfg.compute_ms;
            }
            if (cfg.compress) {  // compress_out of every relay stage (run_wire_local, wire.cpp:640)
              const double t0 = wire_now_ms();
              const int b = pool.take(bb_compress_bound(f.len, cfg.backend, 1) + 16);
              const double t1 = wire_now_ms();
              std::size_t len = 0;
              try {
                codec_ok(bb_compress(rd.ctx(), f.payload, f.len, cfg.backend, 1, pool.get(b),
                                     bb_compress_bound(f.len, cfg.backend, 1), &len, rd.stream()));
              } catch (...) {
                pool.give(b);
                throw;
              }
              enc_ms += wire_now_ms() - t0;
              if (wire_trace())
                std::fprintf(stderr, "[wire] stage %d enc b%llu m%u: take %.3f call %.3f ms\n", r,
                             (unsigned long long)f.head.batch, f.head.micro, t1 - t0, wire_now_ms() - t1);
              drop(f);
              f.inbox_slot = -1;
              f.pool_buf = b;
              f.payload = pool.get(b);
              f.len = len;
              f.head.flags |= WireFrame::kFlagCompressed | WireFrame::kFlagByteSplit;
            }
            outbound.push(f);
          }
          linger.hold();
        } catch (...) {
          fail_stage();
        }
      });
      std::thread tx([&] {
        try {
          Arrival arrival(ready);
          RoleDevice rd(dev);
          Linger linger(teardown);
          out.warm(rd);
          arrival.now();
          for (;;) {
            DevFrame f = outbound.pop().value_or(shutdown());
            const bool last = f.head.type == WireFrame::Type::Shutdown;
            FrameSendRecord rec;
            try {
              rec = out.send(rd, f);
            } catch (...) {
              drop(f);
              throw;
            }
            drop(f);
            if (last) break;
            rep.sent.push_back(rec);
          }
          linger.hold();
        } catch (...) {
          fail_stage();
        }
      });
      rx.join();
      work.join();
      tx.join();
      if (failed) return;
      rep.received = std::move(received);
      rep.codec_ms_total = dec_ms + enc_ms;
      rep.frames_seen = rep.received.size();
      if (!rep.received.empty() && !rep.sent.empty())
        rep.metrics.completion_ms = rep.sent.back().t_sent_ms - rep.received.front().t_recv_ms;
      rep.metrics.stages.push_back({busy_ms, rep.metrics.completion_ms - busy_ms});
    });
  }

  // source (wire.cpp:388-429): compress each micro-batch slice in HBM, send it paced
  threads.emplace_back([&] {
    const int r = 0;
    try {
      RoleDevice rd(src_dev);
      Linger linger(teardown);
      if (cfg.compress) warm_codec(rd, warm_sample, cfg.backend);
      hop.front()->warm(rd);
      ready.arrive();
      ready.wait();  // every role is up (or failed): the first offer starts end_to_end_ms
      HopSender& out = *hop.front();
      WireRoleReport& rep = result.source;
      DevBuf frame;
      frame.ensure(src_dev, frame_cap + 16);
      double first_offer = 0.0, last_sent = 0.0;
      for (int s = 0; s < steps; ++s) {
        const std::uint8_t* stream = src_streams[static_cast<std::size_t>(s)].get();
        for (int m = 0; m < cfg.micro_batches; ++m) {
          const auto [off, bytes] = spans[static_cast<std::size_t>(m)];
          DevFrame f;
          f.head.batch = static_cast<std::uint64_t>(s);
          f.head.micro = static_cast<std::uint16_t>(m);
          if (cfg.compress) {
            const double t0 = wire_now_ms();
            std::size_t len = 0;
            codec_ok(bb_compress(rd.ctx(), stream + off, bytes, cfg.backend, 1, frame.get(), frame.cap(), &len,
                                 rd.stream()));
            rep.codec_ms_total += wire_now_ms() - t0;
            f.payload = frame.get();
            f.len = len;
            f.head.flags = WireFrame::kFlagCompressed | WireFrame::kFlagByteSplit;
          } else {
            f.payload = stream + off;
            f.len = bytes;
          }
          FrameSendRecord rec = out.send(rd, f);
          if (rep.sent.empty()) first_offer = rec.t_offer_ms;
          last_sent = rec.t_sent_ms;
          rep.sent.push_back(rec);
          ++rep.frames_seen;
        }
      }
      DevFrame bye;
      bye.head.type = WireFrame::Type::Shutdown;
      out.send(rd, bye);
      rep.metrics.completion_ms = last_sent - first_offer;
      rep.metrics.step_ms = steps > 0 ? rep.metrics.completion_ms / steps : 0.0;
      linger.hold();
    } catch (...) {
      role_failed(r);
    }
  });

  for (auto& t : threads) t.join();
  failure.rethrow();

  const WireRoleReport* sender = &result.source;
  for (const WireRoleReport& st : result.stages) {
    result.hops.push_back(join_hop_metrics(*sender, st));
    sender = &st;
  }
  result.hops.push_back(join_hop_metrics(*sender, result.sink));
  if (!result.source.sent.empty() && !result.sink.received.empty())
    result.end_to_end_ms = result.sink.received.back().t_recv_ms - result.source.sent.front().t_offer_ms;
  result.summary.completion_ms = result.end_to_end_ms;
  result.summary.step_ms = steps > 0 ? result.end_to_end_ms / steps : 0.0;
  result.summary.throughput_tokens_per_s = result.end_to_end_ms > 0 ? steps * 1000.0 / result.end_to_end_ms : 0.0;
  for (const WireRoleReport& st : result.stages)
    for (const StageMetrics& sm : st.metrics.stages) result.summary.stages.push_back(sm);
  result.summary.hops = result.hops;
  if (placement) {
    placement->role_devices = role_dev;
    placement->hop_bytes.clear();
    placement->hop_peer.clear();
    for (int h = 0; h + 1 < roles; ++h) {
      placement->hop_bytes.push_back(hop[static_cast<std::size_t>(h)]->bytes());
      placement->hop_peer.push_back(role_dev[static_cast<std::size_t>(h)] != role_dev[static_cast<std::size_t>(h) + 1]);
    }
  }
  return result;
}

}  // namespace b200

WireLocalResult run_wire_local(const WireLocalConfig& cfg) { return b200::run_wire_local(cfg, b200::WireLocalOptions{}); }

// ---------------------------------------------------------------------------
// JSON (nlohmann/json, the reference's serializer: same keys, dump(2))

std::string run_metrics_to_json(const RunMetrics& m) {
  nlohmann::json doc;
  doc["throughput_tokens_per_s"] = m.throughput_tokens_per_s;
  doc["completion_ms"] = m.completion_ms;
  doc["step_ms"] = m.step_ms;
  doc["stages"] = nlohmann::json::array();
  for (const StageMetrics& s : m.stages) doc["stages"].push_back({{"busy_ms", s.busy_ms}, {"idle_ms", s.idle_ms}});
  doc["hops"] = nlohmann::json::array();
  for (const HopMetrics& h : m.hops)
    doc["hops"].push_back({{"frames", h.frames},
                           {"transfer_ms_total", h.transfer_ms_total},
                           {"transfer_ms_mean", h.transfer_ms_mean},
                           {"compression_ms_total", h.compression_ms_total}});
  return doc.dump(2);
}

std::string wire_report_to_json(const WireRoleReport& rep) {
  nlohmann::json doc;
  doc["metrics"] = nlohmann::json::parse(run_metrics_to_json(rep.metrics));
  doc["codec_ms_total"] = rep.codec_ms_total;
  doc["payload_ok"] = rep.payload_ok;
  doc["frames_seen"] = rep.frames_seen;
  nlohmann::json sent = nlohmann::json::array(), recv = nlohmann::json::array();
  for (const FrameSendRecord& s : rep.sent)
    sent.push_back({{"batch_id", s.batch_id},
                    {"micro_index", s.micro_index},
                    {"t_offer_ms", s.t_offer_ms},
                    {"t_sent_ms", s.t_sent_ms},
                    {"bytes", s.bytes}});
  for (const FrameRecvRecord& r : rep.received)
    recv.push_back({{"batch_id", r.batch_id}, {"micro_index", r.micro_index}, {"t_recv_ms", r.t_recv_ms}, {"bytes", r.bytes}});
  doc["sent"] = std::move(sent);
  doc["received"] = std::move(recv);
  return doc.dump(2);
}

std::string wire_local_result_to_json(const WireLocalResult& res) {
  nlohmann::json doc;
  doc["end_to_end_ms"] = res.end_to_end_ms;
  doc["summary"] = nlohmann::json::parse(run_metrics_to_json(res.summary));
  doc["payload_ok"] = res.sink.payload_ok;
  doc["hops"] = nlohmann::json::array();
  for (const HopMetrics& h : res.hops)
    doc["hops"].push_back({{"frames", h.frames},
                           {"transfer_ms_total", h.transfer_ms_total},
                           {"transfer_ms_mean", h.transfer_ms_mean},
                           {"compression_ms_total", h.compression_ms_total}});
  doc["source_codec_ms"] = res.source.codec_ms_total;
  doc["sink_codec_ms"] = res.sink.codec_ms_total;
  return doc.dump(2);
}

}  // namespace beeplan
