// beeplan (B200 build): the codec and stage hand-off subcommands of the
// reference CLI on the GPU codec, with the same arguments, JSON documents and
// exit codes (reference proj/tools/beeplan_main.cpp:164-239 handlers,
// :289-324 options, :326-351 exit codes; proj/tests/cli_tests.sh:74-104).
//
//   beeplan [--seed N] [--output PATH] [--format json] <subcommand> ...
//     compress <input> <output> [--backend identity|deflate] [--no-split]
//     decompress <input> <output>
//     entropy <input> [--backend identity|deflate]
//     bench-wire --role local [--payload B] [--micro-batches M] [--steps S]
//                [--shape rate_mbps,latency_ms] [--compute-ms X] [--compress] [--stages K]
//
// Exit codes: 0 ok, 1 domain error ({"error": ...} on stderr) or a lossy
// bench-wire run, 2 usage error.  bench-wire --role local runs the reference's
// loopback harness (wire.cpp:604-684) in-process: source, relay stages (recv /
// compute / send threads with 2-slot queues, wire.cpp:431-541) and sink,
// linked by ShapedWriter-paced hops (wire.cpp:201-248) instead of TCP sockets;
// every compress / decompress runs on the GPU.  The TCP roles
// (source / stage / sink) and the planner subcommands are outside this build.
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <deque>
#include <exception>
#include <fstream>
#include <iostream>
#include <map>
#include <mutex>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "beeplan/codec.hpp"
#include "beeplan/errors.hpp"
#include "beeplan/synth.hpp"

#include <nlohmann/json.hpp>

namespace {

using beeplan::Bytes;
using J = nlohmann::json;
using Clock = std::chrono::steady_clock;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

double now_ms() {
  return std::chrono::duration<double, std::milli>(Clock::now().time_since_epoch()).count();
}

Bytes read_bytes(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw beeplan::ParseError("cannot open file: " + path);
  std::ostringstream buf;
  buf << in.rdbuf();
  const std::string s = buf.str();
  return Bytes(s.begin(), s.end());
}

void write_bytes(const std::string& path, const Bytes& data) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw beeplan::Error("cannot open output file: " + path);
  out.write(reinterpret_cast<const char*>(data.data()), (std::streamsize)data.size());
}

void write_output(const std::string& output, const std::string& text) {
  if (output.empty() || output == "-") {
    std::cout << text << "\n";
    return;
  }
  std::ofstream out(output, std::ios::binary);
  if (!out) throw beeplan::Error("cannot open output file: " + output);
  out << text << "\n";
}

// ---------------------------------------------------------------------------
// command line (CLI11-compatible subset: options before or after the subcommand,
// "--opt value" or "--opt=value", flags, positionals)
struct Args {
  std::string sub;
  std::vector<std::string> pos;
  std::map<std::string, std::string> opt;
  std::set<std::string> flags;
  bool help = false;
};

Args parse_args(int argc, char** argv) {
  static const std::set<std::string> kValued = {"--seed",   "--output",        "--format", "--backend",
                                                "--role",   "--listen",        "--connect", "--shape",
                                                "--payload", "--micro-batches", "--steps",  "--compute-ms",
                                                "--stages"};
  static const std::set<std::string> kFlags = {"--no-split", "--compress"};
  Args a;
  for (int i = 1; i < argc; i++) {
    std::string t = argv[i];
    if (t == "-h" || t == "--help") {
      a.help = true;
      continue;
    }
    if (t.rfind("--", 0) == 0) {
      std::string name = t, val;
      const auto eq = t.find('=');
      if (eq != std::string::npos) name = t.substr(0, eq), val = t.substr(eq + 1);
      if (kFlags.count(name)) {
        a.flags.insert(name);
      } else if (kValued.count(name)) {
        if (eq == std::string::npos) {
          if (i + 1 >= argc) throw UsageError(name + " requires an argument");
          val = argv[++i];
        }
        a.opt[name] = val;
      } else {
        throw UsageError("The following argument was not expected: " + t);
      }
    } else if (a.sub.empty()) {
      a.sub = t;
    } else {
      a.pos.push_back(t);
    }
  }
  return a;
}

template <class T>
T num(const Args& a, const std::string& name, T dflt) {
  auto it = a.opt.find(name);
  if (it == a.opt.end()) return dflt;
  try {
    size_t used = 0;
    T v;
    if constexpr (std::is_floating_point_v<T>) v = (T)std::stod(it->second, &used);
    else if constexpr (std::is_signed_v<T>) v = (T)std::stoll(it->second, &used);
    else v = (T)std::stoull(it->second, &used);
    if (used != it->second.size()) throw std::invalid_argument("trailing");
    return v;
  } catch (const std::exception&) {
    throw UsageError(name + ": Value " + it->second + " could not be converted");
  }
}

// ---------------------------------------------------------------------------
// BBF1 frames (wire.hpp:14-29, wire.cpp:342-370)
constexpr size_t kFrameHeader = 20;
enum : uint8_t { kActivations = 0, kPackedSd = 1, kAck = 2, kShutdown = 3 };
enum : uint8_t { kFlagCompressed = 0x01, kFlagByteSplit = 0x02 };

struct Frame {
  uint8_t type = kActivations;
  uint64_t batch = 0;
  uint16_t micro = 0;
  uint8_t flags = 0;
  Bytes payload;
};

Bytes encode_frame(const Frame& f) {
  Bytes out = {'B', 'B', 'F', '1', f.type};
  for (int k = 0; k < 8; k++) out.push_back((uint8_t)(f.batch >> (8 * k)));
  out.push_back((uint8_t)f.micro), out.push_back((uint8_t)(f.micro >> 8));
  out.push_back(f.flags);
  const uint32_t n = (uint32_t)f.payload.size();
  for (int k = 0; k < 4; k++) out.push_back((uint8_t)(n >> (8 * k)));
  out.insert(out.end(), f.payload.begin(), f.payload.end());
  return out;
}

Frame decode_frame(const Bytes& b) {
  if (b.size() < kFrameHeader) throw beeplan::FrameCorrupt("frame: truncated header");
  if (std::memcmp(b.data(), "BBF1", 4) != 0) throw beeplan::FrameCorrupt("frame: bad magic");
  Frame f;
  f.type = b[4];
  if (f.type > 3) throw beeplan::FrameCorrupt("frame: unknown msg_type " + std::to_string(f.type));
  for (int k = 0; k < 8; k++) f.batch |= (uint64_t)b[5 + k] << (8 * k);
  f.micro = (uint16_t)(b[13] | (b[14] << 8));
  f.flags = b[15];
  uint32_t n = 0;
  for (int k = 0; k < 4; k++) n |= (uint32_t)b[16 + k] << (8 * k);
  if (b.size() != kFrameHeader + n) throw beeplan::FrameCorrupt("frame: payload length does not match the header");
  f.payload.assign(b.begin() + kFrameHeader, b.end());
  return f;
}

// per-step synthetic stream and its micro-batch spans (wire.cpp:315-336)
struct StepSlices {
  Bytes stream;
  std::vector<std::pair<size_t, size_t>> spans;
};
StepSlices make_step_slices(size_t payload, int micro, uint64_t seed, uint64_t step) {
  if (payload % 2 != 0) throw beeplan::ValidationError("payload_bytes: must be even (FP16)");
  if (micro < 1) throw beeplan::ValidationError("micro_batches: must be >= 1");
  const size_t elements = payload / 2;
  StepSlices s;
  s.stream = beeplan::synth_gaussian_fp16(elements, seed + step);
  const size_t base = elements / (size_t)micro, rem = elements % (size_t)micro;
  size_t off = 0;
  for (int k = 0; k < micro; k++) {
    const size_t e = base + ((size_t)k < rem ? 1 : 0);
    s.spans.emplace_back(off * 2, e * 2);
    off += e;
  }
  return s;
}

// ---------------------------------------------------------------------------
// in-process hop: the ShapedWriter's pacing on the sender, a bounded byte queue
// standing in for the socket
struct SendRec {
  uint64_t batch;
  uint16_t micro;
  double t_offer, t_sent;
  size_t bytes;
};
struct RecvRec {
  uint64_t batch;
  uint16_t micro;
  double t_recv;
  size_t bytes;
};

class BoundedQueue {
 public:
  explicit BoundedQueue(size_t cap) : cap_(cap) {}
  void push(Bytes b) {
    std::unique_lock<std::mutex> l(m_);
    cv_.wait(l, [&] { return q_.size() < cap_; });
    q_.push_back(std::move(b));
    cv_.notify_all();
  }
  Bytes pop() {
    std::unique_lock<std::mutex> l(m_);
    cv_.wait(l, [&] { return !q_.empty(); });
    Bytes b = std::move(q_.front());
    q_.pop_front();
    cv_.notify_all();
    return b;
  }

 private:
  size_t cap_;
  std::deque<Bytes> q_;
  std::mutex m_;
  std::condition_variable cv_;
};

struct Shape {
  double rate_bps = 0, latency_ms = 0;
};

class Hop {
 public:
  Hop(Shape s) : shape_(s), q_(4) {}
  SendRec send(const Bytes& bytes, uint64_t batch, uint16_t micro) {
    SendRec r{batch, micro, now_ms(), 0, bytes.size()};
    const auto lat = std::chrono::duration_cast<Clock::duration>(std::chrono::duration<double>(shape_.latency_ms / 1e3));
    if (shape_.rate_bps <= 0) {
      if (shape_.latency_ms > 0) std::this_thread::sleep_until(Clock::now() + lat);
    } else {
      const double rate = shape_.rate_bps / 8.0;
      for (size_t off = 0; off < bytes.size();) {
        const size_t chunk = std::min<size_t>(64 * 1024, bytes.size() - off);
        const auto now = Clock::now();
        if (wire_free_ < now) wire_free_ = now;
        wire_free_ += std::chrono::duration_cast<Clock::duration>(std::chrono::duration<double>(chunk / rate));
        std::this_thread::sleep_until(wire_free_ + lat);
        off += chunk;
      }
    }
    q_.push(bytes);
    r.t_sent = now_ms();
    return r;
  }
  Bytes recv(double* t) {
    Bytes b = q_.pop();
    *t = now_ms();
    return b;
  }

 private:
  Shape shape_;
  BoundedQueue q_;
  Clock::time_point wire_free_{};
};

class FrameQueue {  // wire.cpp:269-313 (capacity = queue_slots)
 public:
  explicit FrameQueue(size_t cap) : cap_(cap) {}
  void push(Frame f) {
    std::unique_lock<std::mutex> l(m_);
    cv_.wait(l, [&] { return q_.size() < cap_; });
    q_.push_back(std::move(f));
    cv_.notify_all();
  }
  Frame pop() {
    std::unique_lock<std::mutex> l(m_);
    cv_.wait(l, [&] { return !q_.empty(); });
    Frame f = std::move(q_.front());
    q_.pop_front();
    cv_.notify_all();
    return f;
  }

 private:
  size_t cap_;
  std::deque<Frame> q_;
  std::mutex m_;
  std::condition_variable cv_;
};

struct RoleReport {
  std::vector<SendRec> sent;
  std::vector<RecvRec> received;
  double codec_ms = 0, completion_ms = 0, step_ms = 0;
  std::vector<std::pair<double, double>> stages;  // busy, idle
  bool payload_ok = true;
  uint64_t frames_seen = 0;
};

struct HopMetrics {
  int frames = 0;
  double total = 0, mean = 0, comp = 0;
};

HopMetrics join_hop(const RoleReport& tx, const RoleReport& rx) {  // wire.cpp:372-386
  HopMetrics h;
  for (const SendRec& s : tx.sent)
    for (const RecvRec& r : rx.received)
      if (r.batch == s.batch && r.micro == s.micro) {
        h.total += r.t_recv - s.t_offer;
        h.frames++;
        break;
      }
  h.mean = h.frames ? h.total / h.frames : 0.0;
  h.comp = tx.codec_ms;
  return h;
}

struct LocalCfg {
  int steps = 1, micro = 1, stages = 1;
  size_t payload = 0;
  uint64_t seed = 1;
  bool compress = false;
  double compute_ms = 0;
  Shape shape;
};

Bytes compress_frame_payload(const Bytes& raw, double& codec_ms) {
  const double t0 = now_ms();
  Bytes c = beeplan::serialize_container(beeplan::compress(raw, beeplan::kBackendDeflate, true));
  codec_ms += now_ms() - t0;
  return c;
}

Bytes decompress_frame_payload(const Bytes& c, double& codec_ms) {
  const double t0 = now_ms();
  Bytes raw = beeplan::decompress(beeplan::parse_container(c));
  codec_ms += now_ms() - t0;
  return raw;
}

void run_source(const LocalCfg& cfg, Hop& out, RoleReport& rep) {  // wire.cpp:388-429
  double first = 0, last = 0;
  for (int step = 0; step < cfg.steps; step++) {
    const StepSlices sl = make_step_slices(cfg.payload, cfg.micro, cfg.seed, (uint64_t)step);
    for (int m = 0; m < cfg.micro; m++) {
      const auto [off, n] = sl.spans[(size_t)m];
      Frame f;
      f.batch = (uint64_t)step;
      f.micro = (uint16_t)m;
      Bytes slice(sl.stream.begin() + (ptrdiff_t)off, sl.stream.begin() + (ptrdiff_t)(off + n));
      if (cfg.compress) {
        f.payload = compress_frame_payload(slice, rep.codec_ms);
        f.flags = kFlagCompressed | kFlagByteSplit;
      } else {
        f.payload = std::move(slice);
      }
      const SendRec r = out.send(encode_frame(f), f.batch, f.micro);
      if (rep.sent.empty()) first = r.t_offer;
      last = r.t_sent;
      rep.sent.push_back(r);
      rep.frames_seen++;
    }
  }
  Frame shut;
  shut.type = kShutdown;
  out.send(encode_frame(shut), 0, 0);
  rep.completion_ms = last - first;
  rep.step_ms = cfg.steps > 0 ? rep.completion_ms / cfg.steps : 0.0;
}

void run_stage(const LocalCfg& cfg, Hop& in, Hop& out, RoleReport& rep) {  // wire.cpp:431-541
  FrameQueue inbound(2), outbound(2);
  double recv_codec = 0, send_codec = 0, busy = 0;
  std::exception_ptr failure;
  std::mutex fm;
  auto fail = [&] {
    std::lock_guard<std::mutex> l(fm);
    if (!failure) failure = std::current_exception();
  };
  std::thread rx([&] {
    try {
      for (;;) {
        double t = 0;
        Frame f = decode_frame(in.recv(&t));
        const bool shut = f.type == kShutdown;
        if (!shut) rep.received.push_back({f.batch, f.micro, t, kFrameHeader + f.payload.size()});
        inbound.push(std::move(f));
        if (shut) break;
      }
    } catch (...) {
      fail();
      Frame p;
      p.type = kShutdown;
      inbound.push(std::move(p));
    }
  });
  std::thread cx([&] {
    try {
      for (;;) {
        Frame f = inbound.pop();
        if (f.type == kShutdown) {
          outbound.push(std::move(f));
          break;
        }
        if (f.flags & kFlagCompressed) {
          f.payload = decompress_frame_payload(f.payload, recv_codec);
          f.flags &= (uint8_t)~(kFlagCompressed | kFlagByteSplit);
        }
        if (cfg.compute_ms > 0) {
          std::this_thread::sleep_for(std::chrono::duration<double>(cfg.compute_ms / 1e3));
          busy += cfg.compute_ms;
        }
        if (cfg.compress) {
          f.payload = compress_frame_payload(f.payload, send_codec);
          f.flags |= kFlagCompressed | kFlagByteSplit;
        }
        outbound.push(std::move(f));
      }
    } catch (...) {
      fail();
      Frame p;
      p.type = kShutdown;
      outbound.push(std::move(p));
    }
  });
  std::thread tx([&] {
    try {
      for (;;) {
        Frame f = outbound.pop();
        const bool shut = f.type == kShutdown;
        const SendRec r = out.send(encode_frame(f), f.batch, f.micro);
        if (!shut) rep.sent.push_back(r);
        if (shut) break;
      }
    } catch (...) {
      fail();
    }
  });
  rx.join();
  cx.join();
  tx.join();
  if (failure) std::rethrow_exception(failure);
  rep.codec_ms = recv_codec + send_codec;
  rep.frames_seen = rep.received.size();
  if (!rep.received.empty() && !rep.sent.empty())
    rep.completion_ms = rep.sent.back().t_sent - rep.received.front().t_recv;
  rep.stages.push_back({busy, rep.completion_ms - busy});
}

void run_sink(const LocalCfg& cfg, Hop& in, RoleReport& rep) {  // wire.cpp:543-602
  uint64_t cur = ~0ull;
  StepSlices want;
  Bytes got;
  auto finish = [&] {
    if (cur == ~0ull) return;
    if (got != want.stream) rep.payload_ok = false;
  };
  for (;;) {
    double t = 0;
    Frame f = decode_frame(in.recv(&t));
    if (f.type == kShutdown) break;
    rep.received.push_back({f.batch, f.micro, t, kFrameHeader + f.payload.size()});
    rep.frames_seen++;
    if (f.type != kActivations) continue;
    if (f.batch != cur) {
      finish();
      cur = f.batch;
      want = make_step_slices(cfg.payload, cfg.micro, cfg.seed, cur);
      got.assign(want.stream.size(), 0);
    }
    if (f.micro >= want.spans.size())
      throw beeplan::FrameCorrupt("sink: micro_index " + std::to_string(f.micro) +
                                  " outside the configured micro-batch count");
    Bytes p = f.payload;
    if (f.flags & kFlagCompressed) p = decompress_frame_payload(p, rep.codec_ms);
    const auto [off, n] = want.spans[f.micro];
    if (p.size() != n) rep.payload_ok = false;
    else std::copy(p.begin(), p.end(), got.begin() + (ptrdiff_t)off);
  }
  finish();
  if (!rep.received.empty()) rep.completion_ms = rep.received.back().t_recv - rep.received.front().t_recv;
}

J hop_json(const HopMetrics& h) {
  return {{"frames", h.frames},
          {"transfer_ms_total", h.total},
          {"transfer_ms_mean", h.mean},
          {"compression_ms_total", h.comp}};
}

int run_bench_wire_local(const std::string& output, const LocalCfg& cfg) {  // wire.cpp:604-684
  if (cfg.stages < 0) throw beeplan::ValidationError("stage_count: must be >= 0");
  std::vector<std::unique_ptr<Hop>> hops;
  for (int i = 0; i <= cfg.stages; i++) hops.push_back(std::make_unique<Hop>(cfg.shape));
  RoleReport src, snk;
  std::vector<RoleReport> st((size_t)cfg.stages);
  std::exception_ptr failure;
  std::mutex fm;
  auto guard = [&](auto&& fn) {
    try {
      fn();
    } catch (...) {
      std::lock_guard<std::mutex> l(fm);
      if (!failure) failure = std::current_exception();
    }
  };
  std::vector<std::thread> th;
  th.emplace_back([&] { guard([&] { run_sink(cfg, *hops.back(), snk); }); });
  for (int i = cfg.stages - 1; i >= 0; i--)
    th.emplace_back([&, i] { guard([&] { run_stage(cfg, *hops[(size_t)i], *hops[(size_t)i + 1], st[(size_t)i]); }); });
  th.emplace_back([&] { guard([&] { run_source(cfg, *hops.front(), src); }); });
  for (auto& t : th) t.join();
  if (failure) std::rethrow_exception(failure);

  std::vector<HopMetrics> hm;
  const RoleReport* tx = &src;
  for (const RoleReport& s : st) {
    hm.push_back(join_hop(*tx, s));
    tx = &s;
  }
  hm.push_back(join_hop(*tx, snk));
  double e2e = 0;
  if (!src.sent.empty() && !snk.received.empty()) e2e = snk.received.back().t_recv - src.sent.front().t_offer;

  // wire_local_result_to_json (wire.cpp:710-724) with run_metrics_to_json (simulator.cpp:193-208)
  J summary;
  summary["throughput_tokens_per_s"] = e2e > 0 ? cfg.steps * 1000.0 / e2e : 0.0;
  summary["completion_ms"] = e2e;
  summary["step_ms"] = cfg.steps > 0 ? e2e / cfg.steps : 0.0;
  summary["stages"] = J::array();
  for (const RoleReport& s : st)
    for (const auto& [b, idle] : s.stages) summary["stages"].push_back({{"busy_ms", b}, {"idle_ms", idle}});
  summary["hops"] = J::array();
  for (const HopMetrics& h : hm) summary["hops"].push_back(hop_json(h));
  J doc;
  doc["end_to_end_ms"] = e2e;
  doc["summary"] = summary;
  doc["payload_ok"] = snk.payload_ok;
  doc["hops"] = J::array();
  for (const HopMetrics& h : hm) doc["hops"].push_back(hop_json(h));
  doc["source_codec_ms"] = src.codec_ms;
  doc["sink_codec_ms"] = snk.codec_ms;
  write_output(output, doc.dump(2));
  return snk.payload_ok ? 0 : 1;
}

Shape parse_shape(const std::string& text) {  // beeplan_main.cpp:58-68
  const auto comma = text.find(',');
  if (comma == std::string::npos) throw beeplan::ValidationError("--shape: expected rate_mbps,latency_ms");
  const std::string rate = text.substr(0, comma);
  Shape s;
  try {
    s.rate_bps = rate == "inf" ? 0.0 : std::stod(rate) * 1e6;
    s.latency_ms = std::stod(text.substr(comma + 1));
  } catch (const std::logic_error&) {
    throw beeplan::ValidationError("--shape: expected rate_mbps,latency_ms");
  }
  return s;
}

const char* kUsage =
    "beeplan (B200 codec build): GPU codec and stage hand-off subcommands\n"
    "Usage: beeplan [--seed N] [--output PATH] [--format json] SUBCOMMAND ...\n"
    "  compress INPUT OUTPUT [--backend identity|deflate] [--no-split]\n"
    "  decompress INPUT OUTPUT\n"
    "  entropy INPUT [--backend identity|deflate]\n"
    "  bench-wire --role local [--payload B] [--micro-batches M] [--steps S] [--shape R,L]\n"
    "             [--compute-ms X] [--compress] [--stages K]\n";

int dispatch(const Args& a) {
  const std::string output = a.opt.count("--output") ? a.opt.at("--output") : "";
  const uint64_t seed = num<uint64_t>(a, "--seed", 1);
  if (a.opt.count("--format") && a.opt.at("--format") != "json")
    throw UsageError("--format: " + a.opt.at("--format") + " not in {json}");
  auto need = [&](size_t k) {
    if (a.pos.size() < k) throw UsageError(a.sub + ": missing positional arguments");
    if (a.pos.size() > k) throw UsageError("The following argument was not expected: " + a.pos[k]);
  };
  const std::string backend = a.opt.count("--backend") ? a.opt.at("--backend") : "deflate";
  if (a.sub == "compress") {
    need(2);
    const Bytes data = read_bytes(a.pos[0]);
    const beeplan::CodecContainer c =
        beeplan::compress(data, beeplan::backend_by_name(backend).id, !a.flags.count("--no-split"));
    write_bytes(a.pos[1], beeplan::serialize_container(c));
    return 0;
  }
  if (a.sub == "decompress") {
    need(2);
    write_bytes(a.pos[1], beeplan::decompress(beeplan::parse_container(read_bytes(a.pos[0]))));
    return 0;
  }
  if (a.sub == "entropy") {
    need(1);
    const Bytes data = read_bytes(a.pos[0]);
    write_output(output, beeplan::entropy_report_to_json(beeplan::analyze(data, beeplan::backend_by_name(backend).id)));
    return 0;
  }
  if (a.sub == "bench-wire") {
    need(0);
    if (!a.opt.count("--role")) throw UsageError("--role is required");
    const std::string role = a.opt.at("--role");
    if (role != "local") {
      if (role == "source" || role == "stage" || role == "sink")
        throw beeplan::ValidationError("--role " + role +
                                       ": the TCP roles are not part of the B200 build; use --role local "
                                       "or python -m paper_2604_21072_b200.pipeline (NVLink)");
      throw beeplan::ValidationError("--role: expected source|stage|sink|local");
    }
    LocalCfg cfg;
    cfg.steps = num<int>(a, "--steps", 1);
    cfg.micro = num<int>(a, "--micro-batches", 1);
    cfg.payload = num<size_t>(a, "--payload", 416400);
    cfg.stages = num<int>(a, "--stages", 1);
    cfg.compute_ms = num<double>(a, "--compute-ms", 0.0);
    cfg.compress = a.flags.count("--compress") > 0;
    cfg.seed = seed;
    if (a.opt.count("--shape")) cfg.shape = parse_shape(a.opt.at("--shape"));
    return run_bench_wire_local(output, cfg);
  }
  if (a.sub == "plan" || a.sub == "simulate" || a.sub == "analyze-sd")
    throw UsageError(a.sub + ": planner subcommands are not part of the B200 codec build");
  throw UsageError(a.sub.empty() ? "A subcommand is required" : "The following argument was not expected: " + a.sub);
}

}  // namespace

int main(int argc, char** argv) {
  Args a;
  try {
    a = parse_args(argc, argv);
    if (a.help) {
      std::cout << kUsage;
      return 0;
    }
    if (a.sub.empty()) throw UsageError("A subcommand is required");
  } catch (const UsageError& e) {
    std::cerr << e.what() << "\nRun with --help for more information.\n";
    return 2;
  }
  try {
    return dispatch(a);
  } catch (const UsageError& e) {
    std::cerr << e.what() << "\nRun with --help for more information.\n";
    return 2;
  } catch (const beeplan::Error& e) {
    std::cerr << J{{"error", e.what()}}.dump() << "\n";
    return 1;
  }
}
