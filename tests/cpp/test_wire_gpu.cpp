// GPU stage-runner cases beyond the reference's test_wire.cpp (TEST INFRASTRUCTURE):
// micro-batch overlap with the GPU codec, multi-GPU placement, NVLink byte accounting,
// failure propagation under injected faults (cf. reference tests/test_wire.cpp:193-243,
// wire.cpp:441-450).  Built by tests/cpp/Makefile, run by tests/test_wire_gpu_runner.py.
#include <doctest.h>

#include <arpa/inet.h>
#include <netinet/in.h>
#include <sys/socket.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <future>
#include <string>

#include "beeplan/errors.hpp"
#include "beeplan/wire.hpp"
#include "beeplan/wire_b200.hpp"

using namespace beeplan;

namespace {

WireLocalConfig relay(int stages, int micro, std::size_t payload, bool compress) {
  WireLocalConfig cfg;
  cfg.steps = 2;
  cfg.micro_batches = micro;
  cfg.payload_bytes = payload;
  cfg.seed = 77;
  cfg.compress = compress;
  cfg.stage_count = stages;
  return cfg;
}

}  // namespace

TEST_CASE("GPU runner: micro-batching overlaps codec, compute and the shaped link (M=4 beats M=1)") {
  auto chain = [](int m) {
    WireLocalConfig cfg = relay(1, m, 416400, true);
    cfg.compute_ms = 160.0 / m;
    cfg.shape.rate_bps = 20e6;
    return run_wire_local(cfg);
  };
  WireLocalResult serial = chain(1), overlapped = chain(4);
  REQUIRE(serial.sink.payload_ok);
  REQUIRE(overlapped.sink.payload_ok);
  std::printf("  M=1 %.1f ms, M=4 %.1f ms\n", serial.end_to_end_ms, overlapped.end_to_end_ms);
  CHECK(overlapped.end_to_end_ms < serial.end_to_end_ms);
}

TEST_CASE("GPU runner: every role on its own GPU, frames bit-exact through 3 relay stages") {
  b200::WireLocalPlacement where;
  WireLocalResult r = b200::run_wire_local(relay(3, 4, 4 << 20, true), b200::WireLocalOptions{}, &where);
  CHECK(r.sink.payload_ok);
  CHECK(r.sink.frames_seen == 8);
  REQUIRE(r.hops.size() == 4);
  for (const HopMetrics& h : r.hops) CHECK(h.frames == 8);
  REQUIRE(where.role_devices.size() == 5);
  REQUIRE(where.hop_bytes.size() == 4);
  for (std::size_t h = 0; h < where.hop_bytes.size(); ++h) {
    CHECK(where.hop_bytes[h] > 0);
    std::printf("  hop %zu: device %d -> %d, %llu B%s\n", h, where.role_devices[h], where.role_devices[h + 1],
                static_cast<unsigned long long>(where.hop_bytes[h]), where.hop_peer[h] ? " (peer copy)" : "");
  }
  // the compressed frames are smaller than the raw micro-batches (header + BBC1 container)
  CHECK(where.hop_bytes[0] < 2ull * (4 << 20));
}

TEST_CASE("GPU runner: uncompressed relay passes the inbox slot through without a copy") {
  WireLocalResult r = run_wire_local(relay(2, 3, 3 * 65536 + 2, false));
  CHECK(r.sink.payload_ok);
  CHECK(r.sink.frames_seen == 6);
}

TEST_CASE("GPU runner: a corrupt frame at a relay stage is FrameCorrupt, and nobody hangs") {
  b200::WireLocalOptions opt;
  opt.fault.kind = b200::WireFault::Kind::CorruptMagic;
  opt.fault.hop = 1;
  opt.fault.frame = 2;
  const auto t0 = std::chrono::steady_clock::now();
  CHECK_THROWS_AS(b200::run_wire_local(relay(2, 4, 1 << 20, true), opt), FrameCorrupt);
  CHECK(std::chrono::steady_clock::now() - t0 < std::chrono::seconds(20));
}

TEST_CASE("GPU runner: a peer vanishing mid-stream is ConnectionLost on every side") {
  b200::WireLocalOptions opt;
  opt.fault.kind = b200::WireFault::Kind::DropLink;
  opt.fault.hop = 0;
  opt.fault.frame = 3;
  CHECK_THROWS_AS(b200::run_wire_local(relay(1, 4, 1 << 20, true), opt), ConnectionLost);
  opt.fault.hop = 2;  // the last hop: the sink sees its upstream close before the shutdown
  CHECK_THROWS_AS(b200::run_wire_local(relay(2, 4, 1 << 20, true), opt), ConnectionLost);
}

TEST_CASE("GPU runner: compression shortens a 100 Mbps hop on Gaussian activations") {
  auto run = [](bool compress) {
    WireLocalConfig cfg = relay(0, 1, 1 << 20, compress);
    cfg.shape.rate_bps = 100e6;
    return run_wire_local(cfg);
  };
  WireLocalResult plain = run(false), squeezed = run(true);
  REQUIRE(plain.sink.payload_ok);
  REQUIRE(squeezed.sink.payload_ok);
  std::printf("  1 MiB frame at 100 Mbps: raw %.1f ms, compressed %.1f ms\n", plain.hops[0].transfer_ms_mean,
              squeezed.hops[0].transfer_ms_mean);
  CHECK(squeezed.hops[0].transfer_ms_mean < plain.hops[0].transfer_ms_mean);
}

TEST_CASE("GPU runner: odd payloads and bad stage counts are ValidationError") {
  CHECK_THROWS_AS(run_wire_local(relay(1, 1, 1001, false)), ValidationError);
  CHECK_THROWS_AS(run_wire_local(relay(-1, 1, 1000, false)), ValidationError);
}

namespace {

int bound_listener(std::string* endpoint) {
  int fd = ::socket(AF_INET, SOCK_STREAM, 0);
  sockaddr_in sin{};
  sin.sin_family = AF_INET;
  sin.sin_port = 0;
  inet_pton(AF_INET, "127.0.0.1", &sin.sin_addr);
  if (fd < 0 || ::bind(fd, reinterpret_cast<sockaddr*>(&sin), sizeof(sin)) != 0 || ::listen(fd, 4) != 0) return -1;
  socklen_t len = sizeof(sin);
  ::getsockname(fd, reinterpret_cast<sockaddr*>(&sin), &len);
  *endpoint = "127.0.0.1:" + std::to_string(ntohs(sin.sin_port));
  return fd;
}

}  // namespace

TEST_CASE("TCP roles: source -> stage -> sink over loopback sockets, codec on the GPU, bit-exact") {
  std::string stage_ep, sink_ep;
  const int stage_fd = bound_listener(&stage_ep), sink_fd = bound_listener(&sink_ep);
  REQUIRE(stage_fd >= 0);
  REQUIRE(sink_fd >= 0);
  WireSinkConfig sk;
  sk.payload_bytes = 1 << 20;
  sk.micro_batches = 4;
  sk.seed = 3;
  sk.listen_fd = sink_fd;
  WireStageConfig sg;
  sg.listen_fd = stage_fd;
  sg.connect = sink_ep;
  sg.compress_out = true;
  sg.compute_ms = 1.0;
  WireSourceConfig so;
  so.connect = stage_ep;
  so.steps = 2;
  so.micro_batches = 4;
  so.payload_bytes = 1 << 20;
  so.seed = 3;
  so.compress = true;
  so.shape.rate_bps = 400e6;
  auto sink = std::async(std::launch::async, [&] { return run_wire_sink(sk); });
  auto stage = std::async(std::launch::async, [&] { return run_wire_stage(sg); });
  auto source = std::async(std::launch::async, [&] { return run_wire_source(so); });
  WireRoleReport src = source.get(), st = stage.get(), dst = sink.get();
  CHECK(dst.payload_ok);
  CHECK(dst.frames_seen == 8);
  CHECK(st.frames_seen == 8);
  CHECK(src.codec_ms_total > 0.0);
  CHECK(st.codec_ms_total > 0.0);
  const HopMetrics h0 = join_hop_metrics(src, st), h1 = join_hop_metrics(st, dst);
  CHECK(h0.frames == 8);
  CHECK(h1.frames == 8);
  ::close(stage_fd);
  ::close(sink_fd);
}

TEST_CASE("GPU runner: identity backend, empty micro-batches and zero steps") {
  WireLocalConfig cfg = relay(1, 4, 4, true);  // 2 elements over 4 micro-batches: two empty spans
  cfg.backend = kBackendIdentity;
  WireLocalResult r = run_wire_local(cfg);
  CHECK(r.sink.payload_ok);
  CHECK(r.sink.frames_seen == 8);
  WireLocalConfig none = relay(2, 2, 1 << 16, true);
  none.steps = 0;
  WireLocalResult z = run_wire_local(none);
  CHECK(z.sink.payload_ok);
  CHECK(z.sink.frames_seen == 0);
  CHECK(z.end_to_end_ms == 0.0);
}

TEST_CASE("GPU runner: queue_slots = 1 and a long relay keep every frame in order") {
  b200::WireLocalOptions opt;
  opt.queue_slots = 1;
  WireLocalConfig cfg = relay(5, 6, 3 << 20, true);
  cfg.steps = 3;
  WireLocalResult r = b200::run_wire_local(cfg, opt);
  CHECK(r.sink.payload_ok);
  CHECK(r.sink.frames_seen == 18);
  for (const HopMetrics& h : r.hops) CHECK(h.frames == 18);
}
