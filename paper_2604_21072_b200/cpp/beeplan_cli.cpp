// beeplan (B200 build): the codec and stage hand-off subcommands of the
// reference CLI on the GPU codec, with the same arguments, JSON documents and
// exit codes (reference proj/tools/beeplan_main.cpp:164-239 handlers,
// :289-324 options, :326-351 exit codes; proj/tests/cli_tests.sh:74-104).
//
//   beeplan [--seed N] [--output PATH] [--format json] <subcommand> ...
//     compress <input> <output> [--backend identity|deflate] [--no-split]
//     decompress <input> <output>
//     entropy <input> [--backend identity|deflate]
//     bench-wire --role local|source|stage|sink [--payload B] [--micro-batches M] [--steps S]
//                [--shape rate_mbps,latency_ms] [--compute-ms X] [--compress] [--stages K]
//                [--listen H:P] [--connect H:P] [--devices 0,1,..] [--placement PATH]
//
// Exit codes: 0 ok, 1 domain error ({"error": ...} on stderr) or a lossy
// bench-wire run, 2 usage error.  bench-wire calls the stage API drop-in
// (include/beeplan/wire.hpp, cpp/wire.cpp): --role local is the multi-GPU runner
// (one GPU per role, frames in HBM, ShapedWriter-paced peer copies), the TCP roles
// relay host frames over sockets with the codec on the GPU.  The planner
// subcommands are outside this build.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <exception>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "beeplan/codec.hpp"
#include "beeplan/errors.hpp"
#include "beeplan/synth.hpp"
#include "beeplan/wire.hpp"
#include "beeplan/wire_b200.hpp"

#include <nlohmann/json.hpp>

namespace {

using beeplan::Bytes;
using J = nlohmann::json;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};


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
                                                "--stages", "--devices", "--placement", "--reports"};
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

beeplan::LinkShape parse_shape(const std::string& text) {  // beeplan_main.cpp:58-68
  const auto comma = text.find(',');
  if (comma == std::string::npos) throw beeplan::ValidationError("--shape: expected rate_mbps,latency_ms");
  const std::string rate = text.substr(0, comma);
  beeplan::LinkShape s;
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
    "  bench-wire --role local|source|stage|sink [--payload B] [--micro-batches M] [--steps S]\n"
    "             [--shape R,L] [--compute-ms X] [--compress] [--stages K] [--listen H:P] [--connect H:P]\n"
    "             [--devices 0,1,..] [--placement PATH]   (local: one GPU per role, frames in HBM)\n";

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
  if (a.sub == "bench-wire") {  // beeplan_main.cpp:188-239
    need(0);
    if (!a.opt.count("--role")) throw UsageError("--role is required");
    const std::string role = a.opt.at("--role");
    const beeplan::LinkShape shape = a.opt.count("--shape") ? parse_shape(a.opt.at("--shape")) : beeplan::LinkShape{};
    const int steps = num<int>(a, "--steps", 1), micro = num<int>(a, "--micro-batches", 1);
    const size_t payload = num<size_t>(a, "--payload", 416400);
    const double compute_ms = num<double>(a, "--compute-ms", 0.0);
    const bool compress = a.flags.count("--compress") > 0;
    const std::string listen = a.opt.count("--listen") ? a.opt.at("--listen") : "";
    const std::string connect = a.opt.count("--connect") ? a.opt.at("--connect") : "";
    if (role == "local") {  // one GPU per role, frames in HBM, paced peer copies
      beeplan::WireLocalConfig cfg;
      cfg.steps = steps;
      cfg.micro_batches = micro;
      cfg.payload_bytes = payload;
      cfg.seed = seed;
      cfg.compress = compress;
      cfg.stage_count = num<int>(a, "--stages", 1);
      cfg.compute_ms = compute_ms;
      cfg.shape = shape;
      beeplan::b200::WireLocalOptions opt;
      if (a.opt.count("--devices")) {
        std::stringstream ds(a.opt.at("--devices"));
        for (std::string d; std::getline(ds, d, ',');)
          if (!d.empty()) opt.devices.push_back(std::stoi(d));
      }
      beeplan::b200::WireLocalPlacement where;
      const beeplan::WireLocalResult r = beeplan::b200::run_wire_local(cfg, opt, &where);
      if (a.opt.count("--placement")) {
        J p;
        p["role_devices"] = where.role_devices;
        p["hop_bytes"] = where.hop_bytes;
        p["hop_peer"] = where.hop_peer;
        std::ofstream(a.opt.at("--placement")) << p.dump(2) << "\n";
      }
      if (a.opt.count("--reports")) {  // every role's records (wire_report_to_json), for diagnosis
        J all;
        all["source"] = J::parse(beeplan::wire_report_to_json(r.source));
        all["stages"] = J::array();
        for (const auto& st : r.stages) all["stages"].push_back(J::parse(beeplan::wire_report_to_json(st)));
        all["sink"] = J::parse(beeplan::wire_report_to_json(r.sink));
        std::ofstream(a.opt.at("--reports")) << all.dump(1) << "\n";
      }
      write_output(output, beeplan::wire_local_result_to_json(r));
      return r.sink.payload_ok ? 0 : 1;
    }
    beeplan::WireRoleReport report;
    if (role == "source") {
      beeplan::WireSourceConfig cfg;
      cfg.connect = connect;
      cfg.steps = steps;
      cfg.micro_batches = micro;
      cfg.payload_bytes = payload;
      cfg.seed = seed;
      cfg.compress = compress;
      cfg.shape = shape;
      report = beeplan::run_wire_source(cfg);
    } else if (role == "stage") {
      beeplan::WireStageConfig cfg;
      cfg.listen = listen;
      cfg.connect = connect;
      cfg.compute_ms = compute_ms;
      cfg.compress_out = compress;
      cfg.shape = shape;
      report = beeplan::run_wire_stage(cfg);
    } else if (role == "sink") {
      beeplan::WireSinkConfig cfg;
      cfg.listen = listen;
      cfg.payload_bytes = payload;
      cfg.micro_batches = micro;
      cfg.seed = seed;
      report = beeplan::run_wire_sink(cfg);
    } else {
      throw beeplan::ValidationError("--role: expected source|stage|sink|local");
    }
    write_output(output, beeplan::wire_report_to_json(report));
    return report.payload_ok ? 0 : 1;
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
