// SPDX-License-Identifier: Apache-2.0
// B200 extensions of the stage API (include/beeplan/wire.hpp): device placement of the
// in-process multi-GPU runner, its per-hop NVLink byte counts, and fault injection for
// the failure-propagation tests.  Not part of the reference interface.
#pragma once

#include <cstdint>
#include <vector>

#include "beeplan/wire.hpp"

namespace beeplan::b200 {

struct WireFault {
  enum class Kind { None, CorruptMagic, DropLink };
  Kind kind = Kind::None;
  int hop = 0;    // 0 = source -> first receiver
  int frame = 0;  // n-th frame the hop's sender offers
};

struct WireLocalOptions {
  std::vector<int> devices;  // role r (0 = source, 1..N = stages, N+1 = sink) runs on
                             // devices[r % size]; empty: BEEPLAN_WIRE_DEVICES or every GPU
  int queue_slots = 2;       // per-stage bounded queues (wire.hpp WireStageConfig)
  WireFault fault;
};

struct WireLocalPlacement {
  std::vector<int> role_devices;         // source, stages..., sink
  std::vector<std::uint64_t> hop_bytes;  // frame bytes moved per hop (header + payload)
  std::vector<int> hop_peer;             // 1 when the hop is a GPU -> other GPU copy
};

WireLocalResult run_wire_local(const WireLocalConfig& cfg, const WireLocalOptions& opt,
                               WireLocalPlacement* placement = nullptr);

}  // namespace beeplan::b200
