// SPDX-License-Identifier: Apache-2.0
// Drop-in synthetic-activation generator (reference proj/include/beeplan/synth.hpp),
// plus the frozen bf16 variant this build adds for LLaMA-2 bf16 configs.
#pragma once

#include <cstdint>

#include "beeplan/codec.hpp"

namespace beeplan {

std::uint16_t fp16_from_float(float value);  // round to nearest even
float float_from_fp16(std::uint16_t bits);
std::uint16_t bf16_from_float(float value);  // round to nearest even

// Standard-normal activations as little-endian 16-bit words (Box-Muller over
// std::mt19937_64, identical bytes on every platform).
Bytes synth_gaussian_fp16(std::size_t elements, std::uint64_t seed);
Bytes synth_gaussian_bf16(std::size_t elements, std::uint64_t seed);

}  // namespace beeplan
