// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// C-ABI wrapper around the UNMODIFIED reference codec (compiled straight from
// /root/reference/proj/src/{codec,synth}.cpp by oracle/Makefile into
// oracle/_ref/libbeeplan_ref.so).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it.
//
// Wraps:
//   beeplan::compress + serialize_container   (reference codec.cpp:127-140,163-179)
//   beeplan::parse_container + decompress     (reference codec.cpp:142-161,181-192)
//   beeplan::synth_gaussian_fp16              (reference synth.cpp:66-94)
//   beeplan::entropy_bits_per_byte            (reference codec.cpp:113-125)
//   beeplan::pack / encode_packed / decode_packed / unpack (reference specdec.cpp:153-220)
// Status codes follow include/bbcodec.h (bb_status).
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>

#include "beeplan/codec.hpp"
#include "beeplan/errors.hpp"
#include "beeplan/specdec.hpp"
#include "beeplan/synth.hpp"

namespace {
thread_local std::string g_err;

int map_exception() {
  try {
    throw;
  } catch (const beeplan::OddLength& e) {
    g_err = e.what();
    return 1;
  } catch (const beeplan::LaneLengthMismatch& e) {
    g_err = e.what();
    return 2;
  } catch (const beeplan::BackendUnknown& e) {
    g_err = e.what();
    return 3;
  } catch (const beeplan::CorruptContainer& e) {
    g_err = e.what();
    return 4;
  } catch (const beeplan::CorruptOffsets& e) {
    g_err = e.what();
    return 8;
  } catch (const beeplan::DimMismatch& e) {
    g_err = e.what();
    return 9;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

unsigned char* dup_bytes(const beeplan::Bytes& b) {
  unsigned char* p = static_cast<unsigned char*>(std::malloc(b.size() ? b.size() : 1));
  if (!b.empty()) std::memcpy(p, b.data(), b.size());
  return p;
}
}  // namespace

extern "C" {

const char* bbref_last_error(void) { return g_err.c_str(); }

void bbref_free(void* p) { std::free(p); }

// Serialized BBC1 container of compress(stream, backend, split).
int bbref_compress(const unsigned char* in, size_t n, int backend, int split,
                   unsigned char** out, size_t* out_len) {
  try {
    beeplan::Bytes stream(in, in + n);
    beeplan::Bytes wire = beeplan::serialize_container(
        beeplan::compress(stream, static_cast<std::uint8_t>(backend), split != 0));
    *out = dup_bytes(wire);
    *out_len = wire.size();
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// decompress(parse_container(container)).
int bbref_decompress(const unsigned char* in, size_t n, unsigned char** out, size_t* out_len) {
  try {
    beeplan::Bytes wire(in, in + n);
    beeplan::Bytes stream = beeplan::decompress(beeplan::parse_container(wire));
    *out = dup_bytes(stream);
    *out_len = stream.size();
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Backend-level lane codec: backend_by_id(id).encode(lane).
int bbref_backend_encode(int backend, const unsigned char* in, size_t n, unsigned char** out,
                         size_t* out_len) {
  try {
    beeplan::Bytes lane(in, in + n);
    beeplan::Bytes blob = beeplan::backend_by_id(static_cast<std::uint8_t>(backend)).encode(lane);
    *out = dup_bytes(blob);
    *out_len = blob.size();
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int bbref_backend_decode(int backend, const unsigned char* in, size_t n, size_t expected,
                         unsigned char** out, size_t* out_len) {
  try {
    beeplan::Bytes blob(in, in + n);
    beeplan::Bytes lane =
        beeplan::backend_by_id(static_cast<std::uint8_t>(backend)).decode(blob, expected);
    *out = dup_bytes(lane);
    *out_len = lane.size();
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int bbref_synth_fp16(size_t elements, unsigned long long seed, unsigned char* out) {
  try {
    beeplan::Bytes s = beeplan::synth_gaussian_fp16(elements, seed);
    std::memcpy(out, s.data(), s.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}

double bbref_entropy(const unsigned char* in, size_t n) {
  beeplan::Bytes b(in, in + n);
  return beeplan::entropy_bits_per_byte(b);
}

// encode_packed(pack(per_request)): request r holds req_counts[r] vectors, vector v has
// row_dims[v] floats; the vectors are concatenated in `flat`.
int bbref_pack_encode(const float* flat, const size_t* row_dims, const unsigned* req_counts,
                      unsigned n_requests, unsigned char** out, size_t* out_len) {
  try {
    std::vector<beeplan::HiddenStates> per_request(n_requests);
    size_t v = 0, f = 0;
    for (unsigned r = 0; r < n_requests; ++r)
      for (unsigned k = 0; k < req_counts[r]; ++k, ++v) {
        per_request[r].emplace_back(flat + f, flat + f + row_dims[v]);
        f += row_dims[v];
      }
    beeplan::Bytes wire = beeplan::encode_packed(beeplan::pack(per_request));
    *out = dup_bytes(wire);
    *out_len = wire.size();
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// encode_packed(decode_packed(data, hidden_dim)): status parity + round trip.
int bbref_decode_packed(const unsigned char* in, size_t n, size_t hidden_dim, unsigned char** out,
                        size_t* out_len) {
  try {
    beeplan::Bytes data(in, in + n);
    beeplan::Bytes wire = beeplan::encode_packed(beeplan::decode_packed(data, hidden_dim));
    *out = dup_bytes(wire);
    *out_len = wire.size();
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// unpack(PackedBatch{hidden_dim, payload, offsets}) validity (CorruptOffsets).
int bbref_unpack_check(const unsigned* offsets, size_t n_offsets, size_t hidden_dim, size_t payload_floats) {
  try {
    beeplan::PackedBatch b;
    b.hidden_dim = hidden_dim;
    b.offsets.assign(offsets, offsets + n_offsets);
    b.payload.assign(payload_floats, 0.0f);
    (void)beeplan::unpack(b);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

}  // extern "C"
