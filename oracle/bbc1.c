/* ORACLE / TEST INFRASTRUCTURE ONLY -- see oracle/bboracle.h.
 *
 * CPU restatement of the reference BBC1 codec and synthetic activations:
 *   byte_split / byte_merge          reference proj/src/codec.cpp:86-111
 *   entropy_bits_per_byte            reference proj/src/codec.cpp:113-125
 *   backend registry 0 identity / 1 deflate   codec.cpp:40-60,74-84
 *   serialize_container / parse_container     codec.cpp:127-161
 *   compress / decompress                     codec.cpp:163-192
 *   fp16_from_float, synth_gaussian_fp16      reference proj/src/synth.cpp:11-36,66-94
 * plus the frozen bf16 generator this build adds (same Box-Muller stream,
 * bf16 round-to-nearest-even), which the reference does not have.
 * Status codes: 0 OK, 1 OddLength, 2 LaneLengthMismatch, 3 BackendUnknown,
 * 4 CorruptContainer, 5 Error, 7 invalid argument (buffer too small).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "bboracle.h"

#define HDR 31

static void put_u64(uint8_t* p, uint64_t v) {
  for (int i = 0; i < 8; i++) p[i] = (uint8_t)(v >> (8 * i));
}
static uint64_t get_u64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; i++) v |= (uint64_t)p[i] << (8 * i);
  return v;
}

int orc_split(const uint8_t* in, size_t n, uint8_t* high, uint8_t* low) {
  if (n % 2) return 1;
  for (size_t k = 0; k < n / 2; k++) {
    low[k] = in[2 * k];
    high[k] = in[2 * k + 1];
  }
  return 0;
}

void orc_merge(const uint8_t* high, const uint8_t* low, size_t count, uint8_t* out) {
  for (size_t k = 0; k < count; k++) {
    out[2 * k] = low[k];
    out[2 * k + 1] = high[k];
  }
}

double orc_entropy(const uint8_t* in, size_t n) {
  if (n == 0) return 0.0;
  uint64_t counts[256] = {0};
  for (size_t i = 0; i < n; i++) counts[in[i]]++;
  double total = (double)n, e = 0.0;
  for (int b = 0; b < 256; b++) {
    if (!counts[b]) continue;
    double p = (double)counts[b] / total;
    e -= p * log2(p);
  }
  return e;
}

static size_t lane_bound(size_t n, int backend) { return backend == 0 ? n : orc_compress_bound(n); }

size_t orc_container_bound(size_t n, int backend, int split) {
  if (split) return HDR + 2 * lane_bound(n / 2, backend);
  return HDR + lane_bound(n, backend);
}

static int encode_lane(int backend, const uint8_t* in, size_t n, uint8_t* out, size_t cap,
                       size_t* len) {
  if (backend == 0) {
    if (cap < n) return 7;
    if (n) memcpy(out, in, n);
    *len = n;
    return 0;
  }
  return orc_zlib_compress(in, n, out, cap, len) ? 7 : 0;
}

int orc_compress(const uint8_t* in, size_t n, int backend, int split, uint8_t* out, size_t cap,
                 size_t* out_len) {
  if (backend != 0 && backend != 1) return 3; /* backend_by_id first (codec.cpp:164) */
  if (n % 2) return 1;
  if (cap < HDR) return 7;
  size_t count = n / 2, hl = 0, ll = 0;
  int rc;
  if (split) {
    uint8_t* lanes = (uint8_t*)malloc(n ? n : 1);
    orc_split(in, n, lanes, lanes + count);
    rc = encode_lane(backend, lanes, count, out + HDR, cap - HDR, &hl);
    if (!rc) rc = encode_lane(backend, lanes + count, count, out + HDR + hl, cap - HDR - hl, &ll);
    free(lanes);
  } else {
    rc = encode_lane(backend, in, n, out + HDR, cap - HDR, &hl);
  }
  if (rc) return rc;
  memcpy(out, "BBC1", 4);
  out[4] = 1;
  out[5] = (uint8_t)backend;
  out[6] = split ? 1 : 0;
  put_u64(out + 7, count);
  put_u64(out + 15, hl);
  put_u64(out + 23, ll);
  *out_len = HDR + hl + ll;
  return 0;
}

typedef struct {
  int backend, split;
  uint64_t count, hl, ll;
  const uint8_t *high, *low;
} parsed;

static int parse(const uint8_t* in, size_t n, parsed* c) {
  if (n < HDR) return 4;
  if (memcmp(in, "BBC1", 4) != 0) return 4;
  if (in[4] != 1) return 4;
  c->backend = in[5];
  c->split = in[6] & 1;
  c->count = get_u64(in + 7);
  c->hl = get_u64(in + 15);
  c->ll = get_u64(in + 23);
  uint64_t avail = n - HDR;
  if (c->hl > avail || c->ll > avail - c->hl || c->hl + c->ll != avail) return 4;
  c->high = in + HDR;
  c->low = in + HDR + c->hl;
  return 0;
}

/* backend.decode(blob, expected) preconditions (codec.cpp:27-31,45-47) */
static int lane_precheck(int backend, uint64_t blob, uint64_t expected) {
  if (backend == 0) return blob != expected ? 4 : 0;
  if (expected > blob * 1040 + 1024) return 4;
  return 0;
}

static int decode_lane(int backend, const uint8_t* blob, uint64_t bl, uint64_t expected,
                       uint8_t* out) {
  int rc = lane_precheck(backend, bl, expected);
  if (rc) return rc;
  if (backend == 0) {
    if (bl) memcpy(out, blob, bl);
    return 0;
  }
  size_t got = 0;
  if (orc_zlib_uncompress(blob, bl, out, expected, &got) != 0 || got != expected) return 4;
  return 0;
}

int orc_decompress(const uint8_t* in, size_t n, uint8_t* out, size_t cap, size_t* out_len) {
  parsed c;
  int rc = parse(in, n, &c);
  if (rc) return rc;
  if (c.backend != 0 && c.backend != 1) return 3;
  uint64_t count = c.count;
  if (c.split) {
    if ((rc = lane_precheck(c.backend, c.hl, count))) return rc;
    if (out == NULL || cap < 2 * count) {
      *out_len = 2 * count;
      return out == NULL ? 0 : 7;
    }
    uint8_t* lanes = (uint8_t*)malloc(count ? 2 * count : 1);
    rc = decode_lane(c.backend, c.high, c.hl, count, lanes);
    if (!rc) rc = decode_lane(c.backend, c.low, c.ll, count, lanes + count);
    if (!rc) orc_merge(lanes, lanes + count, count, out);
    free(lanes);
    if (rc) return rc;
    *out_len = 2 * count;
    return 0;
  }
  if (c.ll != 0) return 4;
  uint64_t expected = count * 2; /* size_t arithmetic, wraps like the reference */
  if ((rc = lane_precheck(c.backend, c.hl, expected))) return rc;
  if (out == NULL || cap < expected) {
    *out_len = expected;
    return out == NULL ? 0 : 7;
  }
  rc = decode_lane(c.backend, c.high, c.hl, expected, out);
  if (rc) return rc;
  *out_len = expected;
  return 0;
}

/* ------------------------------------------------------------------------- */
/* std::mt19937_64                                                            */
typedef struct {
  uint64_t mt[312];
  int i;
} mt64;

static void mt_seed(mt64* m, uint64_t seed) {
  m->mt[0] = seed;
  for (int i = 1; i < 312; i++)
    m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
  m->i = 312;
}

static uint64_t mt_next(mt64* m) {
  if (m->i >= 312) {
    for (int k = 0; k < 312; k++) {
      uint64_t y = (m->mt[k] & 0xFFFFFFFF80000000ULL) | (m->mt[(k + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = m->mt[(k + 156) % 312] ^ (y >> 1);
      if (y & 1) v ^= 0xB5026F5AA96619E9ULL;
      m->mt[k] = v;
    }
    m->i = 0;
  }
  uint64_t y = m->mt[m->i++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

uint16_t orc_fp16_from_float(float value) {
  uint32_t x;
  memcpy(&x, &value, 4);
  uint32_t sign = (x >> 16) & 0x8000u, exp_field = (x >> 23) & 0xFFu, mant = x & 0x7FFFFFu;
  if (exp_field == 0xFFu) return (uint16_t)(sign | 0x7C00u | (mant ? 0x200u : 0));
  int exp = (int)exp_field - 127 + 15;
  if (exp >= 0x1F) return (uint16_t)(sign | 0x7C00u);
  if (exp <= 0) {
    if (exp < -10) return (uint16_t)sign;
    mant |= 0x800000u;
    uint32_t shift = (uint32_t)(14 - exp);
    uint32_t half = mant >> shift, rem = mant & ((1u << shift) - 1u), halfway = 1u << (shift - 1u);
    if (rem > halfway || (rem == halfway && (half & 1u))) ++half;
    return (uint16_t)(sign | half);
  }
  uint32_t half = ((uint32_t)exp << 10) | (mant >> 13), rem = mant & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (half & 1u))) ++half;
  return (uint16_t)(sign | half);
}

uint16_t orc_bf16_from_float(float value) {
  uint32_t x;
  memcpy(&x, &value, 4);
  if ((x & 0x7F800000u) == 0x7F800000u && (x & 0x7FFFFFu)) return (uint16_t)((x >> 16) | 0x40u);
  x += 0x7FFFu + ((x >> 16) & 1u);
  return (uint16_t)(x >> 16);
}

static void synth(size_t elements, uint64_t seed, uint8_t* out, int bf16) {
  mt64 m;
  mt_seed(&m, seed);
  double spare = 0.0;
  int have_spare = 0;
  for (size_t i = 0; i < elements; i++) {
    double z;
    if (have_spare) {
      z = spare;
      have_spare = 0;
    } else {
      double u1 = ((double)(mt_next(&m) >> 11) + 1.0) / 9007199254740993.0;
      double u2 = ((double)(mt_next(&m) >> 11) + 1.0) / 9007199254740993.0;
      double r = sqrt(-2.0 * log(u1));
      double a = 2.0 * 3.141592653589793 * u2;
      z = r * cos(a);
      spare = r * sin(a);
      have_spare = 1;
    }
    uint16_t bits = bf16 ? orc_bf16_from_float((float)z) : orc_fp16_from_float((float)z);
    out[2 * i] = (uint8_t)(bits & 0xFF);
    out[2 * i + 1] = (uint8_t)(bits >> 8);
  }
}

void orc_synth_fp16(size_t elements, uint64_t seed, uint8_t* out) { synth(elements, seed, out, 0); }
void orc_synth_bf16(size_t elements, uint64_t seed, uint8_t* out) { synth(elements, seed, out, 1); }
