// Parallel inflate of whole zlib streams (the fast path of the deflate backend's
// decode; the exact sequential decoder in bb_inflate.cu is the fallback that
// defines uncompress() error parity -- any stream this path cannot fully
// validate is re-decoded there).
//
// A 30+ MiB lane holds thousands of deflate blocks whose boundaries are only
// known after Huffman-decoding their predecessors.  Instead of walking them in
// order, every place a block could start is found and decoded at once:
//
//   P1 k_candidates4  every bit offset is tested for a dynamic-block header
//                     (BTYPE=10, HLIT<=29, HDIST<=29 bit-sliced over 32 offsets,
//                     then a complete code-length code), survivors verified
//                     exactly by k_verify_dynamic; every byte offset for a stored
//                     block (LEN == ~NLEN); bitmaps, so ranks give ordered node ids
//   P2 k_decode_nodes stored / static candidates: one thread each;
//      k_dyn_scan     dynamic candidates: one warp each, the block's bits cut into
//                     32 chunks decoded at once (Huffman self-synchronisation,
//                     Jacobi fix-up), recording end bit, output bytes, matches
//   P3 k_link         each node's successor = the candidate that starts exactly
//                     where it ends (or END / BREAK / BAD)
//   P4 binary lifting the true block chain is the path from the zlib header;
//                     jump tables give the i-th block of the chain in O(log)
//   P5 k_dyn_emit     second decode of the chain's dynamic blocks at their final
//                     output offsets: literals written, matches recorded as
//                     (dst,dist,len); k_copy_stored copies stored blocks; a BREAK
//                     (static block) is finished by one thread (k_tail)
//   P6 LZ77 resolution: pointer jumping in shared memory over 32 KiB windows
//                     (k_resolve_local) or 2-window thread-block clusters
//                     (k_resolve_cluster, distributed shared memory); bytes whose
//                     copy chain leaves the window chase a read-only source map
//                     to a resolved byte (k_resolve_chase)
//   P7 Adler-32 check, size check
#include <cooperative_groups.h>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <mutex>

#include <cstring>
#include <vector>

#include "bb_common.cuh"
#include "bb_kernels.h"

namespace bb {
namespace par {

constexpr uint32_t SENT_END = 0xFFFFFFF0u, SENT_BREAK = 0xFFFFFFF1u, SENT_BAD = 0xFFFFFFF2u;
#ifndef ND_THREADS_OVR
#define ND_THREADS_OVR 128
#endif
constexpr int ND_THREADS = ND_THREADS_OVR;
constexpr uint32_t SUB = 32768;  // resolution window
constexpr uint32_t MOD = 65521;

__constant__ uint16_t p_lbase[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                     31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t p_lext[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t p_dbase[30] = {1,    2,    3,    4,    5,    7,    9,    13,    17,    25,
                                     33,   49,   65,   97,   129,  193,  257,  385,   513,   769,
                                     1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ uint8_t p_dext[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
__constant__ uint8_t p_order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

struct PJob {
  const uint8_t* src;
  uint64_t n;
  uint8_t* dst;
  uint64_t expected;
  uint64_t dbm;     // dynamic-candidate bitmap: first u32 word (1 bit per stream bit)
  uint64_t sbm;     // stored-candidate bitmap: first u32 word (1 bit per stream byte)
  uint32_t node0;   // virtual start node; then ndyn dynamic nodes, then 2*nsto stored nodes
  uint32_t ndyn, nsto;
  uint64_t mbase;   // match list base
  uint64_t mcap;
  uint32_t sub0, nsub;  // resolution windows
  uint32_t dyn_base;    // first slot of this job's dynamic nodes in the per-dynamic-node arrays
  uint64_t xbase;       // first entry of this job's per-output-byte source map
};

struct Node {
  uint64_t end_bit;
  uint64_t out_len;
  uint32_t nmatch;
  uint32_t flags;  // bit0 ok, bit1 final, bit2 stored
  uint64_t start;  // dynamic: header bit; stored: data byte offset (LEN field)
};

struct Chain {
  uint32_t len;       // blocks on the chain (excluding the virtual start)
  uint32_t terminal;  // SENT_END / SENT_BREAK / SENT_BAD
  uint32_t last;      // last node (the virtual start if len == 0)
  uint32_t pad;
};

struct Match {
  uint32_t dst;
  uint16_t dist;
  uint16_t len;
};

// job owning flat index x, given prefix[0..nj] (prefix[0] = 0) of per-job counts
__device__ __forceinline__ int find_job(const uint64_t* __restrict__ prefix, int nj, uint64_t x) {
  int lo = 0, hi = nj - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// ---- bit access -------------------------------------------------------------
__device__ __forceinline__ uint64_t load_le64_slow(const uint8_t* p, uint64_t n, uint64_t byte) {
  uint64_t v = 0;
  for (int i = 0; i < 8; i++)
    if (byte + i < n) v |= (uint64_t)__ldg(p + byte + i) << (8 * i);
  return v;
}

// 64 bits starting at bit `b` (zero beyond the end): two aligned 64-bit loads
__device__ __forceinline__ uint64_t peek64(const uint8_t* p, uint64_t n, uint64_t b) {
  const uint64_t byte = b >> 3;
  if (byte + 16 <= n) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p + byte);
    const uint64_t* w = reinterpret_cast<const uint64_t*>(a & ~uintptr_t(7));
    const uint32_t sh = (uint32_t)(((a & 7) << 3) + (b & 7));  // 0..63
    const uint64_t lo = __ldg(w), hi = __ldg(w + 1);
    return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
  }
  const uint32_t sh = (uint32_t)(b & 7);
  const uint64_t lo = load_le64_slow(p, n, byte);
  if (!sh) return lo;
  const uint64_t hi = byte + 8 < n ? __ldg(p + byte + 8) : 0;
  return (lo >> sh) | (hi << (64 - sh));
}

struct BitReader {
  const uint8_t* p;
  uint64_t n;
  uint64_t pos;  // next bit to consume (absolute)
  uint64_t hold;
  uint32_t bits;
  __device__ __forceinline__ void init(const uint8_t* p_, uint64_t n_, uint64_t bit) {
    p = p_;
    n = n_;
    pos = bit;
    hold = peek64(p, n, pos);
    bits = 64;
  }
  __device__ __forceinline__ void refill() {
    if (bits < 32) {
      hold = peek64(p, n, pos);
      bits = 64;
    }
  }
  __device__ __forceinline__ uint32_t peek(uint32_t k) const { return (uint32_t)(hold & ((1ull << k) - 1)); }
  __device__ __forceinline__ void drop(uint32_t k) {
    hold >>= k;
    bits -= k;
    pos += k;
  }
  __device__ __forceinline__ uint32_t take(uint32_t k) {
    refill();
    uint32_t v = peek(k);
    drop(k);
    return v;
  }
  __device__ __forceinline__ bool past_end() const { return pos > 8 * n; }
};

// ---- canonical decoding tables (limit compare; left-justified 15-bit codes) ----
template <int CAP>
struct HTabT {
  uint16_t lim[16];     // lim[l] for l = 1..15 (lim[0] unused), 15-bit left-justified
  int16_t base[16];     // sym index = base[l] + (w >> (15 - l))
  uint16_t sym[CAP];
  int max;
};
typedef HTabT<288> HLit;
typedef HTabT<32> HDist;

// inftrees.c rules: over-subscribed -> error; incomplete -> error unless
// (type != CODES and max length == 1).  type: 0 CODES, 1 LENS, 2 DISTS
template <int CAP, bool ROLLED, class Lens>
__device__ int htab_build_fn(HTabT<CAP>* t, Lens lens, int n, int type) {
  uint16_t count[16];
  for (int i = 0; i < 16; i++) count[i] = 0;
  if constexpr (ROLLED) {
#pragma unroll 1
    for (int s = 0; s < n; s++) count[lens(s)]++;
  } else {
    for (int s = 0; s < n; s++) count[lens(s)]++;
  }
  int max = 15;
  while (max >= 1 && count[max] == 0) max--;
  t->max = max;
  if (max == 0) {
    for (int l = 1; l < 16; l++) t->lim[l] = 0;
    t->lim[0] = 0;
    return 0;
  }
  int left = 1;
  for (int len = 1; len <= 15; len++) {
    left <<= 1;
    left -= count[len];
    if (left < 0) return -1;
  }
  if (left > 0 && (type == 0 || max != 1)) return -1;
  uint16_t offs[16];
  offs[1] = 0;
  for (int l = 1; l < 15; l++) offs[l + 1] = offs[l] + count[l];
  uint32_t code = 0;
  count[0] = 0;
  for (int l = 1; l <= 15; l++) {
    code = (code + count[l - 1]) << 1;
    t->lim[l] = (uint16_t)min((code + count[l]) << (15 - l), 32768u);
    t->base[l] = (int16_t)((int)offs[l] - (int)code);
  }
  if constexpr (ROLLED) {
#pragma unroll 1
    for (int s = 0; s < n; s++)
      if (lens(s)) t->sym[offs[lens(s)]++] = (uint16_t)s;
  } else {
    for (int s = 0; s < n; s++)
      if (lens(s)) t->sym[offs[lens(s)]++] = (uint16_t)s;
  }
  return 0;
}

template <int CAP>
__device__ int htab_build(HTabT<CAP>* t, const uint8_t* lens, int n, int type) {
  return htab_build_fn<CAP, false>(t, [lens](int s) { return (uint32_t)lens[s]; }, n, type);
}

// limits held in registers while a block is decoded
struct Lims {
  uint32_t v[16];
  template <int CAP>
  __device__ __forceinline__ void load(const HTabT<CAP>* t) {
#pragma unroll
    for (int k = 1; k < 16; k++) v[k] = t->lim[k];
  }
};

// -1 invalid code, -2 past end
template <int CAP>
__device__ __forceinline__ int hdecode(BitReader& r, const HTabT<CAP>* t, const Lims& L) {
  r.refill();
  uint32_t w = __brev((uint32_t)r.hold) >> 17;
  int l = 1;
#pragma unroll
  for (int k = 1; k < 16; k++) l += (w >= L.v[k]);
  if (l > 15) return -1;
  int s = t->sym[t->base[l] + (int)(w >> (15 - l))];
  r.drop((uint32_t)l);
  if (r.past_end()) return -2;
  return s;
}

template <int CAP>
__device__ __forceinline__ int hdecode(BitReader& r, const HTabT<CAP>* t) {
  Lims L;
  L.load(t);
  return hdecode(r, t, L);
}

struct Tables {
  HLit lit;
  HDist dist;
};

__device__ void static_tables(Tables* T) {
  // lengths computed, not stored (no 288-byte array on the stack); loops kept rolled
  htab_build_fn<288, true>(&T->lit, [](int i) { return i < 144 ? 8u : i < 256 ? 9u : i < 280 ? 7u : 8u; }, 288, 1);
  htab_build_fn<32, true>(&T->dist, [](int) { return 5u; }, 32, 2);
}

// The code-length code (19 symbols, lengths <= 7) held in registers: limit compares for the
// length, packed per-length bases and a packed sorted-symbol list for the symbol -- no tables in
// local memory (htab_build's arrays went to the stack of every kernel that parsed a header).
struct ClCode {
  uint32_t lim[6];  // left-justified 7-bit limits of lengths 1..6 (a complete code's lim[7] is 128)
  uint64_t base;    // 8-bit field l: offs[l] - code[l] + 128
  uint64_t lo, hi;  // symbols in canonical order, 5 bits each: entries 0..11 in lo, 12..18 in hi
};

// y: the ncode 3-bit lengths in stream order.  inflate_table's CODES rules: over-subscribed or
// incomplete codes are errors; an empty code (zlib decodes every length as 0, so the block
// fails on its missing end-of-block code) is rejected here directly.
__device__ __forceinline__ bool cl_build(ClCode& c, uint64_t y, uint32_t ncode) {
  constexpr uint8_t slot[19] = {3, 17, 15, 13, 11, 9, 7, 5, 4, 6, 8, 10, 12, 14, 16, 18, 0, 1, 2};
  uint32_t L[19];
  uint64_t cnt = 0;  // 8-bit count per length (field l; field 0 collects the unused symbols)
#pragma unroll
  for (int s = 0; s < 19; s++) {
    L[s] = (uint32_t)slot[s] < ncode ? (uint32_t)(y >> (3 * slot[s])) & 7u : 0u;
    cnt += 1ull << (8 * L[s]);
  }
  uint32_t code = 0, offs = 0;
  int left = 1;
  uint64_t offp = 0;
  c.base = 0;
#pragma unroll
  for (int l = 1; l <= 7; l++) {
    const uint32_t k = (uint32_t)(cnt >> (8 * l)) & 0xffu;
    left = (left << 1) - (int)k;
    if (left < 0) return false;
    offp |= (uint64_t)offs << (8 * l);
    c.base |= (uint64_t)(offs - code + 128u) << (8 * l);
    if (l <= 6) c.lim[l - 1] = (code + k) << (7 - l);
    code = (code + k) << 1;
    offs += k;
  }
  if (left != 0) return false;
  uint64_t run = 0;
  c.lo = c.hi = 0;
#pragma unroll
  for (int s = 0; s < 19; s++) {
    const uint32_t l = L[s];
    const uint32_t pos = (uint32_t)((offp + run) >> (8 * l)) & 0xffu;  // fields <= 38: no carries
    run += 1ull << (8 * l);
    if (l) {
      if (pos < 12) c.lo |= (uint64_t)s << (5 * pos);
      else c.hi |= (uint64_t)s << (5 * (pos - 12));
    }
  }
  return true;
}

// one code-length symbol from the next stream bits (hold: bit 0 = next bit); len = its length
__device__ __forceinline__ uint32_t cl_decode(const ClCode& c, uint64_t hold, uint32_t& len) {
  const uint32_t w = __brev((uint32_t)hold) >> 25;  // next 7 bits, first stream bit most significant
  uint32_t l = 1;
#pragma unroll
  for (int k = 0; k < 6; k++) l += (w >= c.lim[k]);
  const uint32_t idx = (uint32_t)((c.base >> (8 * l)) & 0xffu) - 128u + (w >> (7 - l));
  len = l;
  return idx < 12 ? (uint32_t)(c.lo >> (5 * idx)) & 31u : (uint32_t)(c.hi >> (5 * (idx - 12))) & 31u;
}

// Dynamic block header at r (after the 3 header bits) up to the code lengths: lens[0, nlen + ndist)
// receives the literal/length then distance code lengths.  0 ok, -1 invalid (inflate.c TABLE /
// LENLENS / CODELENS rules, incl. the end-of-block code).
__device__ int read_code_lengths(BitReader& r, uint8_t* lens, uint32_t& nlen, uint32_t& ndist) {
  nlen = r.take(5) + 257, ndist = r.take(5) + 1;
  const uint32_t ncode = r.take(4) + 4;
  if (nlen > 286 || ndist > 30) return -1;
  ClCode ch;
  const uint64_t y = peek64(r.p, r.n, r.pos) & ((1ull << (3 * ncode)) - 1);
  r.init(r.p, r.n, r.pos + 3 * ncode);
  if (r.past_end() || !cl_build(ch, y, ncode)) return -1;
  uint32_t have = 0;
  while (have < nlen + ndist) {
    r.refill();
    uint32_t l;
    const uint32_t sym = cl_decode(ch, r.hold, l);
    r.drop(l);
    if (sym < 16) {
      lens[have++] = (uint8_t)sym;
    } else {
      uint32_t len = 0, copy;
      if (sym == 16) {
        if (have == 0) return -1;
        len = lens[have - 1];
        copy = 3 + r.take(2);
      } else if (sym == 17) {
        copy = 3 + r.take(3);
      } else {
        copy = 11 + r.take(7);
      }
      if (have + copy > nlen + ndist) return -1;
      while (copy--) lens[have++] = (uint8_t)len;
    }
    if (r.past_end()) return -1;
  }
  if (lens[256] == 0) return -1;
  return 0;
}

// Reads a dynamic block header at r (positioned after the 3 header bits); one thread.
__device__ int read_dynamic(BitReader& r, Tables* T) {
  uint8_t lens[320];
  uint32_t nlen, ndist;
  if (read_code_lengths(r, lens, nlen, ndist)) return -1;
  if (htab_build(&T->lit, lens, nlen, 1)) return -1;
  if (htab_build(&T->dist, lens + nlen, ndist, 2)) return -1;
  return 0;
}

// htab_build by a whole warp: lens[0, n) in shared memory, cnt = 16 words of shared scratch.
// Counts and in-length ranks by __match_any_sync per 32 symbols, the limits / bases as a lane scan
// over the lengths, the sorted symbols placed in parallel.  Same tables and return value as
// htab_build (inftrees.c rules).
template <int CAP>
__device__ int warp_htab_build(HTabT<CAP>* t, const uint8_t* lens, int n, int type, int lane, uint32_t* cnt) {
  constexpr int NC = (CAP + 31) / 32;
  if (lane < 16) cnt[lane] = 0;
  __syncwarp();
  const unsigned lt = (1u << lane) - 1;
  uint32_t rank[NC];
#pragma unroll
  for (int c = 0; c < NC; c++) {
    const int sidx = 32 * c + lane;
    const uint32_t l = sidx < n ? lens[sidx] : 0u;
    const unsigned m = __match_any_sync(0xffffffffu, l);
    const uint32_t before = cnt[l];
    rank[c] = before + __popc(m & lt);
    __syncwarp();
    if ((m & lt) == 0) cnt[l] = before + __popc(m);
    __syncwarp();
  }
  const uint32_t k = (lane >= 1 && lane <= 15) ? cnt[lane] : 0u;
  const unsigned nz = __ballot_sync(0xffffffffu, k != 0);
  const int max = nz ? 31 - __clz(nz) : 0;
  // inclusive scans over lengths: left-justified limits (sum of count[j] << (15 - j)) and offsets
  uint32_t lim = (lane >= 1 && lane <= 15) ? k << (15 - lane) : 0u, offs = k;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const uint32_t a = __shfl_up_sync(0xffffffffu, lim, o), b = __shfl_up_sync(0xffffffffu, offs, o);
    if (lane >= o) lim += a, offs += b;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, lim, 15);
  if (max == 0) {
    if (lane < 16) t->lim[lane] = 0;
    if (lane == 0) t->max = 0;
    __syncwarp();
    return 0;
  }
  if (total > 32768u) return -1;                              // over-subscribed
  if (total < 32768u && (type == 0 || max != 1)) return -1;  // incomplete
  const uint32_t excl_lim = lim - ((lane >= 1 && lane <= 15) ? k << (15 - lane) : 0u);
  const uint32_t excl_off = offs - k;
  __syncwarp();
  if (lane >= 1 && lane <= 15) {
    const uint32_t code = excl_lim >> (15 - lane);
    t->lim[lane] = (uint16_t)min(lim, 32768u);
    t->base[lane] = (int16_t)((int)excl_off - (int)code);
    cnt[lane] = excl_off;
  }
  if (lane == 0) t->max = max;
  __syncwarp();
#pragma unroll
  for (int c = 0; c < NC; c++) {
    const int sidx = 32 * c + lane;
    const uint32_t l = sidx < n ? lens[sidx] : 0u;
    if (l) t->sym[cnt[l] + rank[c]] = (uint16_t)sidx;
  }
  __syncwarp();
  return 0;
}

// Decodes symbols until END_BLOCK.  EMIT: writes literals to out[] and match
// records; otherwise only counts.  Returns 0 ok, -1 error.
template <bool EMIT>
__device__ int decode_codes(BitReader& r, const Tables* T, uint64_t& out_len, uint32_t& nmatch, uint64_t limit,
                            uint8_t* out, uint64_t out_off, Match* matches, uint64_t mcap) {
  Lims LL, DL;
  LL.load(&T->lit);
  DL.load(&T->dist);
  uint64_t guard = 0;
  for (;;) {
    if (++guard > (1ull << 26)) return -1;
    int sym = hdecode(r, &T->lit, LL);
    if (sym < 0) return -1;
    if (sym < 256) {
      if (out_len >= limit) return -1;
      if (EMIT) out[out_off + out_len] = (uint8_t)sym;
      out_len++;
    } else if (sym == 256) {
      return 0;
    } else {
      sym -= 257;
      if (sym >= 29) return -1;
      uint32_t len = p_lbase[sym] + r.take(p_lext[sym]);
      int ds = hdecode(r, &T->dist, DL);
      if (ds < 0 || ds >= 30) return -1;
      uint32_t dist = p_dbase[ds] + r.take(p_dext[ds]);
      if (r.past_end()) return -1;
      if (out_len + len > limit) return -1;
      if (EMIT) {
        if (dist > out_off + out_len) return -1;  // invalid distance too far back
        if (nmatch >= mcap) return -1;
        matches[nmatch] = Match{(uint32_t)(out_off + out_len), (uint16_t)dist, (uint16_t)len};
      }
      nmatch++;
      out_len += len;
    }
  }
}


// Exact zlib acceptance of a dynamic block header at bit b (inflate.c TABLE /
// LENLENS / CODELENS + inftrees.c rules), with early rejection as soon as a
// partial Kraft sum is over-subscribed.  Never rejects a header zlib accepts.
__device__ bool verify_dynamic(const uint8_t* p, uint64_t n, uint64_t b) {
  BitReader r;
  r.init(p, n, b + 3);
  uint32_t nlen = r.take(5) + 257, ndist = r.take(5) + 1, ncode = r.take(4) + 4;
  if (nlen > 286 || ndist > 30) return false;
  ClCode ch;
  const uint64_t y = peek64(p, n, r.pos) & ((1ull << (3 * ncode)) - 1);
  r.init(p, n, r.pos + 3 * ncode);
  if (!cl_build(ch, y, ncode)) return false;
  uint32_t have = 0, prev = 0, kl = 0, kd = 0;
  uint16_t cnt1l = 0, cnt1d = 0, maxl = 0, maxd = 0;
  bool eob = false;
  while (have < nlen + ndist) {
    r.refill();
    uint32_t cl;
    const uint32_t sym = cl_decode(ch, r.hold, cl);
    r.drop(cl);
    if (r.past_end()) return false;
    uint32_t len, copy;
    if (sym < 16) {
      len = (uint32_t)sym;
      copy = 1;
    } else if (sym == 16) {
      if (have == 0) return false;
      len = prev;
      copy = 3 + r.take(2);
    } else if (sym == 17) {
      len = 0;
      copy = 3 + r.take(3);
    } else {
      len = 0;
      copy = 11 + r.take(7);
    }
    if (have + copy > nlen + ndist) return false;
    if (!len) {  // zero lengths only advance the count (runs of up to 138: one step, not a loop)
      have += copy;
      prev = len;
      if (r.past_end()) return false;
      continue;
    }
    for (uint32_t k = 0; k < copy; k++, have++) {
      if (have < nlen) {
        kl += 32768u >> len;
        if (kl > 32768u) return false;
        if (have == 256) eob = true;
        maxl = max(maxl, (uint16_t)len);
        cnt1l += len == 1;
      } else {
        kd += 32768u >> len;
        if (kd > 32768u) return false;
        maxd = max(maxd, (uint16_t)len);
        cnt1d += len == 1;
      }
    }
    prev = len;
    if (r.past_end()) return false;
  }
  if (!eob) return false;
  // incomplete sets are allowed only when the longest code has length 1
  if (kl != 32768u && maxl != 1) return false;
  if (kd != 32768u && maxd > 1) return false;
  return true;
}

// ---- P1 --------------------------------------------------------------------

// Survivors of the quick test are appended to a list (warp-aggregated) and
// verified exactly by k_verify_dynamic with one thread each, so the rare long
// verifications do not serialise whole warps.
// P1 (current): four stream bytes / 32 bit offsets per thread.  The cheap
// header conditions (BTYPE = 10, HLIT <= 29, HDIST <= 29) are evaluated for all
// 32 offsets at once on a 64-bit window (bit-sliced), and only the ~20 % that
// survive run the code-length-code Kraft sum, which stops as soon as it is
// over-subscribed.
__global__ void k_candidates4(const PJob* __restrict__ jobs, const uint64_t* __restrict__ blk_prefix, int njobs,
                              uint32_t* __restrict__ sbm, int find_dynamic, uint64_t* __restrict__ surv,
                              unsigned long long* __restrict__ surv_cnt, uint64_t surv_cap) {
  const uint32_t j = (uint32_t)find_job(blk_prefix, njobs, blockIdx.x);
  const PJob J = jobs[j];
  const uint64_t T = (blockIdx.x - blk_prefix[j]) * 256ull + threadIdx.x;  // bytes [4T, 4T + 4)
  const uint64_t B0 = 4 * T;
  const int lane = threadIdx.x & 31;
  uint32_t sbits = 0;
  uint64_t x0_keep = 0;
  if (find_dynamic) {
    uint32_t cm = 0;
    uint64_t x0 = 0, x1 = 0;
    if (B0 < J.n) {
      const uint64_t nbits = 8 * J.n;
      x0 = peek64(J.src, J.n, 8 * B0), x1 = peek64(J.src, J.n, 8 * B0 + 64);
      x0_keep = x0;
      uint64_t m = ~(x0 >> 1) & (x0 >> 2);
      m &= ~((x0 >> 4) & (x0 >> 5) & (x0 >> 6) & (x0 >> 7));
      m &= ~((x0 >> 9) & (x0 >> 10) & (x0 >> 11) & (x0 >> 12));
      cm = (uint32_t)m;
      // stream limits: b >= 16 and b + 17 <= 8 n
      const uint64_t b0 = 8 * B0;
      if (b0 < 16) cm &= 0xffffffffu << (uint32_t)(16 - b0);
      if (b0 + 31 + 17 > nbits) {
        const int64_t keep = (int64_t)nbits - 17 - (int64_t)b0 + 1;  // offsets i < keep are allowed
        cm &= keep <= 0 ? 0u : (keep >= 32 ? 0xffffffffu : ((1u << keep) - 1));
      }
    }
    // the warp's survivors are dealt out one per lane (the Kraft check of the
    // code-length code runs with every lane busy instead of per-lane loops)
    const uint32_t cnt = __popc(cm);
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t x0lo = (uint32_t)x0, x0hi = (uint32_t)(x0 >> 32), x1lo = (uint32_t)x1, x1hi = (uint32_t)(x1 >> 32);
    for (uint32_t base = 0; base < tot; base += 32) {
      const uint32_t k = base + lane;
      // owner: the first lane whose inclusive count exceeds k (binary search over lanes)
      int owner = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, incl, owner + step - 1);
        if (v <= k) owner += step;
      }
      const uint32_t oinc = __shfl_sync(0xffffffffu, incl, owner);
      const uint32_t ocnt = __shfl_sync(0xffffffffu, cnt, owner);
      const uint32_t ocm = __shfl_sync(0xffffffffu, cm, owner);
      const uint64_t wx0 = (uint64_t)__shfl_sync(0xffffffffu, x0lo, owner) |
                           ((uint64_t)__shfl_sync(0xffffffffu, x0hi, owner) << 32);
      const uint64_t wx1 = (uint64_t)__shfl_sync(0xffffffffu, x1lo, owner) |
                           ((uint64_t)__shfl_sync(0xffffffffu, x1hi, owner) << 32);
      bool pass = false;
      uint32_t i = 0;
      if (k < tot) {
        const uint32_t slot = k - (oinc - ocnt);
        i = __fns(ocm, 0, (int)slot + 1);
        // HCLEN and the 19 code-length-code lengths: 61 bits from offset i + 13 (<= 44)
        const uint32_t sh = i + 13;
        const uint64_t y = (wx0 >> sh) | (wx1 << (64 - sh));
        const uint32_t ncode = (uint32_t)(y & 15) + 4;
        // Kraft sum of the first ncode 3-bit lengths, 128 >> l from a byte table
        // (0, 64, 32, 16, 8, 4, 2, 1); complete iff the sum is exactly 128
        uint32_t kraft = 0;
#pragma unroll
        for (uint32_t kk = 0; kk < 19; kk++) {
          const uint32_t l = (uint32_t)(y >> (4 + 3 * kk)) & 7;
          const uint32_t v = __byte_perm(0x10204000u, 0x01020408u, l);
          kraft += kk < ncode ? v : 0u;
        }
        pass = kraft == 128;
      }
      // warp-aggregated append of the round's survivors
      const unsigned bal = __ballot_sync(0xffffffffu, pass);
      if (bal) {
        unsigned long long sbase = 0;
        if (lane == 0) sbase = atomicAdd(surv_cnt, (unsigned long long)__popc(bal));
        sbase = __shfl_sync(0xffffffffu, sbase, 0);
        if (pass) {
          const uint64_t slot = sbase + __popc(bal & ((1u << lane) - 1));
          const uint64_t ob0 = B0 - 4ull * (uint64_t)(lane - owner);  // owner's first byte
          if (slot < surv_cap) surv[slot] = ((uint64_t)j << 48) | (8 * ob0 + i);
        }
      }
    }
  }
  if (B0 + 16 <= J.n) {
    // bytes B0 .. B0 + 7 in one aligned pair of loads: LEN / NLEN at each of the 4 offsets
    const uint64_t x = find_dynamic ? x0_keep : peek64(J.src, J.n, 8 * B0);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const uint64_t B = B0 + k;
      const uint32_t w = (uint32_t)(x >> (8 * k));
      const uint32_t len = w & 0xffff, nlen = w >> 16;
      if (B >= 2 && len == (~nlen & 0xffff) && B + 4 + len <= J.n) sbits |= 1u << k;
    }
  } else if (B0 < J.n) {
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const uint64_t B = B0 + k;
      if (B >= 2 && B + 4 <= J.n) {
        const uint32_t len = __ldg(J.src + B) | ((uint32_t)__ldg(J.src + B + 1) << 8);
        const uint32_t nlen = __ldg(J.src + B + 2) | ((uint32_t)__ldg(J.src + B + 3) << 8);
        if (len == (~nlen & 0xffff) && B + 4 + len <= J.n) sbits |= 1u << k;
      }
    }
  }
  // stored bitmap: 8 lanes (32 bytes) per word
  uint32_t wv = sbits << (4 * (lane & 7));
  wv |= __shfl_xor_sync(0xffffffffu, wv, 1);
  wv |= __shfl_xor_sync(0xffffffffu, wv, 2);
  wv |= __shfl_xor_sync(0xffffffffu, wv, 4);
  if ((lane & 7) == 0 && B0 < J.n + 32) sbm[J.sbm + (B0 >> 5)] = wv;
}

#ifndef VD_THREADS
#define VD_THREADS 256
#endif
#ifndef VD_MINB
#define VD_MINB 4  // 64 registers (small spills): occupancy over the survivors' divergent walks
#endif
__global__ void __launch_bounds__(VD_THREADS, VD_MINB) k_verify_dynamic(const PJob* __restrict__ jobs, const uint64_t* __restrict__ surv,
                                 const unsigned long long* __restrict__ surv_cnt, uint64_t surv_cap,
                                 uint32_t* __restrict__ dbm, uint32_t* __restrict__ fail, int njobs) {
  const uint64_t cnt = *surv_cnt;
  if (cnt > surv_cap) {  // list overflow: let the exact sequential decoder take every job
    if (blockIdx.x == 0)
      for (int i = threadIdx.x; i < njobs; i += blockDim.x) fail[i] = 1;
    return;
  }
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = surv[i];
    const uint32_t j = (uint32_t)(v >> 48);
    const uint64_t b = v & ((1ull << 48) - 1);
    const PJob J = jobs[j];
    if (verify_dynamic(J.src, J.n, b)) atomicOr(&dbm[J.dbm + (b >> 5)], 1u << (b & 31));
  }
}

// Stored-only pass (the incompressible lanes): 16 byte offsets per thread from
// six aligned word loads, realigned once with funnel shifts; same blocks (1 KiB
// of stream each) and the same stored bitmap as k_candidates4.
__global__ void __launch_bounds__(64) k_stored_cand(const PJob* __restrict__ jobs,
                                                   const uint64_t* __restrict__ blk_prefix, int njobs,
                                                   uint32_t* __restrict__ sbm) {
  const uint32_t j = (uint32_t)find_job(blk_prefix, njobs, blockIdx.x);
  const PJob J = jobs[j];
  const uint64_t T = (blockIdx.x - blk_prefix[j]) * 64ull + threadIdx.x;
  const uint64_t B0 = 16 * T;  // bytes [B0, B0 + 16)
  uint32_t bits = 0;
  if (B0 + 24 <= J.n) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(J.src + B0);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
    const uint32_t sh = 8 * (uint32_t)(a & 3);
    uint32_t x[6], y[5];
#pragma unroll
    for (int i = 0; i < 6; i++) x[i] = __ldg(w + i);
#pragma unroll
    for (int i = 0; i < 5; i++) y[i] = __funnelshift_r(x[i], x[i + 1], sh);  // bytes B0 + 4i ..
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const uint32_t v = __funnelshift_r(y[k >> 2], y[(k >> 2) + 1], 8 * (k & 3));
      const uint64_t B = B0 + k;
      const uint32_t len = v & 0xffff, nlen = v >> 16;
      if (B >= 2 && len == (~nlen & 0xffff) && B + 4 + len <= J.n) bits |= 1u << k;
    }
  } else if (B0 < J.n) {
    for (int k = 0; k < 16; k++) {
      const uint64_t B = B0 + k;
      if (B >= 2 && B + 4 <= J.n) {
        const uint32_t len = __ldg(J.src + B) | ((uint32_t)__ldg(J.src + B + 1) << 8);
        const uint32_t nlen = __ldg(J.src + B + 2) | ((uint32_t)__ldg(J.src + B + 3) << 8);
        if (len == (~nlen & 0xffff) && B + 4 + len <= J.n) bits |= 1u << k;
      }
    }
  }
  uint32_t wv = bits << (16 * (threadIdx.x & 1));
  wv |= __shfl_xor_sync(0xffffffffu, wv, 1);
  if ((threadIdx.x & 1) == 0 && B0 < J.n + 32) sbm[J.sbm + (B0 >> 5)] = wv;
}

// node-count prefix values for the host: entries 4i, 4i + 1 index the dynamic
// prefix array, 4i + 2, 4i + 3 the stored one
__global__ void k_gather_prefix(const uint64_t* __restrict__ idx, int n, const uint32_t* __restrict__ dpre,
                                const uint32_t* __restrict__ spre, uint32_t* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = ((k & 3) < 2 ? dpre : spre)[idx[k]];
}

__global__ void k_popc(const uint32_t* __restrict__ words, uint64_t count, uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = __popc(words[i]);
}

// ---- P2 --------------------------------------------------------------------
// rank of the set bit `bit` within job-local bitmap words [w0, ...) via per-word prefix counts
__device__ __forceinline__ uint32_t bm_rank(const uint32_t* words, const uint32_t* prefix, uint64_t w0, uint64_t bit) {
  uint64_t w = w0 + (bit >> 5);
  return prefix[w] - prefix[w0] + __popc(words[w] & ((1u << (bit & 31)) - 1));
}
__device__ __forceinline__ bool bm_test(const uint32_t* words, uint64_t w0, uint64_t bit) {
  return (words[w0 + (bit >> 5)] >> (bit & 31)) & 1;
}

// fill node positions: thread per bitmap word
__global__ void k_node_positions(const PJob* __restrict__ jobs, int njobs, const uint32_t* __restrict__ dbm,
                                 const uint32_t* __restrict__ dpre, const uint32_t* __restrict__ sbm,
                                 const uint32_t* __restrict__ spre, Node* __restrict__ nodes) {
  const int j = blockIdx.y;
  const PJob J = jobs[j];
  const uint64_t dwords = (J.n + 3) / 4, swords = (J.n + 31) / 32 + 1;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < dwords + swords;
       w += (uint64_t)gridDim.x * blockDim.x) {
    if (w < dwords) {
      uint32_t v = dbm[J.dbm + w];
      uint32_t r = dpre[J.dbm + w] - dpre[J.dbm];
      while (v) {
        int k = __ffs(v) - 1;
        v &= v - 1;
        Node nd{};
        nd.start = 32 * w + k;
        nodes[J.node0 + 1 + r++] = nd;
      }
    } else {
      uint64_t ws = w - dwords;
      uint32_t v = sbm[J.sbm + ws];
      uint32_t r = spre[J.sbm + ws] - spre[J.sbm];
      while (v) {
        int k = __ffs(v) - 1;
        v &= v - 1;
        uint64_t B = 32 * ws + k;
        for (int f = 0; f < 2; f++) {
          Node nd{};
          nd.start = B;
          nd.flags = 4 | (f ? 2 : 0);
          nodes[J.node0 + 1 + J.ndyn + 2 * r + f] = nd;
        }
        r++;
      }
    }
  }
}

__device__ int decode_static_run(BitReader& r, Tables* T, uint64_t& out_len, uint32_t& nmatch, uint64_t limit,
                                 bool& final_seen) {
  // continue through static blocks that directly follow (counting only)
  for (;;) {
    r.refill();
    uint32_t hdr = r.peek(3);
    if (((hdr >> 1) & 3) != 1) return 0;  // not static: node ends here
    r.drop(3);
    static_tables(T);
    if (decode_codes<false>(r, T, out_len, nmatch, limit, nullptr, 0, nullptr, 0)) return -1;
    if (hdr & 1) {
      final_seen = true;
      return 0;
    }
  }
}

__global__ void __launch_bounds__(ND_THREADS) k_decode_nodes(const PJob* __restrict__ jobs,
                                                             const uint32_t* __restrict__ node_job,
                                                             uint32_t nnodes, Node* __restrict__ nodes) {
  extern __shared__ __align__(16) uint8_t sm[];
  Tables* T = reinterpret_cast<Tables*>(sm) + threadIdx.x;
  uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nnodes) return;
  const PJob J = jobs[node_job[g]];
  Node nd = nodes[g];
  if (g == J.node0) {  // virtual start: "a block ended at bit 16"
    nd.end_bit = 16;
    nd.out_len = 0;
    nd.nmatch = 0;
    nd.flags = 1;
    nodes[g] = nd;
    return;
  }
  if (nd.flags & 4) {  // stored
    uint64_t B = nd.start;
    uint32_t len = J.src[B] | ((uint32_t)J.src[B + 1] << 8);
    nd.end_bit = 8 * (B + 4 + len);
    nd.out_len = len;
    nd.nmatch = 0;
    nd.flags |= (len <= J.expected) ? 1 : 0;
    nodes[g] = nd;
    return;
  }
  (void)T;  // dynamic nodes: k_dyn_scan (one warp per block)
}


// ---- warp-cooperative dynamic blocks -----------------------------------------
// One warp per dynamic block.  Lane 0 parses the header; the block's bit range
// (header end .. the next candidate, an estimate of the block end) is cut into
// 32 chunks that the lanes decode at once from arbitrary bit offsets.  Huffman
// decoding resynchronises quickly: each lane records its first REC symbol
// starts, and the true decode entering a chunk (the previous lane's exit) is
// advanced only until it lands on one of them.  Pass 2 (k_dyn_emit) then
// decodes every lane's exact sub-range again, writing its output.
#ifndef WD_WARPS_OVR
#define WD_WARPS_OVR 2
#endif
constexpr int WD_WARPS = WD_WARPS_OVR;
__device__ unsigned long long g_wd[8];  // loop-guard trips per site (corrupt-stream safety limits)
#define PROG(d, lane, ph, x) \
  do {                       \
  } while (0)
#define WD_GUARD(site, it, limit, action)        \
  if (++(it) > (limit)) {                        \
    atomicAdd(&g_wd[site], 1ull);                \
    action;                                      \
  }
constexpr int REC = 16;
constexpr uint64_t NONE64 = ~0ull;

struct LanePlan {
  uint64_t begin, end;  // absolute bit positions of the lane's symbols [begin, end)
  uint64_t out_off;     // output bytes before this lane (node-relative)
  uint32_t m_off;       // matches before this lane (node-relative)
  uint32_t m_cnt;       // matches of this lane
  uint64_t out_cnt;     // output bytes of this lane
};

struct DynExtra {
  uint64_t static_begin;  // != NONE64: static blocks follow the dynamic one (lane 0 decodes them)
  uint64_t dyn_out, dyn_nm;
};

// Direct lookup of the next FAST_BITS (literal/length) or FAST_DBITS (distance)
// stream bits, built per block by the warp from the canonical tables.  Entry:
// bits 0-3 code length (0: longer code -> the limit-compare decode), bits 4-5
// kind (0 literal, 1 length, 2 end of block, 3 invalid symbol), bits 6-9 extra
// bits, bits 16-31 literal byte or length / distance base -- so a symbol costs
// one shared load, with no divergent __constant__ lookups.
constexpr int FAST_BITS = 9, FAST_DBITS = 8;
struct FastT {
  uint32_t lit[1 << FAST_BITS];
  uint32_t dist[1 << FAST_DBITS];
};

template <int CAP, int NB>
__device__ __forceinline__ void fast_fill(const HTabT<CAP>* t, uint32_t* f, int lane, bool is_dist) {
  const uint32_t limn = t->lim[NB];
  for (uint32_t idx = lane; idx < (1u << NB); idx += 32) {
    const uint32_t w = (__brev(idx) >> (32 - NB)) << (15 - NB);
    uint32_t e = 0;
    if ((w | ((1u << (15 - NB)) - 1)) < limn) {
      int l = 1;
      for (int k = 1; k < NB; k++) l += (w >= t->lim[k]);
      const uint32_t sym = t->sym[t->base[l] + (int)(w >> (15 - l))];
      uint32_t kind, extra = 0, val = 0;
      if (is_dist) {
        if (sym < 30) kind = 0, extra = p_dext[sym], val = p_dbase[sym];
        else kind = 3;
      } else if (sym < 256) {
        kind = 0, val = sym;
      } else if (sym == 256) {
        kind = 2;
      } else if (sym < 286) {
        kind = 1, extra = p_lext[sym - 257], val = p_lbase[sym - 257];
      } else {
        kind = 3;
      }
      e = (uint32_t)l | (kind << 4) | (extra << 6) | (val << 16);
    }
    f[idx] = e;
  }
}

__device__ __forceinline__ void fast_build(const Tables* T, FastT* F, int lane) {
  fast_fill<288, FAST_BITS>(&T->lit, F->lit, lane, false);
  fast_fill<32, FAST_DBITS>(&T->dist, F->dist, lane, true);
  __syncwarp();
}

// Word-refill bit reader for the hot decode loops: a 64-bit window refilled
// 32 bits at a time from aligned words (one 32-bit load per refill instead of
// peek64's unaligned pair), positions counted as 32-bit offsets from the range
// start.  Words past the stream end read as zero (the callers' range and count
// checks reject any decode that ran into them).
struct WordReader {
  const uint32_t* w;  // aligned words covering the stream
  uint32_t wi, wend;  // next word to load, words available
  uint64_t hold;
  int bits;
  uint32_t used;  // bits consumed since init
  uint32_t nxt;   // word wi, loaded one refill ahead (its latency hides behind ~32 bits of decode)
  __device__ __forceinline__ uint32_t word(uint32_t k) const { return k < wend ? __ldg(w + k) : 0u; }
  __device__ __forceinline__ void init(const uint8_t* p, uint64_t n, uint64_t bitpos) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
    const uint64_t abit = bitpos + 8 * (a & 3);  // bit position in the aligned frame
    wend = (uint32_t)((n + (a & 3) + 3) / 4);
    const uint32_t k = (uint32_t)(abit >> 5), sh = (uint32_t)(abit & 31);
    hold = ((uint64_t)word(k) | ((uint64_t)word(k + 1) << 32)) >> sh;
    bits = 64 - (int)sh;
    wi = k + 2;
    nxt = word(wi);
    used = 0;
  }
  __device__ __forceinline__ void refill() {
    if (bits <= 32) {
      hold |= (uint64_t)nxt << bits;
      bits += 32;
      nxt = word(++wi);
    }
  }
  __device__ __forceinline__ void drop(uint32_t k) {
    hold >>= k;
    bits -= (int)k;
    used += k;
  }
  __device__ __forceinline__ uint32_t take(uint32_t k) {  // k <= 13, bits >= 13 guaranteed by refill
    const uint32_t v = (uint32_t)hold & ((1u << k) - 1);
    drop(k);
    return v;
  }
};

// limit-compare decode of a code longer than the direct table (limits from shared memory)
template <int CAP>
__device__ __forceinline__ int wdecode_slow(WordReader& r, const HTabT<CAP>* t) {
  const uint32_t x = __brev((uint32_t)r.hold) >> 17;
  int l = 1;
#pragma unroll
  for (int k = 1; k < 16; k++) l += (x >= t->lim[k]);
  if (l > 15) return -1;
  const int s = t->sym[t->base[l] + (int)(x >> (15 - l))];
  r.drop((uint32_t)l);
  return s;
}

// one literal/length (+ distance) symbol: 0 literal, 1 match, 2 end of block, -1 invalid
__device__ __forceinline__ int wsym(WordReader& r, const Tables* T, const FastT* F, uint32_t& len, uint32_t& dist,
                                    uint32_t& lit) {
  r.refill();
  const uint32_t e = F->lit[(uint32_t)r.hold & ((1u << FAST_BITS) - 1)];
  uint32_t kind, base, extra;
  if (e & 15) {
    r.drop(e & 15);
    kind = (e >> 4) & 3, base = e >> 16, extra = (e >> 6) & 15;
  } else {
    const int sym = wdecode_slow(r, &T->lit);
    if (sym < 0) return -1;
    if (sym < 256) kind = 0, base = (uint32_t)sym, extra = 0;
    else if (sym == 256) kind = 2, base = 0, extra = 0;
    else if (sym < 286) kind = 1, base = p_lbase[sym - 257], extra = p_lext[sym - 257];
    else return -1;
  }
  if (kind == 0) {
    lit = base;
    len = 1;
    return 0;
  }
  if (kind != 1) return kind == 2 ? 2 : -1;
  len = base + r.take(extra);  // <= 15 + 5 bits used since the refill: >= 13 left
  r.refill();
  const uint32_t ed = F->dist[(uint32_t)r.hold & ((1u << FAST_DBITS) - 1)];
  if (ed & 15) {
    r.drop(ed & 15);
    if (((ed >> 4) & 3) == 3) return -1;
    r.refill();
    dist = (ed >> 16) + r.take((ed >> 6) & 15);
  } else {
    const int ds = wdecode_slow(r, &T->dist);
    if (ds < 0 || ds >= 30) return -1;
    r.refill();
    dist = p_dbase[ds] + r.take(p_dext[ds]);
  }
  return 1;
}

struct EmitSm {
  FastT F;
  Tables T;
};

struct WarpSm {
  FastT F;
  Tables T;
  uint32_t rpos[32][REC];
  uint16_t rout[32][REC];  // output bytes before record j of the lane (<= REC * 258)
  uint16_t rnm[32][REC];   // matches before record j
};

// Two register budgets: MINB 5 (127 registers, no spills) has the shortest latency per block
// (config1's few blocks: 0.39 vs 0.48 ms with the other); MINB 12 (85 registers) has 2.4x the
// resident warps and the best throughput over many blocks (config2: 3.46 ms; MINB 16 3.51,
// MINB 10 3.70, MINB 5 3.82).
#ifndef DS_MINB
#define DS_MINB 5
#endif
#ifndef DS_MINB_WIDE
#define DS_MINB_WIDE 12
#endif
template <int MINB>
__global__ void __launch_bounds__(32 * WD_WARPS, MINB) k_dyn_scan(const PJob* __restrict__ jobs,
                                                           const uint32_t* __restrict__ node_job,
                                                           const uint32_t* __restrict__ dyn_nodes, uint32_t ndyn_total,
                                                           Node* __restrict__ nodes, Tables* __restrict__ tabs,
                                                           LanePlan* __restrict__ plans, DynExtra* __restrict__ extra) {
  extern __shared__ __align__(16) uint8_t smraw[];
  WarpSm& W = reinterpret_cast<WarpSm*>(smraw)[threadIdx.x >> 5];
  const uint32_t d = blockIdx.x * WD_WARPS + (threadIdx.x >> 5);
  if (d >= ndyn_total) return;
  const int lane = threadIdx.x & 31;
  const uint32_t g = dyn_nodes[d];
  const uint32_t jid = node_job[g];
  const PJob J = jobs[jid];
  Node nd = nodes[g];
  PROG(d, lane, 1, 0);
  // header (lane 0)
  uint64_t d0 = 0;
  int rc = 0;
  bool final_blk = false;
  // code lengths (lane 0, register-resident code-length code) into shared scratch -- the record
  // arrays, written only from round 1 on -- then both tables built by the whole warp
  uint8_t* lens = reinterpret_cast<uint8_t*>(&W.rpos[0][0]);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(lens + 320);
  uint32_t nlen = 0, ndist = 0;
  if (lane == 0) {
    BitReader r;
    r.init(J.src, J.n, nd.start);
    uint32_t hdr = r.take(3);
    final_blk = hdr & 1;
    rc = read_code_lengths(r, lens, nlen, ndist);
    d0 = r.pos;
  }
  rc = __shfl_sync(0xffffffffu, rc, 0);
  d0 = __shfl_sync(0xffffffffu, d0, 0);
  final_blk = __shfl_sync(0xffffffffu, (int)final_blk, 0);
  nlen = __shfl_sync(0xffffffffu, nlen, 0);
  ndist = __shfl_sync(0xffffffffu, ndist, 0);
  __syncwarp();
  if (!rc) rc = warp_htab_build(&W.T.lit, lens, (int)nlen, 1, lane, cnt);
  if (!rc) rc = warp_htab_build(&W.T.dist, lens + nlen, (int)ndist, 2, lane, cnt);
  if (rc) {
    if (lane == 0) {
      nd.flags = 8;  // dynamic, not ok
      nodes[g] = nd;
    }
    return;
  }
  __syncwarp();
  fast_build(&W.T, &W.F, lane);
  Lims LL, DL;
  LL.load(&W.T.lit);
  DL.load(&W.T.dist);
  // estimated end: the next dynamic candidate of the same job
  uint64_t E = 8 * J.n;
  if (g + 1 < J.node0 + 1 + J.ndyn) E = min(E, nodes[g + 1].start);
  if (E < d0 + 32 * 64) E = d0 + 32 * 64;
  const uint64_t span = E - d0;
  const uint64_t s_k = d0 + span * lane / 32, s_n = d0 + span * (lane + 1) / 32;
  // round 1
  WordReader r;
  r.init(J.src, J.n, s_k);
  uint64_t out = 0, nm = 0;
  int nrec = 0;
  bool stuck = false;
  // first two end-of-block symbols seen (a garbage one may precede the real one)
  uint64_t eob_at = NONE64, eob_end = 0, eob_out = 0, eob_nm = 0, err_at = NONE64;
  uint64_t eob2_at = NONE64, eob2_end = 0, eob2_out = 0, eob2_nm = 0;
  uint64_t it0 = 0;
  while (s_k + r.used < s_n) {
    WD_GUARD(0, it0, (1ull << 16), { stuck = true; err_at = s_k + r.used; break; })
    PROG(d, lane, 2, it0);
    const uint64_t p = s_k + r.used;
    if (nrec < REC) {
      W.rpos[lane][nrec] = (uint32_t)(p - d0);
      W.rout[lane][nrec] = (uint16_t)out;
      W.rnm[lane][nrec] = (uint16_t)nm;
      nrec++;
    }
    uint32_t len = 0, dist = 0, lit = 0;
    int t = wsym(r, &W.T, &W.F, len, dist, lit);
    if (t < 0) {
      stuck = true;
      err_at = p;
      break;
    }
    if (t == 2) {
      const uint64_t pe = s_k + r.used;
      if (eob_at == NONE64) eob_at = p, eob_end = pe, eob_out = out, eob_nm = nm;
      else if (eob2_at == NONE64) eob2_at = p, eob2_end = pe, eob2_out = out, eob2_nm = nm;
      continue;
    }
    out += len;
    nm += (t == 1);
  }
  const uint64_t f = stuck ? NONE64 : s_k + r.used;
  __syncwarp();
  // fix-up rounds: the true decode enters lane k's chunk at F_{k-1}
  uint64_t F = f, cnt_out = out, cnt_nm = nm;       // corrected results (lane 0 is exact)
  // lane 0 decodes from the true block start: its events are real; others wait for the fix-up
  uint64_t real_eob = lane == 0 ? eob_at : NONE64, real_eob_end = eob_end;
  uint64_t real_err = lane == 0 ? err_at : NONE64;
  uint64_t ev_out = eob_out, ev_nm = eob_nm;
  uint64_t used = lane == 0 ? d0 : NONE64 - 1;
  for (int iter = 0; iter < 33; iter++) {
    PROG(d, lane, 4, iter);
    uint64_t entry = __shfl_up_sync(0xffffffffu, F, 1);
    bool blocked = __shfl_up_sync(0xffffffffu, (int)(real_eob != NONE64 || real_err != NONE64), 1);
    if (lane == 0) entry = d0, blocked = false;
    const bool redo = lane > 0 && entry != used && entry != NONE64 && !blocked;
    if (!__any_sync(0xffffffffu, redo)) break;
    if (redo) {
      used = entry;
      uint64_t t = entry, o = 0, m = 0;
      int j = 0;
      bool done = false;
      real_eob = NONE64;
      real_err = NONE64;
      WordReader q;
      q.init(J.src, J.n, t);
      const uint64_t q0 = t;
      uint64_t it1 = 0;
      while (t < s_n) {
        WD_GUARD(1, it1, (1ull << 16), { real_err = t; done = true; break; })
        PROG(d, lane, 5, it1);
        while (j < nrec && (uint64_t)W.rpos[lane][j] + d0 < t) j++;
        if (j < nrec && (uint64_t)W.rpos[lane][j] + d0 == t) {
          // synchronised with round 1 from record j on
          const uint64_t base_o = W.rout[lane][j], base_m = W.rnm[lane][j];
          // the first end-of-block at or after the synchronisation point is real
          uint64_t ea = eob_at, ee = eob_end, eo = eob_out, en = eob_nm;
          if (ea != NONE64 && ea < t) ea = eob2_at, ee = eob2_end, eo = eob2_out, en = eob2_nm;
          if (ea != NONE64 && ea < t) ea = NONE64;  // more than two: resolved by pass 2's checks
          if (ea != NONE64 && (err_at == NONE64 || ea < err_at)) {
            real_eob = ea;
            real_eob_end = ee;
            ev_out = o + eo - base_o;
            ev_nm = m + en - base_m;
          } else if (err_at != NONE64 && err_at >= t) {
            real_err = err_at;
          }
          cnt_out = o + out - base_o;
          cnt_nm = m + nm - base_m;
          F = f;
          done = true;
          break;
        }
        uint32_t len = 0, dist = 0, lit = 0;
        const uint64_t p = t;
        int ty = wsym(q, &W.T, &W.F, len, dist, lit);
        if (ty < 0) {
          real_err = p;
          done = true;
          break;
        }
        if (ty == 2) {
          real_eob = p;
          real_eob_end = q0 + q.used;
          ev_out = o;
          ev_nm = m;
          cnt_out = o;
          cnt_nm = m;
          F = q0 + q.used;
          done = true;
          break;
        }
        o += len;
        m += (ty == 1);
        t = q0 + q.used;
      }
      if (!done) {
        F = t;
        cnt_out = o;
        cnt_nm = m;
      }
    }
  }
  // the first lane whose true range holds an end-of-block (or an error) ends the block
  const bool ev = real_eob != NONE64 || real_err != NONE64;
  const unsigned evm = __ballot_sync(0xffffffffu, ev);
  int kstar = evm ? __ffs(evm) - 1 : 31;
  uint64_t lane_out = lane < kstar ? cnt_out : (lane == kstar && ev ? ev_out : (lane == kstar ? cnt_out : 0));
  uint64_t lane_nm = lane < kstar ? cnt_nm : (lane == kstar && ev ? ev_nm : (lane == kstar ? cnt_nm : 0));
  bool bad = lane == kstar && real_err != NONE64 && (real_eob == NONE64 || real_err < real_eob);
  // no end-of-block inside the estimate: the last lane keeps decoding
  uint64_t tail_end = 0;
  if (!evm && lane == 31) {
    WordReader q;
    q.init(J.src, J.n, F);
    uint64_t it2 = 0;
    for (;;) {
      WD_GUARD(2, it2, (1ull << 20), { bad = true; break; })
      PROG(d, lane, 6, it2);
      uint32_t len = 0, dist = 0, lit = 0;
      const uint64_t p = F + q.used;
      if (p > 8 * J.n) {  // ran off the stream
        bad = true;
        break;
      }
      int ty = wsym(q, &W.T, &W.F, len, dist, lit);
      if (ty < 0) {
        bad = true;
        break;
      }
      if (ty == 2) {
        real_eob = p;
        real_eob_end = F + q.used;
        break;
      }
      lane_out += len;
      lane_nm += (ty == 1);
      if (lane_out > J.expected) {
        bad = true;
        break;
      }
    }
    tail_end = real_eob;
  }
  PROG(d, lane, 7, 0);
  // prefix sums over lanes
  uint64_t xo = lane_out, xm = lane_nm;
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t a = __shfl_up_sync(0xffffffffu, xo, o), b = __shfl_up_sync(0xffffffffu, xm, o);
    if (lane >= o) xo += a, xm += b;
  }
  const uint64_t tot_o = __shfl_sync(0xffffffffu, xo, 31), tot_m = __shfl_sync(0xffffffffu, xm, 31);
  const bool anybad = __any_sync(0xffffffffu, bad);
  PROG(d, lane, 8, ((unsigned)ev << 23) | ((unsigned)stuck << 22) | ((unsigned)(real_eob_end != 0) << 21) |
                        (unsigned)(F == NONE64 || F - d0 > 0x1fffffull ? 0x1fffffull : F - d0));
  // lane ranges for pass 2
  const uint64_t F_prev = __shfl_up_sync(0xffffffffu, F, 1);  // every lane must take part
  const uint64_t begin = lane == 0 ? d0 : F_prev;
  uint64_t end = lane < kstar ? F : (lane == kstar ? (evm ? real_eob : tail_end) : begin);
  if (lane > kstar) end = begin;
  LanePlan lp;
  lp.begin = lane <= kstar ? begin : 0;
  lp.end = lane <= kstar ? end : 0;
  lp.out_off = xo - lane_out;
  lp.m_off = (uint32_t)(xm - lane_nm);
  lp.m_cnt = lane <= kstar ? (uint32_t)lane_nm : 0;
  lp.out_cnt = lane <= kstar ? lane_out : 0;
  plans[(uint64_t)d * 32 + lane] = lp;
  const uint64_t blk_end = __shfl_sync(0xffffffffu, real_eob_end, kstar);
  // copy the tables for pass 2
  {
    const uint32_t* srcw = reinterpret_cast<const uint32_t*>(&W.T);
    uint32_t* dstw = reinterpret_cast<uint32_t*>(tabs + d);
    for (uint32_t i = lane; i < sizeof(Tables) / 4; i += 32) dstw[i] = srcw[i];
  }
  __syncwarp();
  if (lane == 0) {
    uint64_t out_len = tot_o, nmatch = tot_m;
    bool ok = !anybad && out_len <= J.expected;
    bool fin = final_blk;
    uint64_t e_bit = blk_end;
    DynExtra ex{NONE64, tot_o, tot_m};
    if (ok && !fin) {
      BitReader q;
      q.init(J.src, J.n, blk_end);
      q.refill();
      PROG(d, 0, 10, (unsigned)(blk_end - nd.start));
      if (((q.peek(3) >> 1) & 3) == 1) {
        PROG(d, 0, 11, 0);
        ex.static_begin = blk_end;
        uint32_t nm32 = 0;
        bool fs = false;
        if (decode_static_run(q, &W.T, out_len, nm32, J.expected, fs)) ok = false;
        nmatch += nm32;
        fin = fs;
        e_bit = q.pos;
      }
    }
    extra[d] = ex;
    PROG(d, 0, 9, 0);
    nd.end_bit = e_bit;
    nd.out_len = out_len;
    nd.nmatch = (uint32_t)nmatch;
    nd.flags = 8 | (ok ? 1 : 0) | (fin ? 2 : 0);
    nodes[g] = nd;
  }
}

#ifndef DE_MINB
#define DE_MINB 1
#endif
__global__ void __launch_bounds__(32 * WD_WARPS, DE_MINB) k_dyn_emit(const PJob* __restrict__ jobs, const Chain* __restrict__ chains,
                                                           const uint32_t* __restrict__ chain_nodes,
                                                           const uint32_t* __restrict__ job_of_chain_block,
                                                           const uint32_t* __restrict__ chain_block_base,
                                                           const Node* __restrict__ nodes,
                                                           const uint64_t* __restrict__ out_off,
                                                           const uint64_t* __restrict__ m_off,
                                                           const Tables* __restrict__ tabs,
                                                           const LanePlan* __restrict__ plans,
                                                           const DynExtra* __restrict__ extra,
                                                           Match* __restrict__ matches, uint32_t* __restrict__ fail) {
  extern __shared__ __align__(16) uint8_t smraw[];
  EmitSm& ES = reinterpret_cast<EmitSm*>(smraw)[threadIdx.x >> 5];
  Tables& T = ES.T;
  const int lane = threadIdx.x & 31;
  const uint32_t j = job_of_chain_block[blockIdx.x];
  const PJob J = jobs[j];
  const uint32_t i = (blockIdx.x - chain_block_base[j]) * WD_WARPS + (threadIdx.x >> 5);
  if (i >= chains[j].len) return;
  const uint32_t g = chain_nodes[J.node0 + i];
  const Node nd = nodes[g];
  if (!(nd.flags & 8)) return;
  const uint32_t d = J.dyn_base + (g - J.node0 - 1);
  {
    const uint32_t* srcw = reinterpret_cast<const uint32_t*>(tabs + d);
    uint32_t* dstw = reinterpret_cast<uint32_t*>(&T);
    for (uint32_t k = lane; k < sizeof(Tables) / 4; k += 32) dstw[k] = srcw[k];
  }
  __syncwarp();
  fast_build(&T, &ES.F, lane);
  const LanePlan lp = plans[(uint64_t)d * 32 + lane];
  const uint64_t base = out_off[J.node0 + i];
  Match* mm = matches + J.mbase + m_off[J.node0 + i];
  Lims LL, DL;
  LL.load(&T.lit);
  DL.load(&T.dist);
  bool bad = false;
  if (lp.end > lp.begin && lp.end - lp.begin < (1ull << 31)) {
    WordReader r;
    r.init(J.src, J.n, lp.begin);
    const uint32_t span = (uint32_t)(lp.end - lp.begin);
    uint8_t* dst = J.dst;
    uint64_t o = base + lp.out_off;
    uint32_t m = lp.m_off;
    // every symbol consumes >= 1 bit, so the loop ends within span iterations
    while (r.used < span) {
      uint32_t len = 0, dist = 0, lit = 0;
      const int ty = wsym(r, &T, &ES.F, len, dist, lit);
      if (ty == 0) {
        dst[o++] = (uint8_t)lit;
      } else if (ty == 1) {
        if (dist > o) {
          bad = true;
          break;
        }
        mm[m++] = Match{(uint32_t)o, (uint16_t)dist, (uint16_t)len};
        o += len;
      } else {
        bad = true;  // an end-of-block or invalid code inside the lane's range
        break;
      }
    }
    if (r.used != span || o - (base + lp.out_off) != lp.out_cnt || m - lp.m_off != lp.m_cnt) bad = true;
  } else if (lp.end > lp.begin || lp.out_cnt || lp.m_cnt) {
    bad = true;
  }
  const DynExtra ex = extra[d];
  __syncwarp();
  if (lane == 0 && ex.static_begin != NONE64 && !bad) {
    BitReader r;
    r.init(J.src, J.n, ex.static_begin);
    uint64_t got = 0;
    uint32_t nmatch = 0;
    bool final_seen = false;
    while (!final_seen) {
      r.refill();
      uint32_t h = r.peek(3);
      if (((h >> 1) & 3) != 1) break;
      r.drop(3);
      static_tables(&T);
      if (decode_codes<true>(r, &T, got, nmatch, nd.out_len - ex.dyn_out, J.dst, base + ex.dyn_out,
                             mm + ex.dyn_nm, nd.nmatch - ex.dyn_nm)) {
        bad = true;
        break;
      }
      final_seen = h & 1;
    }
    if (ex.dyn_out + got != nd.out_len) bad = true;
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(&fail[j], 1u);
}

// ---- P3 --------------------------------------------------------------------
__global__ void k_link(const PJob* __restrict__ jobs, const uint32_t* __restrict__ node_job, uint32_t nnodes,
                       const Node* __restrict__ nodes, const uint32_t* __restrict__ dbm,
                       const uint32_t* __restrict__ dpre, const uint32_t* __restrict__ sbm,
                       const uint32_t* __restrict__ spre, uint32_t* __restrict__ next) {
  uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nnodes) return;
  const PJob J = jobs[node_job[g]];
  const Node nd = nodes[g];
  uint32_t nx;
  if (!(nd.flags & 1)) {
    nx = SENT_BAD;
  } else if (nd.flags & 2) {
    nx = SENT_END;
  } else {
    uint64_t e = nd.end_bit;
    if (e + 3 > 8 * J.n) {
      nx = SENT_BAD;
    } else {
      uint32_t h = (uint32_t)(peek64(J.src, J.n, e) & 7);
      uint32_t type = (h >> 1) & 3;
      if (type == 2) {
        nx = bm_test(dbm, J.dbm, e) ? J.node0 + 1 + bm_rank(dbm, dpre, J.dbm, e) : SENT_BAD;
      } else if (type == 0) {
        uint64_t B = (e + 3 + 7) >> 3;
        nx = (B < J.n && bm_test(sbm, J.sbm, B)) ? J.node0 + 1 + J.ndyn + 2 * bm_rank(sbm, spre, J.sbm, B) + (h & 1)
                                                 : SENT_BAD;
      } else if (type == 1) {
        nx = SENT_BREAK;
      } else {
        nx = SENT_BAD;
      }
    }
  }
  next[g] = nx;
}

// ---- P4 --------------------------------------------------------------------
__global__ void k_lift(const uint32_t* __restrict__ prev, uint32_t* __restrict__ cur, uint32_t nnodes) {
  uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nnodes) return;
  uint32_t a = prev[g];
  cur[g] = a >= SENT_END ? a : prev[a];
}

// every lifting level in one CTA when the nodes fit in it (small streams: one launch instead of one
// per level -- config1 has ~11 levels of a few hundred nodes)
constexpr uint32_t LIFT1_MAX = 1024;
__global__ void __launch_bounds__(LIFT1_MAX) k_lift_all(uint32_t* __restrict__ jump, uint32_t nnodes, int levels) {
  const uint32_t g = threadIdx.x;
  for (int k = 1; k < levels; k++) {
    const uint32_t* prev = jump + (size_t)(k - 1) * nnodes;
    if (g < nnodes) {
      const uint32_t a = prev[g];
      jump[(size_t)k * nnodes + g] = a >= SENT_END ? a : prev[a];
    }
    __syncthreads();  // level k is complete (and visible to the block) before level k + 1 reads it
  }
}


__global__ void k_chain_len(const PJob* __restrict__ jobs, int njobs, const uint32_t* __restrict__ jump,
                            uint32_t nnodes, int levels, Chain* __restrict__ chains) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= njobs) return;
  uint32_t v = jobs[j].node0, len = 0;
  for (int k = levels - 1; k >= 0; k--) {
    uint32_t u = jump[(uint64_t)k * nnodes + v];
    if (u < SENT_END) {
      v = u;
      len += 1u << k;
    }
  }
  chains[j] = Chain{len, jump[v], v, 0};
}

// chain[j][i] = node at step i+1 from the start
__global__ void k_chain_nodes(const PJob* __restrict__ jobs, const Chain* __restrict__ chains,
                              const uint32_t* __restrict__ jump, uint32_t nnodes, int levels,
                              uint32_t* __restrict__ chain_nodes) {
  const int j = blockIdx.y;
  const PJob J = jobs[j];
  const uint32_t len = chains[j].len;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
    uint32_t v = J.node0, steps = i + 1;
    for (int k = 0; k < levels; k++)
      if (steps >> k & 1) v = jump[(uint64_t)k * nnodes + v];
    chain_nodes[J.node0 + i] = v;  // node0-based slots: chain length <= node count
  }
}

// exclusive scans of out_len / nmatch along each chain (one CTA per job)
__global__ void __launch_bounds__(256) k_chain_scan(const PJob* __restrict__ jobs, const Chain* __restrict__ chains,
                                                   const uint32_t* __restrict__ chain_nodes,
                                                   const Node* __restrict__ nodes, uint64_t* __restrict__ out_off,
                                                   uint64_t* __restrict__ m_off, uint64_t* __restrict__ totals) {
  typedef cub::BlockScan<uint64_t, 256> Scan;
  __shared__ typename Scan::TempStorage t1, t2;
  __shared__ uint64_t c_out, c_m;
  const int j = blockIdx.x;
  const PJob J = jobs[j];
  const uint32_t len = chains[j].len;
  if (threadIdx.x == 0) c_out = c_m = 0;
  __syncthreads();
  for (uint32_t base = 0; base < len; base += 256) {
    uint32_t i = base + threadIdx.x;
    uint64_t o = 0, m = 0;
    if (i < len) {
      const Node& nd = nodes[chain_nodes[J.node0 + i]];
      o = nd.out_len;
      m = nd.nmatch;
    }
    uint64_t xo, xm, ao, am;
    Scan(t1).ExclusiveSum(o, xo, ao);
    Scan(t2).ExclusiveSum(m, xm, am);
    if (i < len) {
      out_off[J.node0 + i] = c_out + xo;
      m_off[J.node0 + i] = c_m + xm;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      c_out += ao;
      c_m += am;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    totals[2 * j] = c_out;
    totals[2 * j + 1] = c_m;
  }
}

__global__ void k_copy_stored(const PJob* __restrict__ jobs, const Chain* __restrict__ chains,
                              const uint32_t* __restrict__ chain_nodes, const Node* __restrict__ nodes,
                              const uint64_t* __restrict__ out_off, const uint32_t* __restrict__ job_of_block,
                              const uint32_t* __restrict__ block_base) {
  const uint32_t j = job_of_block[blockIdx.x];
  const PJob J = jobs[j];
  const uint32_t i = blockIdx.x - block_base[j];
  if (i >= chains[j].len) return;
  const Node nd = nodes[chain_nodes[J.node0 + i]];
  if (!(nd.flags & 4)) return;
  const uint8_t* s = J.src + nd.start + 4;
  uint8_t* d = J.dst + out_off[J.node0 + i];
  const uint64_t len = nd.out_len;
  // aligned 16-byte output words, sources gathered with aligned loads
  const uintptr_t da = reinterpret_cast<uintptr_t>(d);
  const uint64_t head0 = (16 - (da & 15)) & 15;
  const uint64_t head = head0 < len ? head0 : len;
  const uint64_t words = (len - head) / 16;
  for (uint64_t w = threadIdx.x; w < words; w += blockDim.x) {
    uint32_t v[4];
    gather16(s + head + 16 * w, v);
    *reinterpret_cast<uint4*>(d + head + 16 * w) = make_uint4(v[0], v[1], v[2], v[3]);
  }
  for (uint64_t k = threadIdx.x; k < head; k += blockDim.x) d[k] = s[k];
  for (uint64_t k = head + 16 * words + threadIdx.x; k < len; k += blockDim.x) d[k] = s[k];
}

// Sequential continuation after a BREAK (static block not covered by a node) and
// the trailer.  One thread per job.
__global__ void k_tail(const PJob* __restrict__ jobs, int njobs, const Chain* __restrict__ chains,
                       const Node* __restrict__ nodes, const uint64_t* __restrict__ totals,
                       Match* __restrict__ matches, uint32_t* __restrict__ fail, uint64_t* __restrict__ out_total,
                       uint32_t* __restrict__ want_adler, Tables* __restrict__ tabs) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= njobs) return;
  const PJob J = jobs[j];
  const Chain C = chains[j];
  uint64_t out_len = totals[2 * j];
  uint64_t nm = totals[2 * j + 1];
  const Node last = nodes[C.last];
  uint64_t end = last.end_bit;
  if (C.terminal == SENT_BAD) {
    fail[j] = 1;
    return;
  }
  if (C.terminal == SENT_BREAK) {
    Tables* T = tabs + j;
    BitReader r;
    r.init(J.src, J.n, end);
    bool final_seen = false;
    while (!final_seen) {
      uint32_t h = r.take(3);
      if (r.past_end()) {
        fail[j] = 1;
        return;
      }
      final_seen = h & 1;
      uint32_t type = (h >> 1) & 3;
      int rc = 0;
      uint32_t nmatch = 0;
      uint64_t before = out_len;
      if (type == 0) {
        uint64_t B = (r.pos + 7) >> 3;
        if (B + 4 > J.n) {
          fail[j] = 1;
          return;
        }
        uint32_t len = J.src[B] | ((uint32_t)J.src[B + 1] << 8);
        uint32_t nlen = J.src[B + 2] | ((uint32_t)J.src[B + 3] << 8);
        if (len != (~nlen & 0xffff) || B + 4 + len > J.n || out_len + len > J.expected) {
          fail[j] = 1;
          return;
        }
        for (uint32_t k = 0; k < len; k++) J.dst[out_len + k] = J.src[B + 4 + k];
        out_len += len;
        r.init(J.src, J.n, 8 * (B + 4 + len));
        continue;
      } else if (type == 1) {
        static_tables(T);
      } else if (type == 2) {
        rc = read_dynamic(r, T);
      } else {
        rc = -1;
      }
      uint64_t added = 0;
      if (!rc)
        rc = decode_codes<true>(r, T, added, nmatch, J.expected - before, J.dst, before, matches + J.mbase + nm,
                                J.mcap - nm);
      if (rc) {
        fail[j] = 1;
        return;
      }
      out_len = before + added;
      nm += nmatch;
    }
    end = r.pos;
  }
  out_total[2 * j] = out_len;
  out_total[2 * j + 1] = nm;
  // trailer: byte-aligned big-endian Adler-32
  uint64_t tb = (end + 7) >> 3;
  if (tb + 4 > J.n) {
    fail[j] = 1;
    return;
  }
  want_adler[j] = ((uint32_t)J.src[tb] << 24) | ((uint32_t)J.src[tb + 1] << 16) | ((uint32_t)J.src[tb + 2] << 8) |
                  J.src[tb + 3];
  if (out_len != J.expected) fail[j] = 1;
}

// ---- P6 --------------------------------------------------------------------
// lower bound: first match with dst + len > x (matches sorted by dst)
__device__ uint64_t first_match_after(const Match* m, uint64_t count, uint64_t x) {
  uint64_t lo = 0, hi = count;
  while (lo < hi) {
    uint64_t mid = (lo + hi) >> 1;
    if ((uint64_t)m[mid].dst + m[mid].len > x) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

constexpr uint32_t RESOLVED = 0x80000000u;
#ifndef RS_THREADS_OVR
#define RS_THREADS_OVR 1024
#endif
constexpr int RS_THREADS = RS_THREADS_OVR;
constexpr uint32_t RS_SMEM = SUB * 4 + SUB;  // window entries + the TMA-staged raw bytes

struct ExtEntry {
  uint32_t dst;
  uint32_t src;
};

// window entries <- RESOLVED | byte.  The window's bytes (already written literals and
// stored runs) are staged into shared memory by a TMA bulk copy (16-byte aligned part) and
// expanded from there 16 at a time; `raw` holds SUB bytes behind the SUB entries.
__device__ __forceinline__ void fill_entries(uint32_t* ent, uint8_t* raw, uint64_t* bar, const uint8_t* src,
                                             uint32_t w, uint32_t total) {
  const bool aligned = (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  const uint32_t wa = aligned ? (w & ~15u) : 0u;  // bytes moved by the copy engine
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    if (wa) tma_load_1d(raw, src, wa, bar);
  }
  __syncthreads();
  if (wa) mbar_wait(bar, 0);
  const uint4* r4 = reinterpret_cast<const uint4*>(raw);
  for (uint32_t v = threadIdx.x; v < wa / 16; v += blockDim.x) {
    const uint4 x = r4[v];
    const uint32_t wd[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 16; k++) ent[16 * v + k] = RESOLVED | ((wd[k >> 2] >> (8 * (k & 3))) & 0xff);
  }
  for (uint32_t i = wa + threadIdx.x; i < total; i += blockDim.x) ent[i] = RESOLVED | (i < w ? src[i] : 0u);
}

__global__ void __launch_bounds__(RS_THREADS) k_resolve_local(const PJob* __restrict__ jobs,
                                                              const uint32_t* __restrict__ job_of_sub,
                                                              const uint64_t* __restrict__ out_total,
                                                              uint32_t* __restrict__ fail,
                                                              const Match* __restrict__ matches,
                                                              ExtEntry* __restrict__ ext,
                                                              uint32_t* __restrict__ ext_cnt,
                                                              uint32_t* __restrict__ extp,
                                                              uint8_t* __restrict__ wflag) {
  extern __shared__ uint32_t ent[];  // SUB entries: RESOLVED | value, or source relative to S - 65536
  __shared__ int changed;
  __shared__ __align__(8) uint64_t s_bar;  // TMA completion of the window's bytes
  __shared__ uint32_t s_cnt;
  const uint32_t j = job_of_sub[blockIdx.x];
  const PJob J = jobs[j];
  const uint32_t sub = blockIdx.x - J.sub0;
  if (fail[j]) return;
  const uint64_t total = out_total[2 * j];
  const uint64_t S = (uint64_t)sub * SUB;
  if (S >= total) return;
  const uint32_t W = (uint32_t)min((uint64_t)SUB, total - S);
  const uint64_t nm = out_total[2 * j + 1];
  const Match* M = matches + J.mbase;
  // match bytes -> source pointers
  const uint64_t m0 = first_match_after(M, nm, S);
  if (m0 >= nm || M[m0].dst >= S + W) {  // no match reaches this window: bytes are final
    if (threadIdx.x == 0) {
      wflag[blockIdx.x] = 0;
      ext_cnt[blockIdx.x] = 0;
    }
    return;
  }
  if (threadIdx.x == 0) wflag[blockIdx.x] = 1;
  fill_entries(ent, reinterpret_cast<uint8_t*>(ent + SUB), &s_bar, J.dst + S, W, W);
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  __shared__ int corrupt;
  if (threadIdx.x == 0) corrupt = 0;
  __syncthreads();
  for (uint64_t k = m0 + threadIdx.x; k < nm && M[k].dst < S + W; k += blockDim.x) {
    const Match mt = M[k];
    if (mt.dist == 0 || mt.dist > mt.dst || mt.len < 3 || mt.len > 258) {
      corrupt = 1;  // never produced by a valid decode: let the exact decoder take the job
      continue;
    }
    uint64_t a = max((uint64_t)mt.dst, S), b = min((uint64_t)mt.dst + mt.len, S + W);
    for (uint64_t x = a; x < b; x++) ent[x - S] = (uint32_t)(x - mt.dist - S + 65536);
  }
  __syncthreads();
  if (corrupt) {
    if (threadIdx.x == 0) atomicExch(&fail[j], 1u);
    return;
  }
  // pointer jumping inside the window (every pointer goes strictly backwards)
  int rounds = 0;
  do {
    __syncthreads();
    if (threadIdx.x == 0) changed = 0;
    if (++rounds > 40) {
      if (threadIdx.x == 0) atomicExch(&fail[j], 1u);
      return;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) {
      uint32_t e = ent[i];
      if (e & RESOLVED) continue;
      if (e < 65536) continue;  // source before the window: external
      uint32_t t = ent[e - 65536];
      ent[i] = t;  // either the resolved value or a pointer closer to the root
      changed = 1;
    }
    __syncthreads();
  } while (changed);
  for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) {
    uint32_t e = ent[i];
    if (e & RESOLVED) {
      J.dst[S + i] = (uint8_t)e;
      extp[J.xbase + S + i] = 0xFFFFFFFFu;
    } else {
      uint32_t k = atomicAdd(&s_cnt, 1u);
      const uint32_t src = (uint32_t)(S + e - 65536);
      ext[(uint64_t)blockIdx.x * SUB + k] = ExtEntry{(uint32_t)(S + i), src};
      extp[J.xbase + S + i] = src;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) ext_cnt[blockIdx.x] = s_cnt;
}

// P6 (current): the pointer jumping runs over RS_CL consecutive windows of a
// lane at once -- a thread-block cluster whose CTAs each hold one 32 KiB window
// in shared memory and read their neighbours' entries through distributed
// shared memory.  Copy chains are long (literals are rare in exponent planes and
// each hop goes back up to 32 KiB), so a larger window leaves fewer bytes
// (and shorter chains) to k_resolve_chase.  Entries: RESOLVED | byte, or the
// source as an offset from (cluster base - 65536); < 65536 = before the cluster.
namespace cg = cooperative_groups;
constexpr int RS_CL = 2;

__global__ void __cluster_dims__(RS_CL, 1, 1) __launch_bounds__(RS_THREADS)
    k_resolve_cluster(const PJob* __restrict__ jobs, const uint2* __restrict__ cl_map,
                      const uint64_t* __restrict__ out_total, uint32_t* __restrict__ fail,
                      const Match* __restrict__ matches, ExtEntry* __restrict__ ext, uint32_t* __restrict__ ext_cnt,
                      uint32_t* __restrict__ extp, uint8_t* __restrict__ wflag) {
  extern __shared__ uint32_t ent[];
  __shared__ int s_corrupt, s_anyv[3];
  __shared__ __align__(8) uint64_t s_bar;  // TMA completion of the window's bytes
  __shared__ uint32_t s_cnt;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  const uint2 cm = cl_map[blockIdx.x / RS_CL];  // (job, first window of the cluster)
  const uint32_t j = cm.x;
  const PJob J = jobs[j];
  const uint32_t w = cm.y + rank;
  const bool failed = fail[j] != 0;
  const uint64_t total = out_total[2 * j];
  const uint64_t CB = (uint64_t)cm.y * SUB;  // cluster base position
  const uint64_t S = (uint64_t)w * SUB;
  const uint32_t Wn = (!failed && w < J.nsub && S < total) ? (uint32_t)min((uint64_t)SUB, total - S) : 0;
  const uint32_t g = J.sub0 + w;  // global window index (valid only if w < nsub)
  const uint64_t nm = out_total[2 * j + 1];
  const Match* M = matches + J.mbase;
  uint64_t m0 = 0;
  bool has_m = false;
  if (Wn) {
    m0 = first_match_after(M, nm, S);
    has_m = m0 < nm && M[m0].dst < S + Wn;
  }
  if (threadIdx.x == 0) {
    s_corrupt = 0;
    s_cnt = 0;
    s_anyv[0] = 0;
    if (w < J.nsub) wflag[g] = has_m ? 1 : 0;
  }
  // a cluster none of whose windows holds a match (e.g. stored mantissa planes) is done
  cl.sync();
  if (threadIdx.x == 0 && has_m) atomicOr(cl.map_shared_rank(&s_anyv[0], 0), 1);
  cl.sync();
  if (!*cl.map_shared_rank(&s_anyv[0], 0)) {
    if (threadIdx.x == 0 && w < J.nsub) ext_cnt[g] = 0;
    cl.sync();  // rank 0's flag is read by all before anyone exits
    return;
  }
  fill_entries(ent, reinterpret_cast<uint8_t*>(ent + SUB), &s_bar, J.dst + S, Wn, SUB);
  __syncthreads();
  if (has_m) {
    for (uint64_t k = m0 + threadIdx.x; k < nm && M[k].dst < S + Wn; k += blockDim.x) {
      const Match mt = M[k];
      if (mt.dist == 0 || mt.dist > mt.dst || mt.len < 3 || mt.len > 258) {
        s_corrupt = 1;
        continue;
      }
      const uint64_t a = max((uint64_t)mt.dst, S), b = min((uint64_t)mt.dst + mt.len, S + Wn);
      for (uint64_t x = a; x < b; x++) ent[x - S] = (uint32_t)(x - mt.dist + 65536 - CB);
    }
  }
  cl.sync();
  // pointer jumping over the cluster's windows (reads of neighbours may see an
  // older or newer entry of the same chain: both are valid, pointers only move
  // toward their roots).  Each thread keeps a bit mask of its still-unresolved
  // entries (entry threadIdx.x + 1024 k -> bit k); the cluster-wide "anything
  // changed" flag is triple-buffered in rank 0's shared memory so one cluster
  // barrier per round suffices (flag r+1 is cleared in round r, when every CTA
  // has long finished reading flag r-2, the same slot).
  uint32_t pend = 0;
  for (uint32_t k = 0; k < SUB / RS_THREADS; k++) {
    const uint32_t i = threadIdx.x + k * RS_THREADS;
    if (i < Wn && !(ent[i] & RESOLVED) && ent[i] >= 65536) pend |= 1u << k;
  }
  if (threadIdx.x < 3) s_anyv[threadIdx.x] = 0;
  cl.sync();
  int rounds = 0;
  for (;;) {
    const int slot = rounds % 3;
    if (rank == 0 && threadIdx.x == 0) s_anyv[(rounds + 1) % 3] = 0;
    uint32_t next = 0;
    for (uint32_t m = pend; m; m &= m - 1) {
      const uint32_t k = __ffs(m) - 1;
      const uint32_t i = threadIdx.x + k * RS_THREADS;
      const uint32_t e = ent[i];
      const uint32_t idx = e - 65536;
      const unsigned r = idx / SUB;
      const uint32_t o = idx % SUB;
      const uint32_t t = r == rank ? ent[o] : *cl.map_shared_rank(ent + o, r);
      ent[i] = t;
      if (!(t & RESOLVED) && t >= 65536) next |= 1u << k;
    }
    const int ch = __syncthreads_or(pend != 0);
    pend = next;
    if (threadIdx.x == 0 && ch) atomicOr(cl.map_shared_rank(&s_anyv[slot], 0), 1);
    cl.sync();
    const int any = *cl.map_shared_rank(&s_anyv[slot], 0);
    if (!any || ++rounds > 48) break;
  }
  if (Wn && (s_corrupt || rounds > 48)) {
    if (threadIdx.x == 0) atomicExch(&fail[j], 1u);
  } else if (has_m) {
    for (uint32_t i = threadIdx.x; i < Wn; i += blockDim.x) {
      const uint32_t e = ent[i];
      if (e & RESOLVED) {
        J.dst[S + i] = (uint8_t)e;
        extp[J.xbase + S + i] = 0xFFFFFFFFu;
      } else {
        const uint32_t k = atomicAdd(&s_cnt, 1u);
        const uint32_t src = (uint32_t)(CB + e - 65536);
        ext[(uint64_t)g * SUB + k] = ExtEntry{(uint32_t)(S + i), src};
        extp[J.xbase + S + i] = src;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && w < J.nsub) ext_cnt[g] = has_m && !s_corrupt ? s_cnt : 0;
  cl.sync();  // no CTA may exit while a neighbour can still read its shared memory
}

// Pointer doubling over the unresolved bytes' source map before the chase: one
// round moves every pending pointer to its source's pointer, so after R rounds a
// chain of h hops has ~h / 2^R left.  Chains are long where a lane repeats a
// short period for many windows (the f32 token-tree planes of config3: every
// hop of the chase would be one dependent global load, one window back).
// Entries are read and written concurrently across CTAs; as in the cluster
// pass, a reader sees an older or a newer pointer of the same chain, and both
// lead to the same root.
#ifndef RJ_ROUNDS
#define RJ_ROUNDS 4  // cap on the rounds (the sampled mean chain length decides how many run)
#endif
constexpr int RJ_MAX = 16;
constexpr uint32_t RJ_SAMPLE = 256;  // one sampled chain per 256 unresolved bytes
// The rounds pay off only where chains are long, and each costs a pass over all
// unresolved bytes, so their number is decided on the device from a sampled
// chase: jstat[0] = hops, jstat[1] = chains sampled; round r runs while the mean
// chain is longer than 4 << r hops (the bf16 activations of config2 average a few
// hops and skip the rounds; the f32 token-tree planes of config3 run them).
__global__ void __launch_bounds__(32) k_resolve_sample(const PJob* __restrict__ jobs,
                                                      const uint32_t* __restrict__ job_of_sub,
                                                      const uint32_t* __restrict__ fail,
                                                      const ExtEntry* __restrict__ ext,
                                                      const uint32_t* __restrict__ ext_cnt,
                                                      const uint32_t* __restrict__ extp,
                                                      const uint8_t* __restrict__ wflag, unsigned long long* jstat,
                                                      uint32_t cap) {
  const uint32_t j = job_of_sub[blockIdx.x];
  const PJob J = jobs[j];
  const uint32_t c = fail[j] ? 0u : ext_cnt[blockIdx.x];
  const ExtEntry* E = ext + (uint64_t)blockIdx.x * SUB;
  const uint32_t* X = extp + J.xbase;
  const uint8_t* WF = wflag + J.sub0;
  uint32_t hops = 0, n = 0;
  for (uint32_t k = threadIdx.x * RJ_SAMPLE; k < c; k += 32 * RJ_SAMPLE) {
    uint32_t v = E[k].src, w, h = 1;
    // capped at twice the last round's threshold (cap): the gate needs no more, and
    // the sampled chase is itself a dependent-load walk (133 hops mean on config3)
    while (h < cap && WF[v / SUB] && (w = X[v]) != 0xFFFFFFFFu && w < v) v = w, h++;
    hops += h;
    n++;
  }
  hops = __reduce_add_sync(0xffffffffu, hops);
  n = __reduce_add_sync(0xffffffffu, n);
  if (threadIdx.x == 0 && n) {
    atomicAdd(jstat, (unsigned long long)hops);
    atomicAdd(jstat + 1, (unsigned long long)n);
  }
}

__global__ void __launch_bounds__(1024) k_resolve_jump(const PJob* __restrict__ jobs,
                                                       const uint32_t* __restrict__ job_of_sub,
                                                       const uint32_t* __restrict__ fail,
                                                       const ExtEntry* __restrict__ ext,
                                                       const uint32_t* __restrict__ ext_cnt, uint32_t* extp,
                                                       const uint8_t* __restrict__ wflag,
                                                       const unsigned long long* __restrict__ jstat, int r) {
  if (jstat[0] <= jstat[1] * (4ull << r)) return;
  const uint32_t j = job_of_sub[blockIdx.x];
  const PJob J = jobs[j];
  if (fail[j]) return;
  const uint32_t c = ext_cnt[blockIdx.x];
  const ExtEntry* E = ext + (uint64_t)blockIdx.x * SUB;
  uint32_t* X = extp + J.xbase;
  const uint8_t* WF = wflag + J.sub0;
  for (uint32_t k = threadIdx.x; k < c; k += blockDim.x) {
    const uint32_t d = E[k].dst;
    const uint32_t v = *(volatile uint32_t*)(X + d);
    if (v >= d || !WF[v / SUB]) continue;  // corrupt (left to the chase) or resolved root
    const uint32_t w = *(volatile uint32_t*)(X + v);
    if (w != 0xFFFFFFFFu && w < v) X[d] = w;
  }
}

// Every byte left unresolved by its window points to an earlier byte; chase
// the pointers (read-only map) to a byte its own window resolved.  Fully
// parallel over all windows of all lanes.
#ifndef RC_THREADS
#define RC_THREADS 1024
#endif
__global__ void __launch_bounds__(RC_THREADS) k_resolve_chase(const PJob* __restrict__ jobs,
                                                      const uint32_t* __restrict__ job_of_sub,
                                                      uint32_t* __restrict__ fail,
                                                      const ExtEntry* __restrict__ ext,
                                                      const uint32_t* __restrict__ ext_cnt,
                                                      const uint32_t* __restrict__ extp,
                                                      const uint8_t* __restrict__ wflag) {
  const uint32_t j = job_of_sub[blockIdx.x];
  const PJob J = jobs[j];
  if (fail[j]) return;
  const uint64_t S0 = (uint64_t)(blockIdx.x - J.sub0) * SUB;
  (void)S0;
  const uint32_t c = ext_cnt[blockIdx.x];
  const ExtEntry* E = ext + (uint64_t)blockIdx.x * SUB;
  const uint32_t* X = extp + J.xbase;
  for (uint32_t k = threadIdx.x; k < c; k += blockDim.x) {
    const ExtEntry e = E[k];
    const uint8_t* WF = wflag + J.sub0;
    uint32_t v = e.src, w;
    while (WF[v / SUB] && (w = X[v]) != 0xFFFFFFFFu) {
      if (w >= v) {  // sources always lie strictly earlier
        atomicExch(&fail[j], 1u);
        return;
      }
      v = w;
    }
    J.dst[e.dst] = J.dst[v];
  }
}

// ---- P7 Adler ---------------------------------------------------------------
constexpr int PA_THREADS = 256;
constexpr uint64_t PA_CHUNK = 64 * 1024;

__global__ void __launch_bounds__(PA_THREADS) k_adler_part(const PJob* __restrict__ jobs,
                                                          const uint32_t* __restrict__ job_of_chunk,
                                                          const uint32_t* __restrict__ chunk_base,
                                                          uint4* __restrict__ part) {
  __shared__ uint32_t wa[PA_THREADS / 32], wb[PA_THREADS / 32];
  __shared__ uint64_t wm[PA_THREADS / 32];
  const uint32_t j = job_of_chunk[blockIdx.x];
  const PJob J = jobs[j];
  const uint64_t c = blockIdx.x - chunk_base[j];
  const uint64_t per = PA_CHUNK / PA_THREADS;
  const uint64_t c0 = min(c * PA_CHUNK + threadIdx.x * per, J.expected);
  const uint64_t c1 = min(c0 + per, min((c + 1) * PA_CHUNK, J.expected));
  uint64_t A = 0, B = 0;
  uint64_t i = c0;
  for (; i + 16 <= c1; i += 16) {
    uint32_t v[4];
    gather16(J.dst + i, v);
    // 16 sequential (A += b, B += A) steps: A' = A + sum b, B' = B + 16 A + sum (16 - k) b_k
    const uint32_t sb = __dp4a(v[0], 0x01010101u, __dp4a(v[1], 0x01010101u, __dp4a(v[2], 0x01010101u, __dp4a(v[3], 0x01010101u, 0u))));
    const uint32_t wb = __dp4a(v[0], 0x0d0e0f10u, __dp4a(v[1], 0x090a0b0cu, __dp4a(v[2], 0x05060708u, __dp4a(v[3], 0x01020304u, 0u))));
    B += 16 * A + wb;
    A += sb;
  }
  for (; i < c1; i++) {
    A += J.dst[i];
    B += A;
  }
  A %= MOD;
  B %= MOD;
  uint64_t m = c1 - c0;
  for (int off = 1; off < 32; off <<= 1) {
    uint64_t rA = __shfl_down_sync(0xffffffffu, A, off);
    uint64_t rB = __shfl_down_sync(0xffffffffu, B, off);
    uint64_t rm = __shfl_down_sync(0xffffffffu, m, off);
    int lane = threadIdx.x & 31;
    if (lane + off < 32 && (lane & (2 * off - 1)) == 0) {
      B = (B + rB + (rm % MOD) * A) % MOD;
      A = (A + rA) % MOD;
      m += rm;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    wa[threadIdx.x >> 5] = (uint32_t)A;
    wb[threadIdx.x >> 5] = (uint32_t)B;
    wm[threadIdx.x >> 5] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t TA = 0, TB = 0, TM = 0;
    for (int w = 0; w < PA_THREADS / 32; w++) {
      TB = (TB + wb[w] + (wm[w] % MOD) * TA) % MOD;
      TA = (TA + wa[w]) % MOD;
      TM += wm[w];
    }
    part[blockIdx.x] = make_uint4((uint32_t)TA, (uint32_t)TB, (uint32_t)TM, (uint32_t)(TM >> 32));
  }
}

__global__ void k_adler_check(const PJob* __restrict__ jobs, int njobs, const uint32_t* __restrict__ chunk_base,
                              const uint4* __restrict__ part, const uint32_t* __restrict__ want,
                              uint32_t* __restrict__ fail) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= njobs || fail[j]) return;
  const PJob J = jobs[j];
  // the zlib header (inflate.c HEAD state, as inflate_stream checks it): decoding starts at
  // bit 16, so a bad CMF/FLG must fail here and go to the exact decoder for its status
  {
    const uint32_t cmf = J.src[0], flg = J.src[1];
    if (((cmf << 8) | flg) % 31u != 0 || (cmf & 0x0f) != 8 || (cmf >> 4) > 7 || (flg & 0x20)) {
      fail[j] = 1;
      return;
    }
  }
  uint64_t nch = (J.expected + PA_CHUNK - 1) / PA_CHUNK;
  uint64_t TA = 0, TB = 0;
  for (uint64_t c = 0; c < nch; c++) {
    uint4 p = part[chunk_base[j] + c];
    uint64_t m = p.z | ((uint64_t)p.w << 32);
    TB = (TB + p.y + (m % MOD) * TA) % MOD;
    TA = (TA + p.x) % MOD;
  }
  uint32_t a = (uint32_t)((1 + TA) % MOD), b = (uint32_t)((J.expected % MOD + TB) % MOD);
  if (((b << 16) | a) != want[j]) fail[j] = 1;
}

}  // namespace par

// ---------------------------------------------------------------------------
// host orchestration

struct ParInflate {
  Workspace ws, nodesw, lists;
  uint32_t* h_pin = nullptr;
  size_t h_cap = 0;
  void* scan_tmp = nullptr;
  size_t scan_cap = 0;
  uint64_t* cnt_idx = nullptr;  // device: 4 prefix indices per job (node counts), then the gathered values
  size_t cnt_cap = 0;
  ~ParInflate() {
    if (h_pin) cudaFreeHost(h_pin);
    if (scan_tmp) cudaFree(scan_tmp);
    if (cnt_idx) cudaFree(cnt_idx);
  }
};

ParInflate* par_inflate_create() { return new ParInflate(); }
void par_inflate_destroy(ParInflate* p) { delete p; }

int par_inflate(ParInflate* P, const std::vector<InflateJob>& jobs, cudaStream_t st, int* ok, int find_dynamic) {
  using namespace par;
  const int nj = (int)jobs.size();
  if (!nj) return BB_OK;
  StageTimer T(st);
  T.mark("inflate.setup");
  // shared-memory opt-ins are per device: one flag per device, set under a lock
  static std::mutex attr_mu;
  static bool attr_done[64] = {};
  size_t nd_smem = sizeof(Tables) * ND_THREADS;
  int dev = 0;
  BB_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return BB_INVALID_ARG;
  {
    std::lock_guard<std::mutex> attr_lock(attr_mu);
    if (!attr_done[dev]) {
      BB_CUDA_TRY(cudaFuncSetAttribute(k_decode_nodes, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nd_smem));
      BB_CUDA_TRY(cudaFuncSetAttribute(k_resolve_local, cudaFuncAttributeMaxDynamicSharedMemorySize, RS_SMEM));
      BB_CUDA_TRY(cudaFuncSetAttribute(k_resolve_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, RS_SMEM));
      BB_CUDA_TRY(cudaFuncSetAttribute(k_dyn_scan<DS_MINB_WIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(WarpSm) * WD_WARPS)));
      BB_CUDA_TRY(cudaFuncSetAttribute(k_dyn_scan<DS_MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(WarpSm) * WD_WARPS)));
      attr_done[dev] = true;
    }
  }
  std::vector<PJob> J(nj);
  std::vector<uint32_t> sub_job, chunk_job, chunk_base(nj);
  std::vector<uint64_t> blk_prefix(nj + 1, 0);
  uint64_t dwords = 0, swords = 0, mtot = 0, xtot = 0, ntot_bytes = 0;
  uint32_t subs = 0;
  for (int i = 0; i < nj; i++) {
    PJob& p = J[i];
    p = PJob{};
    p.src = jobs[i].src;
    p.n = jobs[i].n;
    p.dst = jobs[i].dst;
    p.expected = jobs[i].expected;
    p.dbm = dwords;
    p.sbm = swords;
    dwords += (p.n + 3) / 4 + 1;
    swords += (p.n + 31) / 32 + 2;
    p.mbase = mtot;
    p.mcap = p.expected / 3 + 1;
    mtot += p.mcap;
    ntot_bytes += p.n;
    p.xbase = xtot;
    xtot += p.expected;
    p.sub0 = subs;
    p.nsub = (uint32_t)((p.expected + SUB - 1) / SUB);
    subs += p.nsub;
    for (uint32_t s = 0; s < p.nsub; s++) sub_job.push_back(i);
    blk_prefix[i + 1] = blk_prefix[i] + (p.n + 1023) / 1024;
    chunk_base[i] = (uint32_t)chunk_job.size();
    for (uint64_t c = 0; c * PA_CHUNK < p.expected; c++) chunk_job.push_back(i);
  }
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const uint64_t cand_blocks = blk_prefix[nj];
  size_t need = al(sizeof(PJob) * nj) + al(8 * (nj + 1)) + 2 * al(4 * dwords) +
                2 * al(4 * swords) + al(4 * sub_job.size() + 4) + al(4 * chunk_job.size() + 4) + al(4 * nj) +
                al(16 * chunk_job.size() + 16) + al(sizeof(Match) * mtot) + al(sizeof(ExtEntry) * (uint64_t)subs * SUB) +
                al(4 * subs + 4) + al(subs + 4) + al(4 * xtot + 4) + al(8 * (ntot_bytes / 2 + 4096)) + 256 + al(4 * nj) * 6 + al(16 * nj) * 4 + al(sizeof(Chain) * nj) +
                al(sizeof(Tables) * nj) + al(8 * ((uint64_t)subs + nj + 1)) + 65536;
  int rc = P->ws.reserve(need);
  if (rc) return rc;
  Workspace& W = P->ws;
  PJob* d_jobs = W.take<PJob>(nj);
  uint64_t* d_blk_prefix = W.take<uint64_t>(nj + 1);
  uint32_t* d_dbm = W.take<uint32_t>(dwords);
  uint32_t* d_dpre = W.take<uint32_t>(dwords);
  uint32_t* d_sbm = W.take<uint32_t>(swords);
  uint32_t* d_spre = W.take<uint32_t>(swords);
  uint32_t* d_sub_job = W.take<uint32_t>(sub_job.size() + 1);
  uint32_t* d_chunk_job = W.take<uint32_t>(chunk_job.size() + 1);
  uint32_t* d_chunk_base = W.take<uint32_t>(nj);
  uint4* d_part = W.take<uint4>(chunk_job.size() + 1);
  Match* d_matches = W.take<Match>(mtot);
  ExtEntry* d_ext = W.take<ExtEntry>((uint64_t)subs * SUB);
  uint32_t* d_ext_cnt = W.take<uint32_t>(subs + 1);
  uint32_t* d_extp = W.take<uint32_t>(xtot + 1);
  uint8_t* d_wflag = W.take<uint8_t>(subs + 1);
  uint2* d_clm = W.take<uint2>(subs + nj + 1);  // (job, first window) per resolution cluster
  unsigned long long* d_jstat = W.take<unsigned long long>(2);
  const uint64_t surv_cap = find_dynamic ? ntot_bytes / 2 + 4096 : 1;
  uint64_t* d_surv = W.take<uint64_t>(surv_cap);
  unsigned long long* d_surv_cnt = W.take<unsigned long long>(1);
  uint32_t* d_fail = W.take<uint32_t>(nj);
  uint32_t* d_want = W.take<uint32_t>(nj);
  uint64_t* d_totals = W.take<uint64_t>(2 * nj);
  uint64_t* d_out_total = W.take<uint64_t>(2 * nj);
  Chain* d_chains = W.take<Chain>(nj);
  Tables* d_tabs = W.take<Tables>(nj);

  BB_CUDA_TRY(cudaMemcpyAsync(d_jobs, J.data(), sizeof(PJob) * nj, cudaMemcpyHostToDevice, st));
  BB_CUDA_TRY(cudaMemcpyAsync(d_blk_prefix, blk_prefix.data(), 8 * (nj + 1), cudaMemcpyHostToDevice, st));
  if (!sub_job.empty())
    BB_CUDA_TRY(cudaMemcpyAsync(d_sub_job, sub_job.data(), 4 * sub_job.size(), cudaMemcpyHostToDevice, st));
  if (!chunk_job.empty())
    BB_CUDA_TRY(cudaMemcpyAsync(d_chunk_job, chunk_job.data(), 4 * chunk_job.size(), cudaMemcpyHostToDevice, st));
  BB_CUDA_TRY(cudaMemcpyAsync(d_chunk_base, chunk_base.data(), 4 * nj, cudaMemcpyHostToDevice, st));
  if (find_dynamic) BB_CUDA_TRY(cudaMemsetAsync(d_dbm, 0, 4 * dwords, st));
  else BB_CUDA_TRY(cudaMemsetAsync(d_dbm, 0, 4 * dwords, st));  // (bitmap must read as empty)
  BB_CUDA_TRY(cudaMemsetAsync(d_sbm, 0, 4 * swords, st));
  BB_CUDA_TRY(cudaMemsetAsync(d_fail, 0, 4 * nj, st));

  // P1
  BB_CUDA_TRY(cudaMemsetAsync(d_surv_cnt, 0, 8, st));
  T.mark(find_dynamic ? "inflate.candidates_dyn" : "inflate.candidates_stored");
  if (find_dynamic)
    k_candidates4<<<(unsigned)cand_blocks, 256, 0, st>>>(d_jobs, d_blk_prefix, nj, d_sbm, find_dynamic, d_surv,
                                                         d_surv_cnt, surv_cap);
  else
    k_stored_cand<<<(unsigned)cand_blocks, 64, 0, st>>>(d_jobs, d_blk_prefix, nj, d_sbm);
  BB_LAUNCH_CHECK();
  if (find_dynamic) {
    T.mark("inflate.verify_headers");
#ifndef VD_GRID_MUL
#define VD_GRID_MUL 8
#endif
    k_verify_dynamic<<<kNumSMs * VD_GRID_MUL, VD_THREADS, 0, st>>>(d_jobs, d_surv, d_surv_cnt, surv_cap, d_dbm, d_fail, nj);
    BB_LAUNCH_CHECK();
  }
  T.mark("inflate.rank_scan");
  k_popc<<<grid_for(dwords, 256, 8), 256, 0, st>>>(d_dbm, dwords, d_dpre);
  BB_LAUNCH_CHECK();
  k_popc<<<grid_for(swords, 256, 8), 256, 0, st>>>(d_sbm, swords, d_spre);
  BB_LAUNCH_CHECK();
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, d_dpre, d_dpre, (int)dwords, st);
  size_t tmp2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp2, d_spre, d_spre, (int)swords, st);
  tmp = std::max(tmp, tmp2);
  if (tmp > P->scan_cap) {
    if (P->scan_tmp) cudaFree(P->scan_tmp);
    BB_CUDA_TRY(cudaMalloc(&P->scan_tmp, tmp));
    P->scan_cap = tmp;
  }
  // exclusive scan in place (CUB supports aliasing for ExclusiveSum)
  BB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(P->scan_tmp, tmp, d_dpre, d_dpre, (int)dwords, st));
  BB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(P->scan_tmp, tmp, d_spre, d_spre, (int)swords, st));
  count_launch(2);
  // node counts per job -> host
  if ((size_t)(4 * nj + 8) > P->h_cap) {
    if (P->h_pin) cudaFreeHost(P->h_pin);
    BB_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&P->h_pin), 16 * nj + 64, cudaHostAllocDefault));
    P->h_cap = 4 * nj + 8;
  }
  {
    // count = prefix[next job's first word] - prefix[first word]; last words are padding (zero).
    // The 4 nj prefix values are gathered on the device and come back in one copy.
    std::vector<uint64_t> idx(4 * nj);
    for (int i = 0; i < nj; i++) {
      idx[4 * i] = J[i].dbm;
      idx[4 * i + 1] = J[i].dbm + (J[i].n + 3) / 4;
      idx[4 * i + 2] = J[i].sbm;
      idx[4 * i + 3] = J[i].sbm + (J[i].n + 31) / 32 + 1;
    }
    if ((size_t)(8 * nj) > P->cnt_cap) {
      if (P->cnt_idx) cudaFree(P->cnt_idx);
      BB_CUDA_TRY(cudaMalloc(&P->cnt_idx, 8 * 8 * (size_t)nj));
      P->cnt_cap = 8 * nj;
    }
    uint32_t* d_cnt = reinterpret_cast<uint32_t*>(P->cnt_idx + 4 * nj);
    BB_CUDA_TRY(cudaMemcpyAsync(P->cnt_idx, idx.data(), 8 * idx.size(), cudaMemcpyHostToDevice, st));
    k_gather_prefix<<<(4 * nj + 127) / 128, 128, 0, st>>>(P->cnt_idx, 4 * nj, d_dpre, d_spre, d_cnt);
    BB_LAUNCH_CHECK();
    BB_CUDA_TRY(cudaMemcpyAsync(P->h_pin, d_cnt, 16 * (size_t)nj, cudaMemcpyDeviceToHost, st));
  }
  BB_CUDA_TRY(cudaStreamSynchronize(st));
  uint32_t nnodes = 0, ndyn_total = 0;
  std::vector<uint32_t> node_job, dyn_nodes;
  for (int i = 0; i < nj; i++) {
    J[i].ndyn = P->h_pin[4 * i + 1] - P->h_pin[4 * i];
    J[i].nsto = P->h_pin[4 * i + 3] - P->h_pin[4 * i + 2];
    J[i].node0 = nnodes;
    J[i].dyn_base = ndyn_total;
    uint32_t cnt = 1 + J[i].ndyn + 2 * J[i].nsto;
    for (uint32_t k = 0; k < J[i].ndyn; k++) dyn_nodes.push_back(nnodes + 1 + k);
    ndyn_total += J[i].ndyn;
    nnodes += cnt;
    node_job.insert(node_job.end(), cnt, (uint32_t)i);
  }
  int levels = 1;
  while ((1u << levels) <= nnodes + 1) levels++;
  if (debug_sync())
    for (int i = 0; i < nj; i++)
      fprintf(stderr, "[bb] inflate job %d: n=%llu expected=%llu ndyn=%u nsto=%u find_dynamic=%d\n", i,
              (unsigned long long)J[i].n, (unsigned long long)J[i].expected, J[i].ndyn, J[i].nsto, find_dynamic);
  size_t need2 = al(sizeof(Node) * nnodes) + al(4 * nnodes) + al(4ull * nnodes * levels) + al(4 * nnodes) +
                 2 * al(8 * nnodes) + al(4ull * ndyn_total + 4) + al(sizeof(Tables) * (ndyn_total + 1)) +
                 al(sizeof(LanePlan) * 32ull * (ndyn_total + 1)) + al(sizeof(DynExtra) * (ndyn_total + 1)) + 8192;
  Workspace& nodesw = P->nodesw;
  rc = nodesw.reserve(need2);
  if (rc) return rc;
  Node* d_nodes = nodesw.take<Node>(nnodes);
  uint32_t* d_node_job = nodesw.take<uint32_t>(nnodes);
  uint32_t* d_jump = nodesw.take<uint32_t>((size_t)nnodes * levels);
  uint32_t* d_chain_nodes = nodesw.take<uint32_t>(nnodes);
  uint64_t* d_out_off = nodesw.take<uint64_t>(nnodes);
  uint64_t* d_m_off = nodesw.take<uint64_t>(nnodes);
  uint32_t* d_dyn_nodes = nodesw.take<uint32_t>(ndyn_total + 1);
  Tables* d_dtabs = nodesw.take<Tables>(ndyn_total + 1);
  LanePlan* d_plans = nodesw.take<LanePlan>(32ull * (ndyn_total + 1));
  DynExtra* d_extra = nodesw.take<DynExtra>(ndyn_total + 1);
  if (ndyn_total)
    BB_CUDA_TRY(cudaMemcpyAsync(d_dyn_nodes, dyn_nodes.data(), 4ull * ndyn_total, cudaMemcpyHostToDevice, st));
  T.mark("inflate.node_setup");
  BB_CUDA_TRY(cudaMemcpyAsync(d_jobs, J.data(), sizeof(PJob) * nj, cudaMemcpyHostToDevice, st));
  BB_CUDA_TRY(cudaMemcpyAsync(d_node_job, node_job.data(), 4 * nnodes, cudaMemcpyHostToDevice, st));
  BB_CUDA_TRY(cudaMemsetAsync(d_nodes, 0, sizeof(Node) * nnodes, st));
  // P2
  {
    dim3 g(grid_for(dwords + swords, 256, 8), nj);
    k_node_positions<<<g, 256, 0, st>>>(d_jobs, nj, d_dbm, d_dpre, d_sbm, d_spre, d_nodes);
    BB_LAUNCH_CHECK();
  }
  T.mark("inflate.decode_nodes");
  k_decode_nodes<<<(nnodes + ND_THREADS - 1) / ND_THREADS, ND_THREADS, nd_smem, st>>>(d_jobs, d_node_job, nnodes,
                                                                                      d_nodes);
  BB_LAUNCH_CHECK();
  if (ndyn_total) {
    const unsigned ds_grid = (ndyn_total + WD_WARPS - 1) / WD_WARPS;
    if (ndyn_total >= 4u * kNumSMs * WD_WARPS)
      k_dyn_scan<DS_MINB_WIDE><<<ds_grid, 32 * WD_WARPS, sizeof(WarpSm) * WD_WARPS, st>>>(
        d_jobs, d_node_job, d_dyn_nodes, ndyn_total, d_nodes, d_dtabs, d_plans, d_extra);
    else
      k_dyn_scan<DS_MINB><<<ds_grid, 32 * WD_WARPS, sizeof(WarpSm) * WD_WARPS, st>>>(
        d_jobs, d_node_job, d_dyn_nodes, ndyn_total, d_nodes, d_dtabs, d_plans, d_extra);
    BB_LAUNCH_CHECK();
  }
  T.mark("inflate.link_chain");
  // P3, P4
  k_link<<<(nnodes + 255) / 256, 256, 0, st>>>(d_jobs, d_node_job, nnodes, d_nodes, d_dbm, d_dpre, d_sbm, d_spre,
                                               d_jump);
  BB_LAUNCH_CHECK();
  if (nnodes <= LIFT1_MAX) {
    if (levels > 1) k_lift_all<<<1, LIFT1_MAX, 0, st>>>(d_jump, nnodes, levels);
    BB_LAUNCH_CHECK();
  } else {
    for (int k = 1; k < levels; k++) {
      k_lift<<<(nnodes + 255) / 256, 256, 0, st>>>(d_jump + (size_t)(k - 1) * nnodes, d_jump + (size_t)k * nnodes,
                                                   nnodes);
      BB_LAUNCH_CHECK();
    }
  }
  k_chain_len<<<(nj + 63) / 64, 64, 0, st>>>(d_jobs, nj, d_jump, nnodes, levels, d_chains);
  BB_LAUNCH_CHECK();
  {
    dim3 g(std::max<unsigned>(1, std::min<unsigned>((nnodes + 255) / 256, 64)), nj);  // grid-stride over each chain
    k_chain_nodes<<<g, 256, 0, st>>>(d_jobs, d_chains, d_jump, nnodes, levels, d_chain_nodes);
    BB_LAUNCH_CHECK();
  }
  k_chain_scan<<<nj, 256, 0, st>>>(d_jobs, d_chains, d_chain_nodes, d_nodes, d_out_off, d_m_off, d_totals);
  BB_LAUNCH_CHECK();
  // chain lengths to the host for the per-block launches
  std::vector<Chain> hc(nj);
  BB_CUDA_TRY(cudaMemcpyAsync(P->h_pin, d_chains, std::min<size_t>(sizeof(Chain) * nj, 16 * nj + 64),
                              cudaMemcpyDeviceToHost, st));
  BB_CUDA_TRY(cudaStreamSynchronize(st));
  std::memcpy(hc.data(), P->h_pin, sizeof(Chain) * nj);
  std::vector<uint32_t> emit_job, emit_base(nj), copy_job, copy_base(nj);
  for (int i = 0; i < nj; i++) {
    emit_base[i] = (uint32_t)emit_job.size();
    emit_job.insert(emit_job.end(), (hc[i].len + WD_WARPS - 1) / WD_WARPS, (uint32_t)i);
    copy_base[i] = (uint32_t)copy_job.size();
    copy_job.insert(copy_job.end(), hc[i].len, (uint32_t)i);
  }
  Workspace& lists = P->lists;
  rc = lists.reserve(4 * (emit_job.size() + copy_job.size() + 2 * nj) + 4096);
  if (rc) return rc;
  uint32_t* d_emit_job = lists.take<uint32_t>(emit_job.size() + 1);
  uint32_t* d_emit_base = lists.take<uint32_t>(nj);
  uint32_t* d_copy_job = lists.take<uint32_t>(copy_job.size() + 1);
  uint32_t* d_copy_base = lists.take<uint32_t>(nj);
  if (!emit_job.empty())
    BB_CUDA_TRY(cudaMemcpyAsync(d_emit_job, emit_job.data(), 4 * emit_job.size(), cudaMemcpyHostToDevice, st));
  BB_CUDA_TRY(cudaMemcpyAsync(d_emit_base, emit_base.data(), 4 * nj, cudaMemcpyHostToDevice, st));
  if (!copy_job.empty())
    BB_CUDA_TRY(cudaMemcpyAsync(d_copy_job, copy_job.data(), 4 * copy_job.size(), cudaMemcpyHostToDevice, st));
  BB_CUDA_TRY(cudaMemcpyAsync(d_copy_base, copy_base.data(), 4 * nj, cudaMemcpyHostToDevice, st));
  // P5
  T.mark("inflate.emit");
  if (!emit_job.empty()) {
    k_dyn_emit<<<(unsigned)emit_job.size(), 32 * WD_WARPS, sizeof(EmitSm) * WD_WARPS, st>>>(
        d_jobs, d_chains, d_chain_nodes, d_emit_job, d_emit_base, d_nodes, d_out_off, d_m_off, d_dtabs, d_plans,
        d_extra, d_matches, d_fail);
    BB_LAUNCH_CHECK();
  }
  if (!copy_job.empty()) {
    k_copy_stored<<<(unsigned)copy_job.size(), 256, 0, st>>>(d_jobs, d_chains, d_chain_nodes, d_nodes, d_out_off,
                                                             d_copy_job, d_copy_base);
    BB_LAUNCH_CHECK();
  }
  k_tail<<<(nj + 31) / 32, 32, 0, st>>>(d_jobs, nj, d_chains, d_nodes, d_totals, d_matches, d_fail, d_out_total,
                                        d_want, d_tabs);
  BB_LAUNCH_CHECK();
  // P6
  T.mark("inflate.resolve");
  if (!sub_job.empty()) {
    // stored-only pass (A): windows rarely hold matches, per-window CTAs exit at once;
    // the dynamic pass (B) resolves copy chains over clusters of windows
    static const bool single = getenv("BB_RESOLVE_SINGLE") != nullptr;
    if (single || !find_dynamic) {
      k_resolve_local<<<(unsigned)sub_job.size(), RS_THREADS, RS_SMEM, st>>>(d_jobs, d_sub_job, d_out_total, d_fail,
                                                                       d_matches, d_ext, d_ext_cnt, d_extp, d_wflag);
    } else {
      std::vector<uint2> clm;
      for (int i = 0; i < nj; i++)
        for (uint32_t w0 = 0; w0 < J[i].nsub; w0 += RS_CL) clm.push_back(make_uint2((uint32_t)i, w0));
      BB_CUDA_TRY(cudaMemcpyAsync(d_clm, clm.data(), sizeof(uint2) * clm.size(), cudaMemcpyHostToDevice, st));
      k_resolve_cluster<<<(unsigned)(clm.size() * RS_CL), RS_THREADS, RS_SMEM, st>>>(
          d_jobs, d_clm, d_out_total, d_fail, d_matches, d_ext, d_ext_cnt, d_extp, d_wflag);
    }
    BB_LAUNCH_CHECK();
    static const int jumps = std::min(RJ_MAX, getenv("BB_RESOLVE_JUMPS") ? atoi(getenv("BB_RESOLVE_JUMPS")) : RJ_ROUNDS);
    if (jumps > 0) {
      BB_CUDA_TRY(cudaMemsetAsync(d_jstat, 0, sizeof(unsigned long long) * 2, st));
      // each sampled chase is capped at 8 << jumps hops = 4x the last round's threshold (round r runs
      // while the mean exceeds 4 << r); the capped mean is biased low, so a long-chain workload can
      // run fewer rounds than it needs -- the chase after the rounds stays exact either way
      k_resolve_sample<<<(unsigned)sub_job.size(), 32, 0, st>>>(d_jobs, d_sub_job, d_fail, d_ext, d_ext_cnt, d_extp,
                                                                d_wflag, d_jstat, 8u << jumps);
      BB_LAUNCH_CHECK();
    }
    for (int r = 0; r < jumps; r++) {
      k_resolve_jump<<<(unsigned)sub_job.size(), 1024, 0, st>>>(d_jobs, d_sub_job, d_fail, d_ext, d_ext_cnt, d_extp,
                                                                 d_wflag, d_jstat, r);
      BB_LAUNCH_CHECK();
    }
    static const bool jdbg = getenv("BB_RESOLVE_DEBUG") != nullptr;
    if (jumps > 0 && jdbg) {
      unsigned long long h[2];
      BB_CUDA_TRY(cudaMemcpyAsync(h, d_jstat, sizeof(h), cudaMemcpyDeviceToHost, st));
      BB_CUDA_TRY(cudaStreamSynchronize(st));
      fprintf(stderr, "resolve: sampled %llu chains, mean %.1f hops\n", h[1], h[1] ? (double)h[0] / h[1] : 0.0);
    }
    k_resolve_chase<<<(unsigned)sub_job.size(), RC_THREADS, 0, st>>>(d_jobs, d_sub_job, d_fail, d_ext, d_ext_cnt, d_extp,
                                                             d_wflag);
    BB_LAUNCH_CHECK();
  }
  // P7
  T.mark("inflate.adler");
  if (!chunk_job.empty()) {
    k_adler_part<<<(unsigned)chunk_job.size(), PA_THREADS, 0, st>>>(d_jobs, d_chunk_job, d_chunk_base, d_part);
    BB_LAUNCH_CHECK();
  }
  k_adler_check<<<(nj + 63) / 64, 64, 0, st>>>(d_jobs, nj, d_chunk_base, d_part, d_want, d_fail);
  BB_LAUNCH_CHECK();
  BB_CUDA_TRY(cudaMemcpyAsync(P->h_pin, d_fail, 4 * nj, cudaMemcpyDeviceToHost, st));
  BB_CUDA_TRY(cudaStreamSynchronize(st));
  T.finish();
  for (int i = 0; i < nj; i++) ok[i] = P->h_pin[i] == 0;
  return BB_OK;
}

}  // namespace bb

extern "C" BB_API void bb_debug_inflate_guards(unsigned long long* out8) {
  cudaMemcpyFromSymbol(out8, bb::par::g_wd, sizeof(unsigned long long) * 8);
}
