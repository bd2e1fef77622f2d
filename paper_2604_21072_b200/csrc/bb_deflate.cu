// The deflate backend: zlib 1.3 compress2(level 6)-exact encoding on sm_100a.
//
// Reference: the deflate backend of the BBC1 codec (/root/reference/proj/src/
// codec.cpp:17-25) = zlib 1.3 compress2(..., Z_DEFAULT_COMPRESSION).  zlib is a
// third-party dependency (not vendored); its algorithm is restated on the CPU in
// oracle/zlib6.c, and every kernel below reproduces one stage of that
// restatement's decomposition (orc_zlib_compress_profiled), which is pinned
// byte-for-byte against libz.so.1.3 (tests/test_oracle.py).
//
// Pipeline over all lanes of a call (lanes = byte planes of every tensor):
//   K3 k_hash_prev6   prev-same-hash distance per position (zlib's head/prev
//      k_hash_fix2    chains, which are parse-independent: every position with
//                     3 bytes of lookahead is inserted, in order)
//   K4 k_profile3     longest_match() for every position: first maximum over the
//                     hash chain truncated at nice_match, after 32 and after 128
//                     candidates (the two chain budgets deflate_slow can use)
//   K5 k_parse_spec   deflate_slow's lazy-match state machine, one thread per
//                     segment, speculatively started from a fresh state
//      k_parse_fixup  re-parses each segment from its predecessor's true exit
//                     state until it meets the speculative parse in the same
//                     state at the same position (lazy parses resynchronise fast);
//                     repeated (Jacobi rounds) until no exit state changes
//   K6 k_compact      final symbol stream per lane
//      k_blocks       16383-symbol blocks: lit/len + dist histograms, zlib's
//                     build_tree / gen_bitlen / gen_codes / build_bl_tree, the
//                     dynamic header bits, opt_len / static_len
//      k_layout       per lane: stored / static / dynamic decision exactly as
//                     _tr_flush_block (incl. the slid-window stored rule), bit offsets
//   K7 k_emit         parallel bit packing of every block into the container
//      k_adler*       Adler-32 (chunk sums + ordered combine), zlib header/trailer,
//      k_finalize     BBC1 header
#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "bb_common.cuh"
#include "bb_kernels.h"

namespace bb {
namespace cg = cooperative_groups;

namespace {

constexpr uint32_t MIN_MATCH = 3, MAX_MATCH = 258, WSIZE = 32768, MAX_DIST = 32506;
constexpr uint32_t TOO_FAR = 4096, GOOD_LENGTH = 8, MAX_LAZY = 16, NICE_LENGTH = 128, MAX_CHAIN = 128;
constexpr uint32_t SYM_LIMIT = 16383;
constexpr uint32_t L_CODES = 286, D_CODES = 30, BL_CODES = 19, HEAP_SIZE = 2 * L_CODES + 1;
constexpr uint32_t PROF_AT_MAXDIST = 0x80000000u;

// K3 / K4 / K5 geometry
constexpr uint32_t HP_SEG = 32767;      // hash-prev segment (u16 relative heads)
constexpr uint32_t PF_SEG = 16384;      // profile segment
#ifndef PF_THREADS_OVR
constexpr int PF_THREADS = 1024;
#else
constexpr int PF_THREADS = PF_THREADS_OVR;
#endif
constexpr uint32_t CONV_W = 512;        // convergence window at each parse segment start
constexpr uint32_t HDR_BYTES = 640;     // dynamic tree header bits per block (<= 5000 bits)

// symbol: bit 31 = match; bits 0-7 = lc (literal or len-3); bits 8-22 = dist-1
constexpr uint32_t SYM_MATCH = 0x80000000u;

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint32_t sym_len(uint32_t s) { return (s & SYM_MATCH) ? (s & 0xff) + 3 : 1; }

// ---------------------------------------------------------------------------
// zlib static tables (trees.c tr_static_init), built once on the host
struct ZTables {
  uint8_t length_code[256];
  uint8_t dist_code[512];
  uint16_t base_length[29];
  uint16_t base_dist[30];
  uint16_t sl_code[288];
  uint8_t sl_len[288];
  uint16_t sd_code[30];
};
__constant__ ZTables c_z;
__constant__ uint8_t c_extra_lbits[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2,
                                          2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint8_t c_extra_dbits[30] = {0, 0, 0, 0, 1, 1, 2, 2,  3,  3,  4,  4,  5,  5,  6,
                                          6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
__constant__ uint8_t c_extra_blbits[19] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 2, 3, 7};
__constant__ uint8_t c_bl_order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

unsigned host_bi_reverse(unsigned code, int len) {
  unsigned res = 0;
  do {
    res |= code & 1;
    code >>= 1, res <<= 1;
  } while (--len > 0);
  return res >> 1;
}

ZTables make_tables() {
  static const int xl[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
  static const int xd[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
  ZTables t;
  memset(&t, 0, sizeof t);
  int length = 0, code, n, dist;
  for (code = 0; code < 28; code++) {
    t.base_length[code] = (uint16_t)length;
    for (n = 0; n < (1 << xl[code]); n++) t.length_code[length++] = (uint8_t)code;
  }
  t.length_code[length - 1] = (uint8_t)code;
  t.base_length[28] = 0;
  dist = 0;
  for (code = 0; code < 16; code++) {
    t.base_dist[code] = (uint16_t)dist;
    for (n = 0; n < (1 << xd[code]); n++) t.dist_code[dist++] = (uint8_t)code;
  }
  dist >>= 7;
  for (; code < 30; code++) {
    t.base_dist[code] = (uint16_t)(dist << 7);
    for (n = 0; n < (1 << (xd[code] - 7)); n++) t.dist_code[256 + dist++] = (uint8_t)code;
  }
  unsigned bl_count[16] = {0};
  for (n = 0; n <= 143; n++) t.sl_len[n] = 8, bl_count[8]++;
  for (; n <= 255; n++) t.sl_len[n] = 9, bl_count[9]++;
  for (; n <= 279; n++) t.sl_len[n] = 7, bl_count[7]++;
  for (; n <= 287; n++) t.sl_len[n] = 8, bl_count[8]++;
  unsigned next_code[16];
  unsigned c = 0;
  for (int bits = 1; bits <= 15; bits++) {
    c = (c + bl_count[bits - 1]) << 1;
    next_code[bits] = c;
  }
  for (n = 0; n <= 287; n++) t.sl_code[n] = (uint16_t)host_bi_reverse(next_code[t.sl_len[n]]++, t.sl_len[n]);
  for (n = 0; n < 30; n++) t.sd_code[n] = (uint16_t)host_bi_reverse((unsigned)n, 5);
  return t;
}

__device__ __forceinline__ uint32_t d_code(uint32_t dist) {
  return dist < 256 ? c_z.dist_code[dist] : c_z.dist_code[256 + (dist >> 7)];
}

// ---------------------------------------------------------------------------
// device-side per-lane descriptor
struct LaneDev {
  const uint8_t* src;
  uint64_t n;
  uint64_t pbase;    // base into per-position arrays (pd, prof)
  uint32_t seg0;     // first parse segment (global index)
  uint32_t nseg;     // parse segments
  uint32_t G;        // parse segment length
  uint32_t blk0;     // first block slot (global index)
  uint32_t nblk_max; // block slots reserved
  uint64_t sym_base; // base into the compacted symbol array
  int container, slot;
};

struct WorkItem {
  uint32_t lane;
  uint32_t start;
};

// parse state: bits 0-8 L (prev_length), bit 9 match_available, bits 10-24 prev
// distance (only when L >= 3), bit 31 valid
__device__ __forceinline__ uint32_t pack_state(uint32_t L, uint32_t avail, uint32_t dist) {
  return 0x80000000u | L | (avail << 9) | ((L >= MIN_MATCH ? dist : 0u) << 10);
}

struct SegExit {
  uint32_t p;      // exit loop-top position (lane-relative)
  uint32_t state;  // packed state at that loop top
};

// slides performed by zlib's fill_window() at or before loop top t (lane of n bytes)
__device__ __forceinline__ bool nil_head_at(uint64_t p, uint64_t n) {
  // a head MAX_DIST back is relative position 0 (NIL) right after a slide at
  // strstart == wsize + MAX_DIST, which fill_window only does near the end
  return p >= 65274 && ((p - 65274) & (WSIZE - 1)) == 0 && n - p <= 261;
}

__device__ __forceinline__ uint64_t slides_at(uint64_t t, uint64_t n) {
  uint64_t s = t >= 65275 ? (t - 65275) / WSIZE + 1 : 0;
  if (t >= 65274 && ((t - 65274) & (WSIZE - 1)) == 0 && t + 261 >= n) s++;
  return s;
}

// ---------------------------------------------------------------------------
// K3: previous position with the same 15-bit hash, as a distance (0 = none
// within 32767).  One warp per segment; a 64 KiB u16 head table in shared
// memory; positions are inserted in order, 32 at a time, with __match_any_sync
// resolving same-hash lanes inside the warp.
__device__ __forceinline__ void hp_load_tile(const uint8_t* src, uint64_t n, uint64_t c, int lane, uint32_t& w,
                                             uint32_t& x) {
  // lane holds bytes [c + 4 lane, c + 4 lane + 4); x = bytes [c + 128, c + 132).
  // Word-aligned tiles away from the end are single 32-bit loads whose values
  // are first used one tile later (so the prefetch really overlaps).
  const uint64_t a = c + 4 * (uint64_t)lane;
  if (((reinterpret_cast<uintptr_t>(src) + c) & 3) == 0 && c + 132 <= n) {
    w = __ldg(reinterpret_cast<const uint32_t*>(src + a));
    x = __ldg(reinterpret_cast<const uint32_t*>(src + c + 128));
    return;
  }
  w = 0;
#pragma unroll
  for (int t = 0; t < 4; t++)
    if (a + t < n) w |= (uint32_t)__ldg(src + a + t) << (8 * t);
  x = 0;
#pragma unroll
  for (int t = 0; t < 4; t++)
    if (c + 128 + t < n) x |= (uint32_t)__ldg(src + c + 128 + t) << (8 * t);
}

// K3 (two-phase warp scan): the segments are independent.
//   k_hash_prev6: one warp per 32 Ki-position segment scans it in order with an
//     empty 64 KiB u16 head table, 128 positions per tile (__match_any_sync
//     orders same-hash lanes), bytes prefetched HP6_D tiles ahead into registers
//     so the serial head-table chain does not also wait on DRAM; positions whose
//     hash has not yet been seen in the segment get 0xffff ("look in the
//     previous segment"), and the final table (last occurrence of every hash in
//     the segment) is stored.
//   k_hash_fix2: those positions read the previous segment's table.
// No history pass: each position is scanned once.  (Measured alternatives --
// one warp per 1024 positions with a block radix sort, a block-parallel scan with
// per-hash warp masks, a device-wide key sort -- were slower; see profiles/.)
#ifndef HP4_SEG_OVR
#define HP4_SEG_OVR 32768
#endif
constexpr uint32_t HP4_SEG = HP4_SEG_OVR;
// a position whose hash is new to its segment leaves HP_MARK | hash for k_hash_fix2 (in-segment
// distances are < 0x8000, so the marker is unambiguous and fix-up needs no byte reloads)
constexpr uint32_t HP_MARK = 0x8000u;
static_assert(HP4_SEG <= 32768, "distances within a segment must stay below HP_MARK");
constexpr int HP6_D = 8;

__device__ __forceinline__ uint32_t hp_hash_at(uint32_t w, uint32_t x, int k, int lane) {
  // hash bytes of tile position i = 32 k + lane: words j = i / 4 and j + 1 (x past the tile)
  const int j = 8 * k + (lane >> 2);
  const uint32_t a = __shfl_sync(0xffffffffu, w, j & 31);
  uint32_t b = __shfl_sync(0xffffffffu, w, (j + 1) & 31);
  if (j == 31) b = x;
  const uint32_t v = __funnelshift_r(a, b, 8 * (lane & 3));
  return (((v & 0xff) << 10) ^ (((v >> 8) & 0xff) << 5) ^ ((v >> 16) & 0xff)) & 0x7fff;
}

__global__ void __launch_bounds__(32) k_hash_prev6(const LaneDev* __restrict__ lanes,
                                                   const WorkItem* __restrict__ work, uint16_t* __restrict__ pd,
                                                   uint16_t* __restrict__ seg_heads) {
  extern __shared__ uint16_t hp6_head[];  // position - s + 1 (0 = none)
  const WorkItem w = work[blockIdx.x];
  const LaneDev L = lanes[w.lane];
  const uint64_t n = L.n;
  const uint64_t s = w.start;
  const uint64_t e = umin64(s + HP4_SEG, n);
  const int lane = threadIdx.x;
  uint16_t* head = hp6_head;
  uint4* h4 = reinterpret_cast<uint4*>(head);
  const uint8_t* src = L.src;
  uint16_t* out = pd + L.pbase;
  uint32_t cw[HP6_D], cx[HP6_D], nw[HP6_D], nx[HP6_D];
#pragma unroll
  for (int t = 0; t < HP6_D; t++) {
    const uint64_t c = s + 128ull * t;
    cw[t] = cx[t] = 0;
    if (c < e) hp_load_tile(src, n, c, lane, cw[t], cx[t]);
  }
  for (int i = lane; i < 32768 * 2 / 16; i += 32) h4[i] = make_uint4(0, 0, 0, 0);
  __syncwarp();
  for (uint64_t cs = s; cs < e; cs += 128ull * HP6_D) {
#pragma unroll
    for (int t = 0; t < HP6_D; t++) {
      const uint64_t c = cs + 128ull * (HP6_D + t);
      nw[t] = nx[t] = 0;
      if (c < e) hp_load_tile(src, n, c, lane, nw[t], nx[t]);
    }
#pragma unroll
    for (int t = 0; t < HP6_D; t++) {
      const uint64_t c = cs + 128ull * t;
      if (c >= e) break;
      uint32_t h[4];
      unsigned peers[4];
      bool valid[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint64_t q = c + 32 * k + lane;
        valid[k] = q < e && q + MIN_MATCH <= n;
        const uint32_t hh = hp_hash_at(cw[t], cx[t], k, lane);
        h[k] = valid[k] ? hh : 0x10000u + lane;
      }
#pragma unroll
      for (int k = 0; k < 4; k++) peers[k] = __match_any_sync(0xffffffffu, h[k]);
      uint32_t d[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint64_t q = c + 32 * k + lane;
        const unsigned lower = peers[k] & ((1u << lane) - 1);
        d[k] = 0;
        if (valid[k]) {
          if (lower) {
            d[k] = lane - (31 - __clz(lower));
          } else {
            const uint32_t r = head[h[k]];
            d[k] = r ? (uint32_t)(q - (s + r - 1)) : HP_MARK | h[k];  // resolve from the previous segment
          }
        }
        __syncwarp();
        if (valid[k] && (peers[k] >> lane) == 1u) head[h[k]] = (uint16_t)(q - s + 1);
        __syncwarp();
      }
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint64_t q = c + 32 * k + lane;
        if (q < e) out[q] = (uint16_t)d[k];
      }
    }
#pragma unroll
    for (int t = 0; t < HP6_D; t++) cw[t] = nw[t], cx[t] = nx[t];
  }
  __syncwarp();
  uint4* dst = reinterpret_cast<uint4*>(seg_heads + (uint64_t)blockIdx.x * 32768);
  for (int i = lane; i < 32768 * 2 / 16; i += 32) dst[i] = h4[i];
}

// K3 (current): k_hash_prev6's scan with HP7_W warps sharing one segment and
// its head table.  Warp w takes tiles w, w + HP7_W, ...: hashing, loads and the
// in-tile __match_any_sync groups of different tiles proceed in parallel, and
// only the head-table part of each tile (read heads, then store the tile's last
// occurrences) runs in tile order, handed from warp to warp by named barriers
// (the finishing warp arrives, the next one syncs).
#ifndef HP7_W_OVR
#define HP7_W_OVR 4
#endif
constexpr int HP7_W = HP7_W_OVR;

#ifndef HP7_TP
#define HP7_TP 4  // consecutive 128-position tiles per warp turn (one hand-over per turn)
#endif
__global__ void __launch_bounds__(32 * HP7_W) k_hash_prev7(const LaneDev* __restrict__ lanes,
                                                          const WorkItem* __restrict__ work,
                                                          uint16_t* __restrict__ pd,
                                                          uint16_t* __restrict__ seg_heads) {
  constexpr int TP = HP7_TP;
  extern __shared__ uint16_t hp7_head[];  // position - s + 1 (0 = none)
  const WorkItem w = work[blockIdx.x];
  const LaneDev L = lanes[w.lane];
  const uint64_t n = L.n;
  const uint64_t s = w.start;
  const uint64_t e = umin64(s + HP4_SEG, n);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint16_t* head = hp7_head;
  uint4* h4 = reinterpret_cast<uint4*>(head);
  const uint8_t* src = L.src;
  uint16_t* out = pd + L.pbase;
  for (int i = threadIdx.x; i < 32768 * 2 / 16; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
  const uint32_t ntiles = (uint32_t)((e - s + 127) / 128);
  uint32_t cw[TP], cx[TP];
#pragma unroll
  for (int u = 0; u < TP; u++) {
    cw[u] = cx[u] = 0;
    const uint32_t t = (uint32_t)wid * TP + u;
    if (t < ntiles) hp_load_tile(src, n, s + 128ull * t, lane, cw[u], cx[u]);
  }
  __syncthreads();
  for (uint32_t t0 = (uint32_t)wid * TP; t0 < ntiles; t0 += HP7_W * TP) {
    uint32_t nw[TP], nx[TP];
#pragma unroll
    for (int u = 0; u < TP; u++) {  // this warp's next turn
      nw[u] = nx[u] = 0;
      const uint32_t t = t0 + HP7_W * TP + u;
      if (t < ntiles) hp_load_tile(src, n, s + 128ull * t, lane, nw[u], nx[u]);
    }
    uint32_t h[TP][4];
    unsigned peers[TP][4];
    bool valid[TP][4];
#pragma unroll
    for (int u = 0; u < TP; u++) {
      const uint64_t c = s + 128ull * (t0 + u);
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint64_t q = c + 32 * k + lane;
        valid[u][k] = q < e && q + MIN_MATCH <= n;
        const uint32_t hh = hp_hash_at(cw[u], cx[u], k, lane);
        h[u][k] = valid[u][k] ? hh : 0x10000u + lane;
      }
#pragma unroll
      for (int k = 0; k < 4; k++) peers[u][k] = __match_any_sync(0xffffffffu, h[u][k]);
    }
    // wait for the previous turn's head updates (named barrier: its warp arrives, this one syncs)
    if (t0 > 0) asm volatile("bar.sync %0, 64;" ::"r"(1 + (wid + HP7_W - 1) % HP7_W) : "memory");
    uint32_t d[TP][4];
#pragma unroll
    for (int u = 0; u < TP; u++) {
      const uint64_t c = s + 128ull * (t0 + u);
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint64_t q = c + 32 * k + lane;
        const unsigned lower = peers[u][k] & ((1u << lane) - 1);
        d[u][k] = 0;
        if (valid[u][k]) {
          if (lower) {
            d[u][k] = lane - (31 - __clz(lower));
          } else {
            const uint32_t r = head[h[u][k]];
            d[u][k] = r ? (uint32_t)(q - (s + r - 1)) : HP_MARK | h[u][k];  // resolve from the previous segment
          }
        }
        __syncwarp();
        if (valid[u][k] && (peers[u][k] >> lane) == 1u) head[h[u][k]] = (uint16_t)(q - s + 1);
        __syncwarp();
      }
    }
    if (t0 + TP < ntiles) asm volatile("bar.arrive %0, 64;" ::"r"(1 + wid) : "memory");
#pragma unroll
    for (int u = 0; u < TP; u++) {
      const uint64_t c = s + 128ull * (t0 + u);
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint64_t q = c + 32 * k + lane;
        if (q < e) out[q] = (uint16_t)d[u][k];
      }
      cw[u] = nw[u], cx[u] = nx[u];
    }
  }
  __syncthreads();
  uint4* dst = reinterpret_cast<uint4*>(seg_heads + (uint64_t)blockIdx.x * 32768);
  for (int i = threadIdx.x; i < 32768 * 2 / 16; i += blockDim.x) dst[i] = h4[i];
}

// K3 (current): k_hash_prev7's warps and tile order, with each 128-position tile's
// same-hash structure found before the in-order phase instead of inside it.  A warp sorts
// its tile's (hash, index) keys (bitonic, four per lane); in sorted order a position's
// previous occurrence inside the tile is its left neighbour, the first occurrence of a hash
// reads the head table, the last one writes it.  The in-order phase is then only those
// loads and stores -- no data flows from the loads to the stores, so a tile's turn costs
// their issue, not k_hash_prev7's four load -> store -> __syncwarp rounds.
__device__ __forceinline__ void hp_sort128(uint32_t (&v)[4]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 128; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
#pragma unroll
        for (int r = 0; r < 4; r++) {
          const int rp = r ^ (j >> 5);
          if (rp > r) {
            const bool up = ((32 * r + lane) & k) == 0;
            const uint32_t a = v[r], b = v[rp];
            v[r] = up ? min(a, b) : max(a, b);
            v[rp] = up ? max(a, b) : min(a, b);
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < 4; r++) {
          const uint32_t o = __shfl_xor_sync(0xffffffffu, v[r], j);
          const bool up = ((32 * r + lane) & k) == 0;
          const bool lo = ((lane & j) == 0) == up;
          v[r] = lo ? min(v[r], o) : max(v[r], o);
        }
      }
    }
  }
}

#ifndef HP8_W_OVR
#define HP8_W_OVR 8  // sweep (config2 K3+fix ms): 8 4.39, 10 4.47, 12 4.37, 15 4.58; 15 with 2 tiles per turn 5.31
#endif
#ifndef HP8_TP
#define HP8_TP 1
#endif
constexpr int HP8_W = HP8_W_OVR;
static_assert(HP8_W <= 15, "named barriers 1 .. 15");
__global__ void __launch_bounds__(32 * HP8_W) k_hash_prev8(const LaneDev* __restrict__ lanes,
                                                          const WorkItem* __restrict__ work,
                                                          uint16_t* __restrict__ pd,
                                                          uint16_t* __restrict__ seg_heads) {
  constexpr int TP = HP8_TP;
  extern __shared__ uint16_t hp8_head[];  // position - s + 1 (0 = none)
  const WorkItem w = work[blockIdx.x];
  const LaneDev L = lanes[w.lane];
  const uint64_t n = L.n;
  const uint64_t s = w.start;
  const uint64_t e = umin64(s + HP4_SEG, n);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint16_t* head = hp8_head;
  uint4* h4 = reinterpret_cast<uint4*>(head);
  const uint8_t* src = L.src;
  uint16_t* out = pd + L.pbase + s;
  const uint32_t se = (uint32_t)(e - s);  // segment positions
  const uint32_t sv = (uint32_t)umin64(n - s, 1u << 30) >= 2 ? (uint32_t)umin64(n - s, 1u << 30) - 2 : 0;  // q - s < sv: 3 bytes of lookahead
  for (int i = threadIdx.x; i < 32768 * 2 / 16; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
  const uint32_t ntiles = (se + 127) / 128;
  uint32_t cw[TP], cx[TP];
#pragma unroll
  for (int u = 0; u < TP; u++) {
    cw[u] = cx[u] = 0;
    const uint32_t t = (uint32_t)wid * TP + u;
    if (t < ntiles) hp_load_tile(src, n, s + 128ull * t, lane, cw[u], cx[u]);
  }
  __syncthreads();
  for (uint32_t t0 = (uint32_t)wid * TP; t0 < ntiles; t0 += HP8_W * TP) {
    uint32_t nw[TP], nx[TP];
#pragma unroll
    for (int u = 0; u < TP; u++) {  // this warp's next turn
      nw[u] = nx[u] = 0;
      const uint32_t t = t0 + HP8_W * TP + u;
      if (t < ntiles) hp_load_tile(src, n, s + 128ull * t, lane, nw[u], nx[u]);
    }
    // per tile and sorted slot r: key = hash (16 bits; invalid positions get 0x8000 + index,
    // unique) << 7 | tile index; first / last occurrence flags; in-tile distance
    uint32_t key[TP][4], d[TP][4];
    unsigned fl[TP];  // bit r: first occurrence (reads the head), bit 4 + r: last (writes it)
#pragma unroll
    for (int u = 0; u < TP; u++) {
      const uint32_t c = 128u * (t0 + u);  // segment-relative tile start
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const uint32_t i = 32u * r + lane, q = c + i;
        const bool valid = q < se && q < sv;
        const uint32_t hh = hp_hash_at(cw[u], cx[u], r, lane);
        key[u][r] = ((valid ? hh : 0x8000u + i) << 7) | i;
      }
      hp_sort128(key[u]);
      fl[u] = 0;
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const uint32_t k = key[u][r];
        uint32_t left = __shfl_up_sync(0xffffffffu, k, 1);
        uint32_t right = __shfl_down_sync(0xffffffffu, k, 1);
        const uint32_t lprev = __shfl_sync(0xffffffffu, r > 0 ? key[u][r > 0 ? r - 1 : 0] : 0u, 31);
        const uint32_t rnext = __shfl_sync(0xffffffffu, r < 3 ? key[u][r < 3 ? r + 1 : 3] : 0u, 0);
        if (lane == 0) left = r > 0 ? lprev : 0xffffffffu;
        if (lane == 31) right = r < 3 ? rnext : 0xffffffffu;
        const bool real = (k >> 22) == 0;  // hash < 0x8000
        const bool first = real && (left >> 7) != (k >> 7);
        const bool last = real && (right >> 7) != (k >> 7);
        fl[u] |= (first ? 1u << r : 0u) | (last ? 16u << r : 0u);
        d[u][r] = real ? (first ? 0u : (k & 127) - (left & 127)) : 0u;
      }
    }
    // wait for the previous turn's head updates (named barrier: its warp arrives, this one syncs;
    // ids 1 .. HP8_W, so HP8_W <= 15)
    if (t0 > 0) asm volatile("bar.sync %0, 64;" ::"r"(1 + (wid + HP8_W - 1) % HP8_W) : "memory");
    uint32_t hv[TP][4];
#pragma unroll
    for (int u = 0; u < TP; u++) {
      const uint32_t c = 128u * (t0 + u);
#pragma unroll
      for (int r = 0; r < 4; r++) hv[u][r] = (fl[u] >> r) & 1 ? head[key[u][r] >> 7] : 0u;
      __syncwarp();  // the tile's loads see the table before its own stores
#pragma unroll
      for (int r = 0; r < 4; r++)
        if ((fl[u] >> (4 + r)) & 1) head[key[u][r] >> 7] = (uint16_t)(c + (key[u][r] & 127) + 1);
      __syncwarp();
    }
    if (t0 + TP < ntiles) asm volatile("bar.arrive %0, 64;" ::"r"(1 + wid) : "memory");
#pragma unroll
    for (int u = 0; u < TP; u++) {
      const uint32_t c = 128u * (t0 + u);
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const uint32_t q = c + (key[u][r] & 127);
        uint32_t dd = d[u][r];
        if ((fl[u] >> r) & 1) dd = hv[u][r] ? q + 1 - hv[u][r] : HP_MARK | (key[u][r] >> 7);  // the previous segment
        if (q < se) out[q] = (uint16_t)dd;
      }
      cw[u] = nw[u], cx[u] = nx[u];
    }
  }
  __syncthreads();
  uint4* dst = reinterpret_cast<uint4*>(seg_heads + (uint64_t)blockIdx.x * 32768);
  for (int i = threadIdx.x; i < 32768 * 2 / 16; i += blockDim.x) dst[i] = h4[i];
}

// k_hash_fix2: one CTA per segment, eight positions per thread and step
// (one 16-byte load of their links); only positions marked 0xffff compute their
// hash and read the previous segment's final head table.
__global__ void __launch_bounds__(256) k_hash_fix2(const LaneDev* __restrict__ lanes,
                                                   const WorkItem* __restrict__ work, uint16_t* __restrict__ pd,
                                                   const uint16_t* __restrict__ seg_heads) {
  const WorkItem w = work[blockIdx.x];
  const LaneDev L = lanes[w.lane];
  const uint64_t n = L.n;
  const uint64_t s = w.start;
  const uint64_t e = umin64(s + HP4_SEG, n);
  const bool first = s == 0;
  const uint16_t* prev = seg_heads + (uint64_t)(blockIdx.x - 1) * 32768;  // same lane's previous segment
  uint16_t* out = pd + L.pbase;
  const uint8_t* src = L.src;
  for (uint64_t q0 = s + 8 * threadIdx.x; q0 < e; q0 += 8 * 256) {
    uint16_t v[8];
    const bool vec = q0 + 8 <= e && ((reinterpret_cast<uintptr_t>(out + q0) & 15) == 0);
    if (vec) {
      *reinterpret_cast<uint4*>(v) = *reinterpret_cast<const uint4*>(out + q0);
    } else {
#pragma unroll
      for (int k = 0; k < 8; k++) v[k] = q0 + k < e ? out[q0 + k] : 0;
    }
    bool any = false;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      if (!(v[k] & HP_MARK)) continue;
      any = true;
      const uint64_t q = q0 + k;
      uint32_t d = 0;
      if (!first) {
        const uint32_t h = v[k] & 0x7fffu;  // the position's hash, carried in the marker
        const uint32_t r = prev[h];
        if (r) {
          const uint64_t dd = q - ((s - HP4_SEG) + r - 1);
          d = dd < WSIZE ? (uint32_t)dd : 0;
        }
      }
      v[k] = (uint16_t)d;
    }
    if (!any) continue;
    if (vec) {
      *reinterpret_cast<uint4*>(out + q0) = *reinterpret_cast<const uint4*>(v);
    } else {
#pragma unroll
      for (int k = 0; k < 8; k++)
        if (q0 + k < e) out[q0 + k] = v[k];
    }
  }
}

static int hash_prev_two_phase(Workspace& sortws, Workspace& W, const LaneDev* d_lanes, int nl,
                               const std::vector<uint64_t>& lane_prefix, uint16_t* d_pd, cudaStream_t st) {
  std::vector<WorkItem> work;
  std::vector<uint32_t> seg0(nl);
  for (int i = 0; i < nl; i++) {
    seg0[i] = (uint32_t)work.size();
    const uint64_t n = lane_prefix[i + 1] - lane_prefix[i];
    for (uint64_t s = 0; s < n; s += HP4_SEG) work.push_back(WorkItem{(uint32_t)i, (uint32_t)s});
  }
  if (work.empty()) return BB_OK;
  int rc = sortws.reserve(2ull * 32768 * work.size() + 4096);
  if (rc) return rc;
  uint16_t* heads = sortws.take<uint16_t>(32768ull * work.size());
  WorkItem* d_work = W.take<WorkItem>(work.size());
  uint32_t* d_seg0 = W.take<uint32_t>(nl);
  uint64_t* d_lp = W.take<uint64_t>(nl + 1);
  BB_CUDA_TRY(cudaMemcpyAsync(d_work, work.data(), sizeof(WorkItem) * work.size(), cudaMemcpyHostToDevice, st));
  BB_CUDA_TRY(cudaMemcpyAsync(d_seg0, seg0.data(), 4 * nl, cudaMemcpyHostToDevice, st));
  BB_CUDA_TRY(cudaMemcpyAsync(d_lp, lane_prefix.data(), 8 * (nl + 1), cudaMemcpyHostToDevice, st));
  static const bool k3_single = getenv("BB_K3_SINGLE_WARP") != nullptr;
  static const bool k3_v7 = getenv("BB_K3_V7") != nullptr;
  if (k3_single)
    k_hash_prev6<<<(unsigned)work.size(), 32, 65536, st>>>(d_lanes, d_work, d_pd, heads);
  else if (k3_v7)
    k_hash_prev7<<<(unsigned)work.size(), 32 * HP7_W, 65536, st>>>(d_lanes, d_work, d_pd, heads);
  else
    k_hash_prev8<<<(unsigned)work.size(), 32 * HP8_W, 65536, st>>>(d_lanes, d_work, d_pd, heads);
  BB_LAUNCH_CHECK();
  k_hash_fix2<<<(unsigned)work.size(), 256, 0, st>>>(d_lanes, d_work, d_pd, heads);
  BB_LAUNCH_CHECK();
  return BB_OK;
}

// ---------------------------------------------------------------------------
// K4: match profiles.  One CTA per PF_SEG positions; the 32 KiB history window,
// the segment and 258 bytes of lookahead are staged in shared memory together
// with the prev-distance links, so every chain step is two shared-memory loads.
__device__ __forceinline__ uint32_t prof_pack(uint32_t best, uint32_t bestd) {
  if (best < MIN_MATCH) return 0;
  if (best == MIN_MATCH && bestd > TOO_FAR) return 0;  // TOO_FAR
  return best | (bestd << 9);
}

// Shared-memory window word per position q: bits 0-15 prev-same-hash distance,
// bits 16-23 byte q, bits 24-31 byte q+1.  One 32-bit load yields a chain link
// and a byte pair, so a chain step costs two loads: the candidate's word (link
// + bytes 0,1) and the word at candidate + best_len - 1 (bytes best-1, best --
// zlib's scan_end1 / scan_end quick reject).
constexpr uint32_t PF_WIN = WSIZE + PF_SEG + MAX_MATCH + 32;

// K4 (current): first-maximum chain search with the passes of each lane
// batched.  Window word (shared memory, word 0 = a dead-end sentinel):
// (1-based window index of the previous same-hash position, 0 = none) | bytes
// (q, q+1) << 16.  A chain step is: the candidate's word, the candidate's bytes
// (best-1, best), one byte_perm compare against the lane's key, and the next
// link; a lane whose chain ends moves to the sentinel with a key that cannot
// match, so all 32 lanes step in lock-step without per-lane control flow.
// Candidates that pass the quick reject are only recorded (a bit per step of
// the batch); after every batch the lanes extend their recorded candidates in
// chain order, re-testing each against the best found so far.  best therefore
// lags by at most one batch during the walk: a candidate that fails the quick
// reject against the lagging best mismatches at or before it and cannot beat
// the final best either, so the result is exactly zlib's first maximum.
// c[t] for a run-time t: a binary select tree on the bits of t (B - 1 selects and
// log2 B bit tests instead of a compare per element)
template <int B>
__device__ __forceinline__ uint32_t pf_pick(const uint32_t (&c)[B], int t) {
  static_assert((B & (B - 1)) == 0, "power-of-two batch");
  uint32_t l[B];
#pragma unroll
  for (int k = 0; k < B; k++) l[k] = c[k];
#pragma unroll
  for (int w = 1; w < B; w <<= 1) {
    const bool bit = (t & w) != 0;
#pragma unroll
    for (int k = 0; k + w < B; k += 2 * w) l[k] = bit ? l[k + w] : l[k];
  }
  return l[0];
}

constexpr uint32_t PF_DEAD_KEY = 0xffffffffu;
#ifdef PF_STATS
__device__ unsigned long long g_pf_stats[4];  // flushes, recorded candidates, warp flush iterations, batches
#endif
#ifndef PF_B1
#define PF_B1 4  // chain steps per batch within the first 32 (budget-32 snapshot); 4 since the long
                 // chains went to K4G (classic lanes walk ~1-6 steps: config4 K4 44.0 vs 44.7 ms at 8)
#endif
#ifndef PF_B2
#define PF_B2 16  // chain steps per batch for candidates 33..128
#endif  // sentinel word is 0: its byte_perm low half never equals 0xffff

__global__ void __launch_bounds__(PF_THREADS, 1) k_profile3(const LaneDev* __restrict__ lanes,
                                                            const WorkItem* __restrict__ work,
                                                            const uint16_t* __restrict__ pd,
                                                            uint2* __restrict__ prof, int with_bytes) {
  extern __shared__ __align__(16) uint32_t w32[];
  const WorkItem w = work[blockIdx.x];
  const LaneDev L = lanes[w.lane];
  const uint64_t n = L.n;
  const uint64_t s = w.start;
  const uint64_t e = umin64(s + PF_SEG, n);
  const uint64_t wlo = s > WSIZE ? s - WSIZE : 0;
  const uint32_t wlen = (uint32_t)(e - wlo) + MAX_MATCH + 16;  // <= PF_WIN
  const uint8_t* src = L.src;
  const uint16_t* pdl = pd + L.pbase;
  if (threadIdx.x == 0) w32[0] = 0;
  {
    // four window positions per thread: one 8-byte load of their links, two 4-byte
    // loads of their bytes (wlo, the lane bases and the link array are 4-aligned)
    const bool aligned = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(pdl)) & 7) == 0;
    const uint32_t nq = (wlen + 3) / 4;
    // groups j < jf take the vector path (q0 + 4 <= e, q0 + 8 <= n); their loads are
    // issued PF_STAGE_U groups at a time so several L2 round trips are in flight
    uint32_t jf = 0;
    if (aligned) {
      const uint64_t lim = umin64(e >= 4 ? e - 4 : 0, n >= 8 ? n - 8 : 0);
      jf = lim >= wlo ? (uint32_t)umin64((lim - wlo) / 4 + 1, nq) : 0;
    }
    constexpr int U = 4;
    for (uint32_t j0 = threadIdx.x; j0 < jf; j0 += U * blockDim.x) {
      uint2 l4[U];
      uint32_t b0[U], b1[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const uint32_t j = j0 + u * blockDim.x;
        if (j < jf) {
          const uint64_t q0 = wlo + 4 * j;
          l4[u] = __ldg(reinterpret_cast<const uint2*>(pdl + q0));
          b0[u] = __ldg(reinterpret_cast<const uint32_t*>(src + q0));
          b1[u] = __ldg(reinterpret_cast<const uint32_t*>(src + q0 + 4));
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const uint32_t j = j0 + u * blockDim.x;
        if (j < jf) {
          const uint32_t i0 = 4 * j;
          const uint32_t ls[4] = {l4[u].x & 0xffff, l4[u].x >> 16, l4[u].y & 0xffff, l4[u].y >> 16};
          uint32_t v[4];
#pragma unroll
          for (int k = 0; k < 4; k++) {
            const uint32_t i = i0 + k, l = ls[k];
            v[k] = (l && l <= i) ? i - l + 1 : 0;                                 // 1-based predecessor index
            v[k] |= __byte_perm(b0[u], b1[u], (k | ((k + 1) << 4)) & 0xff) << 16;  // bytes q, q + 1
          }
#pragma unroll
          for (int k = 0; k < 4; k++) w32[i0 + k + 1] = v[k];
        }
      }
    }
    for (uint32_t j = jf + threadIdx.x; j < nq; j += blockDim.x) {
      const uint32_t i0 = 4 * j;
      for (uint32_t i = i0; i < i0 + 4 && i < wlen; i++) {
        const uint64_t q = wlo + i;
        uint32_t v = 0;
        if (q < e) {
          const uint32_t l = pdl[q];
          if (l && l <= i) v = i - l + 1;
        }
        if (q < n) v |= (uint32_t)__ldg(src + q) << 16;
        if (q + 1 < n) v |= (uint32_t)__ldg(src + q + 1) << 24;
        w32[i + 1] = v;
      }
    }
  }
  __syncthreads();
  const uint32_t sw = (uint32_t)__cvta_generic_to_shared(w32);

  // positions as 1-based window indices (32-bit): ip1 = p - wlo + 1
  const uint32_t nrel = (uint32_t)umin64(n - wlo, 1u << 30);
  const uint32_t ie = (uint32_t)(e - wlo) + 1;  // ip1 < ie: p < e
  const uint32_t ix0 = wlo == 0 ? 1u : 0u;     // the index of absolute position 0 (NIL), if in the window
  uint2* profw = prof + L.pbase + wlo - 1;
  for (uint32_t i0 = (uint32_t)(s - wlo) + 1; i0 < ie; i0 += blockDim.x) {
    const uint32_t ip1 = i0 + threadIdx.x;
    const bool inb = ip1 < ie;
    const uint32_t wp = inb ? w32[ip1] : 0;
    const uint32_t c0 = wp & 0xffff;
    const uint32_t d0 = ip1 - c0;
    const bool live = inb && ip1 + 2 <= nrel && c0 != 0 && d0 <= MAX_DIST && c0 != ix0;
    uint32_t best = MIN_MATCH - 1, bestd = 0, flag = 0, nice = 0, maxl = 0, lim1 = 0;
    // ic4: 4 x the candidate's 1-based window index (byte offset of its word)
    uint32_t ic4 = 0, key = PF_DEAD_KEY, offb = sw + 4 * (MIN_MATCH - 2) + 2;
    if (live) {
      const uint32_t la = min(nrel - ip1 + 1, 1u << 20);
      nice = min(NICE_LENGTH, la);
      maxl = min(MAX_MATCH, la);
      lim1 = (uint32_t)max((int)ip1 - (int)MAX_DIST, 1);
      flag = d0 == MAX_DIST ? PROF_AT_MAXDIST : 0;
      ic4 = 4 * c0;
      key = (wp >> 16) | (w32[ip1 + best - 1] & 0xffff0000u);
    }
    // zlib tests the limit only from the second candidate on (do ... while (prev > limit)):
    // a head exactly at MAX_DIST is still compared, and every later candidate is below it
    const uint32_t lim4 = 4 * lim1 - (live && c0 == lim1 ? 4u : 0u);
    const uint32_t qw2 = inb ? w32[ip1 + 2] : 0u;  // bytes p + 2, p + 3 (wlen covers e + 274)
#ifdef PF_HEAD_SEED  // off since the long chains went to K4G: config4 K4 43.6 vs 44.7 ms, config2 2.37 vs 2.43
    // The head candidate (chain step 1) is extended exactly before the walk, so best starts at its
    // length: the batches' quick test then records only candidates that can beat it (with best = 2,
    // every same-3-gram candidate of the first batch was recorded and extended in the flush).  The
    // head is first in chain order, so seeding best with it leaves the first maximum unchanged; its
    // own step in the first batch fails the quick test (its byte `best` mismatches) or re-tests to no
    // change.
    if (live && ((w32[c0] ^ wp) & 0xffff0000u) == 0) {
      uint32_t len = 2;
      const uint32_t x2 = (w32[c0 + 2] ^ qw2) >> 16;
      if (x2) {
        len += (x2 & 0xff) == 0;
      } else {
        len = 4;
        while (len < maxl) {
          const uint32_t x = (w32[c0 + len] ^ w32[ip1 + len]) >> 16;
          if (x) {
            len += (x & 0xff) == 0;
            break;
          }
          len += 2;
        }
      }
      len = min(len, maxl);
      if (len > best) {
        best = len;
        bestd = d0;
        offb = sw + 4 * (best - 1) + 2;
        key = (wp >> 16) | (w32[ip1 + best - 1] & 0xffff0000u);
        if (len >= nice) ic4 = 0;  // zlib stops at nice_match: the lane walks the dead sentinel
      }
    }
#endif
    // one batch of B chain steps, then the recorded candidates in chain order
    auto batch = [&](auto bsize) {
      constexpr int B = decltype(bsize)::value;
      uint32_t cand[B];
      uint32_t mask = 0;
#pragma unroll
      for (int t = 0; t < B; t++) {
        // past the distance limit (or at the sentinel, which links to itself) a
        // candidate is walked but never recorded: chains only go backwards
        uint32_t wc, we;  // the candidate's word; bytes (best - 1, best) of the candidate
        asm("ld.shared.u32 %0, [%1];" : "=r"(wc) : "r"(sw + ic4));
#ifdef PF_COND_LD2
        // variant: the scan_end pair fetched only for candidates whose bytes 0, 1 match (hash
        // collisions and dead lanes issue no second load).  Measured slower: 39.7 vs 35.0 ms
        asm("{\n\t.reg .pred q;\n\tsetp.eq.u32 q, %2, %3;\n\tmov.u32 %0, 0xffffffff;\n\t"
            "@q ld.shared.u16 %0, [%1];\n\t}"
            : "=r"(we) : "r"(ic4 + offb), "r"(wc >> 16), "r"(key & 0xffffu));
        cand[t] = ic4;
        mask |= ((we == key >> 16) && (wc >> 16) == (key & 0xffffu) && ic4 > lim4) ? 1u << t : 0u;
#else
        asm("ld.shared.u16 %0, [%1];" : "=r"(we) : "r"(ic4 + offb));
        cand[t] = ic4;
        mask |= (__byte_perm(wc, we, 0x5432) == key && ic4 > lim4) ? 1u << t : 0u;
#endif
        ic4 = (wc << 2) & 0x3fffc;
      }
      if (__any_sync(0xffffffffu, mask != 0)) {
#ifdef PF_STATS
        {
          const uint32_t rec = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(mask));
          const uint32_t mx = __reduce_max_sync(0xffffffffu, (uint32_t)__popc(mask));
          if ((threadIdx.x & 31) == 0) {
            atomicAdd(&g_pf_stats[0], 1ull);                      // flushes
            atomicAdd(&g_pf_stats[1], (unsigned long long)rec);   // recorded candidates
            atomicAdd(&g_pf_stats[2], (unsigned long long)mx);    // warp iterations (max popc)
          }
        }
#endif
        bool improved = false;
        while (mask) {
          const int t = __ffs(mask) - 1;
          mask &= mask - 1;
          const uint32_t c = pf_pick(cand, t) >> 2;
          // re-test only if best grew in this flush (else it is the test the step already made)
          if (improved && (((w32[c] ^ wp) | (w32[c + best - 1] ^ w32[ip1 + best - 1])) & 0xffff0000u) != 0)
            continue;
          // bytes 2, 3 against the position's own pair held in a register (most matches end there)
          uint32_t len = 2;
          const uint32_t x2 = (w32[c + 2] ^ qw2) >> 16;
          if (x2) {
            len += (x2 & 0xff) == 0;
          } else {
            len = 4;
            while (len < maxl) {
              const uint32_t x = (w32[c + len] ^ w32[ip1 + len]) >> 16;
              if (x) {
                len += (x & 0xff) == 0;
                break;
              }
              len += 2;
            }
          }
          len = min(len, maxl);
          if (len > best) {
            best = len;
            bestd = ip1 - c;
            improved = true;
            if (len >= nice) {
              mask = 0;
              ic4 = 0;
            }
          }
        }
        if (improved) {
          offb = sw + 4 * (best - 1) + 2;
          key = (wp >> 16) | (w32[ip1 + best - 1] & 0xffff0000u);
        }
      }
    };
    for (int cnt = 0; cnt < 32; cnt += PF_B1) {
      if (!__any_sync(0xffffffffu, ic4 > lim4)) break;
#ifdef PF_STATS
      if ((threadIdx.x & 31) == 0) atomicAdd(&g_pf_stats[3], 1ull);
#endif
      batch(std::integral_constant<int, PF_B1>());
    }
    const uint32_t r32 = prof_pack(best, bestd);  // budget 32 (prev_length >= good_length)
    for (int cnt = 32; cnt < (int)MAX_CHAIN; cnt += PF_B2) {
      if (!__any_sync(0xffffffffu, ic4 > lim4)) break;
#ifdef PF_STATS
      if ((threadIdx.x & 31) == 0) atomicAdd(&g_pf_stats[3], 1ull);
#endif
      batch(std::integral_constant<int, PF_B2>());
    }
    if (inb) {
      // y: the 32-chain profile (the flag lives in x) | the byte before p << 24 for the parse
      const uint32_t yb = with_bytes ? (w32[ip1 - 1] << 8) & 0xff000000u : (live ? flag : 0u);
      profw[ip1] = make_uint2(live ? prof_pack(best, bestd) | flag : 0, (live ? r32 : 0u) | yb);
    }
  }
}

// ---------------------------------------------------------------------------
// K4G (default): the chain walk restricted to the candidates that can matter.
//
// longest_match() returns the first candidate of maximal length among the first B
// (32 or 128) entries of p's hash chain.  A candidate can replace best only if its
// match is longer, i.e. it shares p's first best + 1 bytes; once best >= 3 every
// such candidate shares p's 4-gram.  And two positions with the same 4-gram have
// the same hash, so the same-4-gram positions before p form a subsequence of p's
// chain, and for any candidate c on it the rest of that subsequence is c's own.
// K4G therefore splits the walk in two exact passes:
//
//   k_gram4     per position x, walking x's zlib chain (K3 links): the first
//               candidate sharing x's 3-gram and the first sharing its 4-gram, each
//               with its chain step number (budget 128, the MAX_DIST rules of the
//               head and of later entries).  On bf16 exponent planes ~17 steps
//               instead of ~108.
//   k_profile4  per position p: the first same-3-gram candidate (the only one that
//               matters while best < 4, i.e. a match of exactly 3), then the
//               same-4-gram subsequence, hopping link to link and adding the step
//               counts so the budget (32 snapshot, 128) and the distance limit are
//               applied exactly as the full walk applies them; quick reject on bytes
//               (best - 1, best), extension, nice_match, first maximum.  ~11 hops.
//
// Profiles are bit-identical to K4's (tests compare both with the oracle's
// orc_match_profile and the full-size goldens).
//
// g3[x]: d3 (15 bits, 0 = none) | s3 << 15 (8 bits) | head-at-MAX_DIST << 23 | live << 24
// g4[x]: d4 (15 bits, 0 = none) | s4 << 15 (8 bits)
constexpr uint32_t G3_FLAG = 1u << 23, G3_LIVE = 1u << 24;
constexpr uint32_t PF2_SEG = 12288;  // k_profile4 positions per CTA
constexpr uint32_t PF2_WIN = WSIZE + PF2_SEG + MAX_MATCH + 32;
constexpr uint32_t PF2_SMEM = 5 * PF2_WIN;  // u32 words (link4 index | bytes q, q+1) + u8 step counts

// K4's window staging: w32[i + 1] = 1-based index of the previous same-hash position
// (0 = none) | bytes (q, q+1) << 16 for window position q = wlo + i
__device__ __forceinline__ void pf_stage_links(uint32_t* w32, const uint8_t* src, const uint16_t* pdl, uint64_t n,
                                               uint64_t wlo, uint64_t e, uint32_t wlen) {
  if (threadIdx.x == 0) w32[0] = 0;
  const bool aligned = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(pdl)) & 7) == 0;
  const uint32_t nq = (wlen + 3) / 4;
  uint32_t jf = 0;
  if (aligned) {
    const uint64_t lim = umin64(e >= 4 ? e - 4 : 0, n >= 8 ? n - 8 : 0);
    jf = lim >= wlo ? (uint32_t)umin64((lim - wlo) / 4 + 1, nq) : 0;
  }
  constexpr int U = 4;
  for (uint32_t j0 = threadIdx.x; j0 < jf; j0 += U * blockDim.x) {
    uint2 l4[U];
    uint32_t b0[U], b1[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t j = j0 + u * blockDim.x;
      if (j < jf) {
        const uint64_t q0 = wlo + 4 * j;
        l4[u] = __ldg(reinterpret_cast<const uint2*>(pdl + q0));
        b0[u] = __ldg(reinterpret_cast<const uint32_t*>(src + q0));
        b1[u] = __ldg(reinterpret_cast<const uint32_t*>(src + q0 + 4));
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t j = j0 + u * blockDim.x;
      if (j < jf) {
        const uint32_t i0 = 4 * j;
        const uint32_t ls[4] = {l4[u].x & 0xffff, l4[u].x >> 16, l4[u].y & 0xffff, l4[u].y >> 16};
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const uint32_t i = i0 + k, l = ls[k];
          uint32_t v = (l && l <= i) ? i - l + 1 : 0;
          v |= __byte_perm(b0[u], b1[u], (k | ((k + 1) << 4)) & 0xff) << 16;
          w32[i + 1] = v;
        }
      }
    }
  }
  for (uint32_t j = jf + threadIdx.x; j < nq; j += blockDim.x) {
    const uint32_t i0 = 4 * j;
    for (uint32_t i = i0; i < i0 + 4 && i < wlen; i++) {
      const uint64_t q = wlo + i;
      uint32_t v = 0;
      if (q < e) {
        const uint32_t l = pdl[q];
        if (l && l <= i) v = i - l + 1;
      }
      if (q < n) v |= (uint32_t)__ldg(src + q) << 16;
      if (q + 1 < n) v |= (uint32_t)__ldg(src + q + 1) << 24;
      w32[i + 1] = v;
    }
  }
}

// Lock-step batches with refill: each warp owns a contiguous run of positions; a lane
// walks one position's chain, GB steps per batch, and lanes whose walk ended take the
// warp's next positions at the batch boundary (ballot + rank), so the walks' different
// lengths cost at most one partial batch each instead of diverging the whole warp.
#ifndef GB_STEPS
#define GB_STEPS 8
#endif
#ifndef PB_STEPS
#define PB_STEPS 8
#endif
__device__ __forceinline__ void warp_range(uint64_t s, uint64_t e, uint64_t& qn, uint64_t& qe) {
  const uint32_t nw = blockDim.x >> 5, wid = threadIdx.x >> 5;
  const uint64_t per = (e - s + nw - 1) / nw;
  qn = umin64(s + wid * per, e);
  qe = umin64(qn + per, e);
}

// k_gram4's window word for position q: the K3 link as a distance (15 bits; 0x7fff =
// none, outside the window, or beyond MAX_DIST -- any of them ends the walk through the
// distance limit) | z(q) << 15 | byte q+3 << 24, where z(q) = the top three bits of
// bytes q, q+1, q+2.  zlib's 15-bit hash ((b0 << 10) ^ (b1 << 5) ^ b2) keeps everything
// of a 3-gram but those nine bits, and every entry of q's chain has q's hash, so along a
// chain "same 3-gram" is "same z" and "same 4-gram" is "same z and byte 3": one load and
// two masked compares per chain step instead of two loads and a byte permute.
constexpr uint32_t GZ_NONE = 0x7fffu, GZ_Z = 0x00ff8000u, GZ_Z4 = 0xffff8000u;
__device__ __forceinline__ uint32_t gz_word(uint32_t l, uint32_t i, uint32_t b) {  // b: bytes q .. q+3
  const uint32_t d = (l && l <= i && l <= MAX_DIST) ? l : GZ_NONE;
  const uint32_t z = ((b >> 5) & 7u) | ((b >> 10) & 0x38u) | ((b >> 15) & 0x1c0u);
  return d | (z << 15) | (b & 0xff000000u);
}
__device__ __forceinline__ void gz_stage(uint32_t* w32, const uint8_t* src, const uint16_t* pdl, uint64_t n,
                                         uint64_t wlo, uint64_t e) {
  if (threadIdx.x == 0) w32[0] = 0;
  const uint32_t wlen = (uint32_t)(e - wlo);
  const bool aligned = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(pdl)) & 7) == 0;
  const uint32_t nq = (wlen + 3) / 4;
  uint32_t jf = 0;
  if (aligned) {
    const uint64_t lim = umin64(e >= 4 ? e - 4 : 0, n >= 8 ? n - 8 : 0);
    jf = lim >= wlo ? (uint32_t)umin64((lim - wlo) / 4 + 1, nq) : 0;
  }
  constexpr int U = 4;
  for (uint32_t j0 = threadIdx.x; j0 < jf; j0 += U * blockDim.x) {
    uint2 l4[U];
    uint32_t b0[U], b1[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t j = j0 + u * blockDim.x;
      if (j < jf) {
        const uint64_t q0 = wlo + 4 * j;
        l4[u] = __ldg(reinterpret_cast<const uint2*>(pdl + q0));
        b0[u] = __ldg(reinterpret_cast<const uint32_t*>(src + q0));
        b1[u] = __ldg(reinterpret_cast<const uint32_t*>(src + q0 + 4));
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t j = j0 + u * blockDim.x;
      if (j < jf) {
        const uint32_t i0 = 4 * j;
        const uint32_t ls[4] = {l4[u].x & 0xffff, l4[u].x >> 16, l4[u].y & 0xffff, l4[u].y >> 16};
        uint4 v;
        v.x = gz_word(ls[0], i0 + 0, b0[u]);
        v.y = gz_word(ls[1], i0 + 1, __byte_perm(b0[u], b1[u], 0x4321));
        v.z = gz_word(ls[2], i0 + 2, __byte_perm(b0[u], b1[u], 0x5432));
        v.w = gz_word(ls[3], i0 + 3, __byte_perm(b0[u], b1[u], 0x6543));
        w32[i0 + 1] = v.x, w32[i0 + 2] = v.y, w32[i0 + 3] = v.z, w32[i0 + 4] = v.w;
      }
    }
  }
  for (uint32_t i = 4 * jf + threadIdx.x; i < wlen; i += blockDim.x) {
    const uint64_t q = wlo + i;
    uint32_t b = 0;
#pragma unroll
    for (int k = 0; k < 4; k++)
      if (q + k < n) b |= (uint32_t)__ldg(src + q + k) << (8 * k);
    w32[i + 1] = gz_word(pdl[q], i, b);
  }
}

__global__ void __launch_bounds__(PF_THREADS, 1) k_gram4(const LaneDev* __restrict__ lanes,
                                                         const WorkItem* __restrict__ work,
                                                         const uint16_t* __restrict__ pd, uint32_t* __restrict__ g3,
                                                         uint32_t* __restrict__ g4) {
  extern __shared__ __align__(16) uint32_t w32[];
  const WorkItem w = work[blockIdx.x];
  const LaneDev L = lanes[w.lane];
  const uint64_t n = L.n;
  const uint64_t s = w.start;
  const uint64_t e = umin64(s + PF_SEG, n);
  const uint64_t wlo = s > WSIZE ? s - WSIZE : 0;
  gz_stage(w32, L.src, pd + L.pbase, n, wlo, e);
  __syncthreads();
  // positions as 1-based window indices (32-bit): ix = p - wlo + 1
  uint32_t* G3 = g3 + L.pbase + wlo - 1;
  uint32_t* G4 = g4 + L.pbase + wlo - 1;
  const uint32_t nrel = (uint32_t)umin64(n - wlo, 1u << 30);  // n as a window index bound
  const uint32_t ix0 = wlo == 0 ? 1u : 0u;                     // absolute position 0 (NIL), if in the window
  const unsigned lt = (1u << (threadIdx.x & 31)) - 1;
  uint32_t qn, qe;
  {
    uint64_t a, b;
    warp_range(s, e, a, b);
    qn = (uint32_t)(a - wlo) + 1, qe = (uint32_t)(b - wlo) + 1;
  }
  const int sw = (int)__cvta_generic_to_shared(w32);
  bool has = false, done = true, four = false;
  // lane state: cb = shared byte address of the current candidate's word; a lane without a
  // walk sits on the sentinel word 0 with done set
  uint32_t ix = 0, key = 0, stp = 0, f3s = 0, hd = 0;
  int cb = sw, limb = sw, f3c = 0;
  for (;;) {
    // refill (once per batch): idle lanes take the warp's next positions in order
    const unsigned need = __ballot_sync(0xffffffffu, !has);
    if (need && qn < qe) {
      const uint32_t myp = qn + __popc(need & lt);
      qn = min(qn + __popc(need), qe);
      if (!has && myp < qe) {
        ix = myp;
        const uint32_t wp = w32[ix];
        const uint32_t d0 = wp & GZ_NONE;
        // zlib: the head must be within MAX_DIST and not absolute position 0 (NIL)
        if (ix + 2 <= nrel && d0 != GZ_NONE && ix - d0 != ix0) {
          limb = sw + 4 * max((int)ix - (int)MAX_DIST, 1);
          hd = G3_LIVE | (d0 == MAX_DIST ? G3_FLAG : 0u);
          four = ix + 3 <= nrel;
          key = wp & GZ_Z4;
          cb = sw + 4 * (int)(ix - d0);
          stp = 1;
          f3s = 0;
          has = true;
          done = false;
        } else {
          G3[ix] = 0;
          G4[ix] = 0;
        }
      }
    }
    if (!__any_sync(0xffffffffu, has)) {
      if (qn >= qe) break;
      continue;
    }
    // GB chain steps, branch-free; a lane whose walk ended stays on its last candidate
#pragma unroll
    for (int t = 0; t < GB_STEPS; t++) {
      uint32_t wc;
      asm("ld.shared.u32 %0, [%1];" : "=r"(wc) : "r"(cb));
      const uint32_t x = wc ^ key;
      const bool h3 = !done && (x & GZ_Z) == 0;
      const bool first3 = h3 && f3s == 0;
      f3c = first3 ? cb : f3c;
      f3s = first3 ? stp : f3s;
      const bool h4 = h3 && (x & GZ_Z4) == 0;
      const int nb = cb - 4 * (int)(wc & GZ_NONE);  // entries after the head must lie above the limit
      const bool end = h4 || stp >= MAX_CHAIN || nb <= limb;
      const bool adv = !done && !end;
      done = done || end;
      cb = adv ? nb : cb;
      stp = adv ? stp + 1 : stp;
    }
    if (has && done) {
      // the walk ended on a same-4-gram candidate iff the candidate it stopped on is one
      const uint32_t c4 = (uint32_t)(cb - sw) >> 2;
      const bool found4 = four && ((w32[c4] ^ key) & GZ_Z4) == 0;
      G3[ix] = f3s ? (ix - ((uint32_t)(f3c - sw) >> 2)) | (f3s << 15) | hd : hd;
      G4[ix] = found4 ? (ix - c4) | (stp << 15) : 0u;
      has = false;
    }
  }
}

// K4G second pass: one CTA per PF2_SEG positions.  Window word: 1-based index of the
// previous same-4-gram position (0 = none or outside the window) | bytes (q, q+1) << 16,
// plus the zlib step count of that hop in a byte array behind the words.  A lane's
// candidates are the first same-3-gram one, then the 4-gram hops.  As in K4, a batch of
// PB_STEPS candidates is walked branch-free and only records which pass the quick test
// (bytes best - 1, best against a best that may lag by one batch); the recorded ones
// are then extended in chain order.  Lanes refill at batch boundaries.
__global__ void __launch_bounds__(PF_THREADS, 1) k_profile4(const LaneDev* __restrict__ lanes,
                                                            const WorkItem* __restrict__ work,
                                                            const uint32_t* __restrict__ g3,
                                                            const uint32_t* __restrict__ g4, uint2* __restrict__ prof,
                                                            int with_bytes) {
  extern __shared__ __align__(16) uint32_t w32[];
  const WorkItem w = work[blockIdx.x];
  const LaneDev L = lanes[w.lane];
  const uint64_t n = L.n;
  const uint64_t s = w.start;
  const uint64_t e = umin64(s + PF2_SEG, n);
  const uint64_t wlo = s > WSIZE ? s - WSIZE : 0;
  const uint32_t wlen = (uint32_t)(e - wlo) + MAX_MATCH + 16;  // <= PF2_WIN - 1
  uint8_t* sk = reinterpret_cast<uint8_t*>(w32 + PF2_WIN);
  const uint8_t* src = L.src;
  const uint32_t* G4 = g4 + L.pbase;
  const uint32_t* G3 = g3 + L.pbase;
  if (threadIdx.x == 0) w32[0] = 0, sk[0] = 0;
  {
    // four window positions per thread and step: one 16-byte load of their g4 records, two
    // 4-byte loads of their bytes (wlo, the lane bases and the arrays are 4-aligned)
    const bool aligned = ((reinterpret_cast<uintptr_t>(src) & 3) | (reinterpret_cast<uintptr_t>(G4) & 15)) == 0;
    const uint32_t nq = (wlen + 3) / 4;
    uint32_t jf = 0;
    if (aligned) {
      const uint64_t lim = umin64(e >= 4 ? e - 4 : 0, n >= 8 ? n - 8 : 0);
      jf = lim >= wlo ? (uint32_t)umin64((lim - wlo) / 4 + 1, nq) : 0;
    }
    constexpr int U = 4;
    for (uint32_t j0 = threadIdx.x; j0 < jf; j0 += U * blockDim.x) {
      uint4 gv[U];
      uint32_t b0[U], b1[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const uint32_t j = j0 + u * blockDim.x;
        if (j < jf) {
          const uint64_t q0 = wlo + 4 * j;
          gv[u] = __ldg(reinterpret_cast<const uint4*>(G4 + q0));
          b0[u] = __ldg(reinterpret_cast<const uint32_t*>(src + q0));
          b1[u] = __ldg(reinterpret_cast<const uint32_t*>(src + q0 + 4));
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const uint32_t j = j0 + u * blockDim.x;
        if (j < jf) {
          const uint32_t i0 = 4 * j;
          const uint32_t gs[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
          uint32_t kk = 0;
#pragma unroll
          for (int k = 0; k < 4; k++) {
            const uint32_t i = i0 + k, g = gs[k], d = g & 0x7fff;
            const bool in = d && d <= i;
            w32[i + 1] = (in ? i - d + 1 : 0u) | (__byte_perm(b0[u], b1[u], (k | ((k + 1) << 4)) & 0xff) << 16);
            kk |= (in ? g >> 15 : 0u) << (8 * k);
          }
          // bytes i0 + 1 .. i0 + 4 of sk: two aligned 16-bit stores are not possible at odd
          // offsets, so four byte stores
#pragma unroll
          for (int k = 0; k < 4; k++) sk[i0 + k + 1] = (uint8_t)(kk >> (8 * k));
        }
      }
    }
    for (uint32_t j = jf + threadIdx.x; j < nq; j += blockDim.x) {
      for (uint32_t i = 4 * j; i < 4 * j + 4 && i < wlen; i++) {
        const uint64_t q = wlo + i;
        uint32_t v = 0, k = 0;
        if (q < e) {
          const uint32_t g = __ldg(G4 + q), d = g & 0x7fff;
          if (d && d <= i) v = i - d + 1, k = g >> 15;
        }
        if (q < n) v |= (uint32_t)__ldg(src + q) << 16;
        if (q + 1 < n) v |= (uint32_t)__ldg(src + q + 1) << 24;
        w32[i + 1] = v;
        sk[i + 1] = (uint8_t)k;
      }
    }
  }
  __syncthreads();
  const uint32_t sw = (uint32_t)__cvta_generic_to_shared(w32);
  const uint32_t skb = sw + 4 * PF2_WIN;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1;
  // positions as 1-based window indices (32-bit): ip1 = p - wlo + 1
  const uint32_t* G3w = G3 + wlo - 1;
  uint2* profw = prof + L.pbase + wlo - 1;
  const uint32_t nrel = (uint32_t)umin64(n - wlo, 1u << 30);
  uint32_t qn, qe;
  {
    uint64_t a, b;
    warp_range(s, e, a, b);
    qn = (uint32_t)(a - wlo) + 1, qe = (uint32_t)(b - wlo) + 1;
  }
  // the warp's next 32 positions' g3 records, one per lane, loaded a batch ahead
  uint32_t gbuf = qn + lane < qe ? __ldg(G3w + qn + lane) : 0u;
  bool has = false, done = true, snap = false;
  uint32_t ip1 = 0, maxl = 0, nice = 0, lim1 = 0, flag = 0, best = MIN_MATCH - 1, bestd = 0, r32 = 0;
  uint32_t key = 0;  // bytes (best - 1, best) of p (best >= 4 while a lane walks)
  uint32_t c = 0, stp = 0;
  auto store = [&](bool live) {
    const uint32_t yb = with_bytes ? (w32[ip1 - 1] << 8) & 0xff000000u : (live ? flag : 0u);
    if (live && !snap) r32 = prof_pack(best, bestd);
    profw[ip1] = make_uint2(live ? prof_pack(best, bestd) | flag : 0, (live ? r32 : 0u) | yb);
  };
  // a walking lane has best >= 4 (its first same-4-gram candidate matched), so neither
  // of prof_pack's "no match" rules can apply
  auto store_walked = [&]() {
    const uint32_t pk = best | (bestd << 9);
    const uint32_t yb = with_bytes ? (w32[ip1 - 1] << 8) & 0xff000000u : flag;
    profw[ip1] = make_uint2(pk | flag, (snap ? r32 : pk) | yb);
  };
  // match length of candidate cx whose first `from` (>= 4) bytes are known to match p's
  auto extend = [&](uint32_t cx, uint32_t from) {
    uint32_t len = from;
    while (len < maxl) {
      const uint32_t x = (w32[cx + len] ^ w32[ip1 + len]) >> 16;
      if (x) {
        len += (x & 0xff) == 0;
        break;
      }
      len += 2;
    }
    return min(len, maxl);
  };
  for (;;) {
    const unsigned need = __ballot_sync(0xffffffffu, !has);
    if (need && qn < qe) {
      const uint32_t cnt = __popc(need), r = __popc(need & lt);
      const uint32_t gg = __shfl_sync(0xffffffffu, gbuf, r & 31);
      const uint32_t myp = qn + r;
      // the buffer moves on by cnt positions; the lanes past its end load new records
      const uint32_t moved = __shfl_down_sync(0xffffffffu, gbuf, cnt & 31);
      const uint32_t qn2 = min(qn + cnt, qe);
      gbuf = lane + cnt < 32 ? moved : (qn2 + lane < qe ? __ldg(G3w + qn2 + lane) : 0u);
      if (!has && myp < qe) {
        ip1 = myp;
        const uint32_t d3 = gg & 0x7fff;
        flag = gg & G3_FLAG ? PROF_AT_MAXDIST : 0u;
        best = MIN_MATCH - 1, bestd = 0, r32 = 0, snap = false;
        bool walk = false;
        if (d3) {  // live, with a same-3-gram candidate within the budget
          const uint32_t la = min(nrel - ip1 + 1, 1u << 20);
          nice = min(NICE_LENGTH, la), maxl = min(MAX_MATCH, la);
          lim1 = (uint32_t)max((int)ip1 - (int)MAX_DIST, 1);
          // the first same-3-gram candidate (the only source of a match of exactly 3)
          const uint32_t c3 = ip1 - d3, s3 = (gg >> 15) & 0xff;
          if (s3 > 32) snap = true;  // r32 stays "no match"
          best = (w32[c3 + 2] ^ w32[ip1 + 2]) >> 16 ? 3u : 4u;  // byte 3
          if (best == 4) best = extend(c3, 4);
          best = min(best, maxl);
          bestd = d3;
          // then the first same-4-gram candidate (it matches >= 4 > 3, so it is extended at once)
          const uint32_t c4 = w32[ip1] & 0xffff, s4 = sk[ip1];
          if (best < nice && best < maxl && c4 != 0 && s4 <= MAX_CHAIN && (c4 > lim1 || (s4 == 1 && c4 == lim1))) {
            if (c4 != c3) {
              if (s4 > 32 && !snap) {
                r32 = prof_pack(best, bestd);
                snap = true;
              }
              const uint32_t len = extend(c4, 4);
              if (len > best) best = len, bestd = ip1 - c4;
            }
            c = w32[c4] & 0xffff;
            stp = s4 + sk[c4];
            walk = best < nice && best < maxl && c != 0 && stp <= MAX_CHAIN && c > lim1;
          }
        }
        if (walk) {
          key = w32[ip1 + best - 1] >> 16;
          has = true;
          done = false;
        } else {
          store((gg & G3_LIVE) != 0);
        }
      }
      qn = qn2;
    }
    if (!__any_sync(0xffffffffu, has)) {
      if (qn >= qe) break;
      continue;
    }
#ifndef PF4_NO_PAUSE
    // PB_STEPS hops along the 4-gram subsequence, branch-free.  A lane whose candidate passes
    // the quick test (bytes best - 1, best) pauses there for the rest of the batch; after the
    // batch every paused lane extends its one candidate.  best never lags the test, and the
    // extension is one candidate per lane instead of each lane's recorded list in turn (the
    // warp ran the longest list: ~45 % of the kernel's instructions).
    const uint32_t qb = sw + 4 * best - 2;  // + 4 c: the candidate's bytes (best - 1, best)
    bool paused = false;
    uint32_t pc = 0, ps = 0;  // the paused-on candidate and its chain step
#pragma unroll
    for (int t = 0; t < PB_STEPS; t++) {
      uint32_t wc, we, k;
      asm("ld.shared.u32 %0, [%1];" : "=r"(wc) : "r"(sw + 4 * c));
      asm("ld.shared.u16 %0, [%1];" : "=r"(we) : "r"(qb + 4 * c));
      asm("ld.shared.u8 %0, [%1];" : "=r"(k) : "r"(skb + c));
      const bool live = !done && !paused;
      const bool hit = live && we == key;
      pc = hit ? c : pc;
      ps = hit ? stp : ps;
      const uint32_t nc = wc & 0xffff, ns = stp + k;
      const bool ok = nc > lim1 && ns <= MAX_CHAIN;
      const bool adv = live && ok;
      done = done || (live && !ok);
      paused = paused || hit;
      c = adv ? nc : c;
      stp = adv ? ns : stp;
    }
    if (__any_sync(0xffffffffu, paused) && paused) {
      if (ps > 32 && !snap) {  // the budget-32 result: everything before this candidate
        r32 = best | (bestd << 9);  // best >= 4 while walking
        snap = true;
      }
      // bytes 0-3 (same 4-gram) and best - 1, best (quick test) are known to match: up to
      // best = 5 that is every byte before best + 1
      const uint32_t len = extend(pc, best <= 5 ? best + 1 : 4);
      if (len > best) {
        best = len;
        bestd = ip1 - pc;
        key = w32[ip1 + best - 1] >> 16;
        if (best >= nice || best >= maxl) done = true;
      }
    }
    if (has && done) {
      store_walked();
      has = false;
    }
#else
    // PB_STEPS hops along the 4-gram subsequence, branch-free; candidates passing the quick
    // test (bytes best - 1, best of the lagging best) are recorded
    uint32_t cand[PB_STEPS];
    uint32_t mask = 0, m32 = 0;  // m32: the steps whose candidate lies beyond the budget-32 prefix
    const uint32_t qb = sw + 4 * best - 2;  // + 4 c: the candidate's bytes (best - 1, best)
#pragma unroll
    for (int t = 0; t < PB_STEPS; t++) {
      uint32_t wc, we, k;
      asm("ld.shared.u32 %0, [%1];" : "=r"(wc) : "r"(sw + 4 * c));
      asm("ld.shared.u16 %0, [%1];" : "=r"(we) : "r"(qb + 4 * c));
      asm("ld.shared.u8 %0, [%1];" : "=r"(k) : "r"(skb + c));
      cand[t] = c;
      m32 |= stp > 32 ? 1u << t : 0u;
      mask |= (!done && we == key) ? 1u << t : 0u;
      const uint32_t nc = wc & 0xffff, ns = stp + k;
      const bool adv = !done && nc > lim1 && ns <= MAX_CHAIN;
      done = !adv;
      c = adv ? nc : c;
      stp = adv ? ns : stp;
    }
    // extend the recorded candidates in chain order
    bool improved = false;
    while (mask) {
      const int t = __ffs(mask) - 1;
      mask &= mask - 1;
      const uint32_t cx = pf_pick(cand, t);
      if (((m32 >> t) & 1) && !snap) {  // the budget-32 result: everything before this candidate
        r32 = best | (bestd << 9);  // best >= 4 while walking
        snap = true;
      }
      // re-test against the current best if it grew in this flush
      if (improved && (w32[cx + best - 1] >> 16) != (w32[ip1 + best - 1] >> 16)) continue;
      // bytes 0-3 (same 4-gram) and best - 1, best (quick test) are known to match: up to
      // best = 5 that is every byte before best + 1
      const uint32_t len = extend(cx, best <= 5 ? best + 1 : 4);
      if (len > best) {
        best = len;
        bestd = ip1 - cx;
        improved = true;
        if (best >= nice || best >= maxl) {
          done = true;
          mask = 0;
        }
      }
    }
    if (improved) key = w32[ip1 + best - 1] >> 16;
    if (has && done) {
      store_walked();
      has = false;
    }
#endif
  }
}

// Which walk a lane takes.  K4G pays off where chains are long and same-4-gram candidates
// sparse (bf16 exponent planes: 110 chain steps per position vs 17 to the first 4-gram
// candidate + 11 hops); on short chains (fp16 planes: ~6 steps, no 4-gram candidates) its
// two passes cost more than K4's one.  A sampled walk per lane (1024 positions, K3 links in
// global memory) measures the chain length L, the steps to the first same-4-gram candidate
// S4 and the same-4-gram hops H4; the host picks K4G where L >= S4 + H4 + K4G_MARGIN on average
// (K4G's one-load steps are cheaper than the classic walk's, its two passes cost a couple of
// steps per position: config3's f32 planes with L = 35 / 119 gain, fp16 planes with L = 6 = S4 lose).
constexpr uint32_t K4S_CTAS = 4;  // x 256 threads = samples per lane
static std::atomic<uint64_t> g_k4_positions[2];  // positions profiled by the classic walk / by K4G
constexpr uint64_t K4G_MIN_LANE = 1u << 20;
#ifndef K4G_MARGIN
#define K4G_MARGIN 2  // K4G where L >= S4 + H4 + K4G_MARGIN (means per sampled position)
#endif
__global__ void __launch_bounds__(256) k_k4_sample(const LaneDev* __restrict__ lanes, const uint16_t* __restrict__ pd,
                                                   unsigned long long* __restrict__ stat) {
  const LaneDev L = lanes[blockIdx.y];
  const uint64_t n = L.n;
  if (n < K4G_MIN_LANE) return;
  const uint32_t ns = gridDim.x * blockDim.x, k = blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t p = n * (2ull * k + 1) / (2ull * ns);
  const uint8_t* src = L.src;
  const uint16_t* P = pd + L.pbase;
  uint32_t len = 0, s4 = 0, h4 = 0;
  if (p + 4 <= n) {
    auto four = [&](uint64_t q) {
      return (uint32_t)__ldg(src + q) | ((uint32_t)__ldg(src + q + 1) << 8) | ((uint32_t)__ldg(src + q + 2) << 16) |
             ((uint32_t)__ldg(src + q + 3) << 24);
    };
    const uint32_t key = four(p);
    const uint64_t limit = p > MAX_DIST ? p - MAX_DIST : 0;
    uint32_t d = P[p];
    uint64_t c = p - d;
    bool ok = d != 0 && d <= MAX_DIST && c != 0;
    while (ok && len < MAX_CHAIN) {
      len++;
      if (four(c) == key) {
        h4++;
        if (!s4) s4 = len;
      }
      d = P[c];
      ok = d != 0 && d < c && c - d > limit;
      c -= d;
    }
    if (!s4) s4 = len;
  }
  const unsigned full = 0xffffffffu;
  len = __reduce_add_sync(full, len);
  s4 = __reduce_add_sync(full, s4);
  h4 = __reduce_add_sync(full, h4);
  if ((threadIdx.x & 31) == 0) {
    unsigned long long* S = stat + 4 * blockIdx.y;
    atomicAdd(S, (unsigned long long)len);
    atomicAdd(S + 1, (unsigned long long)s4);
    atomicAdd(S + 2, (unsigned long long)h4);
    atomicAdd(S + 3, 32ull);
  }
}

// ---------------------------------------------------------------------------
// K3S + K4S: match profiles over BUCKET-SORTED chains (variant, BB_K4_SORTED=1).
//
// zlib's hash chain of position p is the list of earlier positions with the same
// 15-bit hash, most recent first (parse-independent, see K3).  A stable sort of
// all positions by (lane, hash) lays every chain out contiguously: p's t-th
// candidate is simply the sorted entry t places before p's own.  K4S gives each
// thread one sorted entry, so the 32 lanes of a warp are 32 consecutive entries
// and at chain step t they read 32 consecutive candidate records from shared
// memory -- conflict-free, with no dependent link loads.  A record is the 8
// bytes starting at the candidate, so the quick reject and the match length up
// to 8 bytes come from one 64-bit load: x = cand ^ own, the candidate can beat
// best only if bytes 0..best of x are zero, and the length is ctz(x) / 8.
// Longer matches extend from the lane's bytes in global memory (rare on
// activation planes).  The chain budget (32 / 128 candidates), the distance rule
// (the head at <= MAX_DIST, later entries < MAX_DIST, position 0 never a
// source), nice_match and the first-maximum rule are exactly K4's, so the
// profiles are bit-identical (tests/test_gpu_deflate.py compares both with the
// oracle's orc_match_profile).
//
//   k_sort_keys      key = lane << 16 | hash(p) (0xffff: fewer than 3 bytes left,
//                    never inserted), value = p
//   cub radix sort   stable: positions stay ascending inside a bucket
//   k_profile_sorted CTA per KS_T sorted entries; stages the KS_H entries before
//                    them (the longest chain a thread can walk) with their bytes
constexpr uint32_t KS_NOHASH = 0xffffu;
constexpr int KS_T = 1024;  // sorted entries (threads) per CTA
constexpr int KS_H = 128;   // history entries staged before them (MAX_CHAIN)

// 8 bytes starting at src + q (bytes at or past n read as 0)
__device__ __forceinline__ uint64_t ks_load8(const uint8_t* src, uint64_t n, uint64_t q) {
  const uint64_t a = q & ~uint64_t(7);
  const uint32_t sh = (uint32_t)(q & 7) * 8;
  const bool aligned_src = (reinterpret_cast<uintptr_t>(src) & 7) == 0;
  if (aligned_src && a + 16 <= n) {
    const uint64_t lo = __ldg(reinterpret_cast<const unsigned long long*>(src + a));
    if (!sh) return lo;
    const uint64_t hi = __ldg(reinterpret_cast<const unsigned long long*>(src + a + 8));
    return (lo >> sh) | (hi << (64 - sh));
  }
  uint64_t v = 0;
#pragma unroll
  for (int k = 0; k < 8; k++)
    if (q + k < n) v |= (uint64_t)__ldg(src + q + k) << (8 * k);
  return v;
}

// grid (chunks, lanes): KS_KP positions per thread, keys = 15-bit hash (KS_NOHASH when fewer
// than 3 bytes remain: never inserted, never searched), values = position
constexpr int KS_KP = 8;
__global__ void __launch_bounds__(256) k_sort_keys(const LaneDev* __restrict__ lanes,
                                                   const uint64_t* __restrict__ lane_prefix,
                                                   uint16_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const LaneDev L = lanes[blockIdx.y];
  const uint64_t o = lane_prefix[blockIdx.y];
  for (uint64_t p0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * KS_KP; p0 < L.n;
       p0 += (uint64_t)gridDim.x * blockDim.x * KS_KP) {
    const uint64_t a = ks_load8(L.src, L.n, p0), b = ks_load8(L.src, L.n, p0 + 8);
#pragma unroll
    for (int k = 0; k < KS_KP; k++) {
      const uint64_t p = p0 + k;
      if (p >= L.n) break;
      const uint32_t b0 = (uint32_t)(a >> (8 * k)) & 0xff;
      const uint32_t b1 = (uint32_t)(k + 1 < 8 ? a >> (8 * (k + 1)) : b >> (8 * (k - 7))) & 0xff;
      const uint32_t b2 = (uint32_t)(k + 2 < 8 ? a >> (8 * (k + 2)) : b >> (8 * (k - 6))) & 0xff;
      const uint32_t h = p + MIN_MATCH <= L.n ? ((b0 << 10) ^ (b1 << 5) ^ b2) & 0x7fffu : KS_NOHASH;
      keys[o + p] = (uint16_t)h;
      vals[o + p] = (uint32_t)p;
    }
  }
}

// common-prefix length of src[c..] and src[p..] from byte `from` (bytes below it match), capped at maxl
__device__ __noinline__ uint32_t ks_extend(const uint8_t* src, uint64_t n, uint64_t c, uint64_t p, uint32_t from,
                                           uint32_t maxl) {
  uint32_t len = from;
  while (len < maxl) {
    const uint64_t x = ks_load8(src, n, c + len) ^ ks_load8(src, n, p + len);
    if (x) {
      len += (uint32_t)(__ffsll((long long)x) - 1) >> 3;
      break;
    }
    len += 8;
  }
  return min(len, maxl);
}

__device__ __forceinline__ uint32_t ks_ctz(uint32_t x) {  // x != 0
  uint32_t r;
  asm("brev.b32 %0, %1;" : "=r"(r) : "r"(x));
  asm("bfind.shiftamt.u32 %0, %0;" : "+r"(r));
  return r;
}

constexpr int KS_B = 8;    // chain steps per batch (the quick tests of a batch are branch-free)
constexpr int KS_PAD = 8;  // staged records before the window: a batch may overrun the chain

__global__ void __launch_bounds__(KS_T, 1) k_profile_sorted(const LaneDev* __restrict__ lanes,
                                                            const uint64_t* __restrict__ lane_prefix,
                                                            const uint16_t* __restrict__ skeys,
                                                            const uint32_t* __restrict__ spos,
                                                            uint2* __restrict__ prof, int with_bytes) {
  __shared__ uint64_t sb[KS_PAD + KS_H + KS_T];  // 8 bytes at each staged entry's position
  __shared__ uint32_t sk[KS_H + KS_T];           // its hash (KS_NOHASH outside the lane)
  __shared__ uint32_t sp[KS_H + KS_T];           // its position
  const LaneDev L = lanes[blockIdx.y];
  const uint64_t n = L.n;
  const uint64_t j0 = (uint64_t)blockIdx.x * KS_T;  // lane-relative sorted index
  if (j0 >= n) return;
  const uint16_t* keys = skeys + lane_prefix[blockIdx.y];
  const uint32_t* poss = spos + lane_prefix[blockIdx.y];
  const int64_t base = (int64_t)j0 - KS_H;  // staged index i <-> sorted entry base + i
  if (threadIdx.x < KS_PAD) sb[threadIdx.x] = ~0ull;
  for (int i = threadIdx.x; i < KS_H + KS_T; i += blockDim.x) {
    const int64_t j = base + i;
    uint32_t k = KS_NOHASH, q = 0;
    uint64_t b = 0;
    if (j >= 0 && (uint64_t)j < n) {
      k = keys[j];
      q = poss[j];
      b = ks_load8(L.src, n, q);
    }
    sk[i] = k;
    sp[i] = q;
    sb[KS_PAD + i] = b;
  }
  __syncthreads();
  const int me = KS_H + threadIdx.x;
  const uint64_t j = j0 + threadIdx.x;
  const bool in = j < n;
  const uint32_t key = sk[me];
  const uint32_t p = sp[me];
  // candidates: staged entries [lo, me) with the same hash, newest first.  The head (me - 1)
  // is searched when it lies within MAX_DIST and is not position 0 (deflate_slow's test);
  // later ones must lie above limit = p - MAX_DIST (longest_match's do-while).
  int K = 0;
  uint32_t flag = 0;
  if (in && key != KS_NOHASH && sk[me - 1] == key) {
    const uint32_t c1 = sp[me - 1];
    const uint32_t d0 = p - c1;
    if (d0 <= MAX_DIST && c1 != 0) {
      flag = d0 == MAX_DIST ? PROF_AT_MAXDIST : 0;
      const uint32_t limit = p > MAX_DIST ? p - MAX_DIST : 0;
      int lo = me - (int)MAX_CHAIN, hi = me - 1;  // first index in [me - 128, me - 2] with the hash, > limit
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sk[mid] == key && sp[mid] > limit) hi = mid;
        else lo = mid + 1;
      }
      K = me - lo;  // the head plus entries lo .. me - 2
    }
  }
  const uint32_t la = in ? (uint32_t)umin64(n - p, 1u << 20) : 0;
  const uint32_t nice = min(NICE_LENGTH, la), maxl = min(MAX_MATCH, la);
  const uint2* rec = reinterpret_cast<const uint2*>(sb) + KS_PAD + me;
  const uint2 ownr = rec[0];
  const uint32_t olo = ownr.x, ohi = ownr.y;
  // A candidate can only be longer than best if bytes 0 .. best all match (mlo / mhi), and then
  // it is -- unless best grew earlier in the same batch, so every recorded candidate is
  // re-tested in chain order when the batch is flushed: the result is the first maximum.
  uint32_t best = MIN_MATCH - 1, tb = 0, mlo = 0xffffffu, mhi = 0u;
  uint32_t b32 = MIN_MATCH - 1, tb32 = 0;
  int Kw = K;
#pragma unroll
  for (int o = 16; o; o >>= 1) Kw = max(Kw, __shfl_xor_sync(0xffffffffu, Kw, o));
  for (int t0 = 1; t0 <= Kw; t0 += KS_B) {
    uint32_t bits = 0;
#pragma unroll
    for (int u = 0; u < KS_B; u++) {
      const uint2 r = rec[-(t0 + u)];
      const bool pass = (((r.x ^ olo) & mlo) | ((r.y ^ ohi) & mhi)) == 0u;
      bits |= (pass && t0 + u <= K) ? 1u << u : 0u;
    }
    while (bits) {
      const int t = t0 + __ffs(bits) - 1;
      bits &= bits - 1;
      const uint2 r = rec[-t];
      const uint32_t xl = r.x ^ olo, xh = r.y ^ ohi;
      if (((xl & mlo) | (xh & mhi)) != 0u) continue;  // best grew within this batch
      uint32_t len = xl ? ks_ctz(xl) >> 3 : xh ? 4u + (ks_ctz(xh) >> 3) : 8u;
      if (len == 8u && maxl > 8u) len = ks_extend(L.src, n, sp[me - t], p, 8, maxl);
      len = min(len, maxl);
      if (len > best) {
        best = len;
        tb = t;
        mlo = best >= 3 ? 0xffffffffu : (2u << (8 * best + 7)) - 1;
        mhi = best <= 3 ? 0u : best >= 7 ? 0xffffffffu : (2u << (8 * (best - 4) + 7)) - 1;
        if (best >= nice) {  // zlib stops at nice_match
          K = t;
          bits = 0;
        }
      }
    }
    if (t0 + KS_B - 1 == 32) b32 = best, tb32 = tb;  // budget 32 (prev_length >= good_match)
  }
  if (Kw < 32) b32 = best, tb32 = tb;
  if (!in) return;
  const uint32_t yb = with_bytes ? (p ? (uint32_t)__ldg(L.src + p - 1) << 24 : 0u) : 0u;
  if (K == 0) {
    prof[L.pbase + p] = make_uint2(0u, yb);
    return;
  }
  const uint32_t bestd = tb ? p - sp[me - tb] : 0;
  const uint32_t bestd32 = tb32 ? p - sp[me - tb32] : 0;
  prof[L.pbase + p] = make_uint2(prof_pack(best, bestd) | flag, yb | prof_pack(b32, bestd32) | (with_bytes ? 0u : flag));
}

// K3S + K4S over all lanes of a call: keys, one stable 16-bit radix sort per lane (two
// passes), profiles (see k_profile_sorted)
template <class Timer>
static int profile_sorted(Workspace& sortws, Workspace& W, const LaneDev* d_lanes, int nl,
                          const std::vector<uint64_t>& lane_prefix, uint2* d_prof, int with_bytes, Timer& T,
                          cudaStream_t st) {
  const uint64_t total = lane_prefix[nl];
  if (!total) return BB_OK;
  uint64_t longest = 0;
  for (int i = 0; i < nl; i++) longest = std::max(longest, lane_prefix[i + 1] - lane_prefix[i]);
  if (longest >= (1ull << 31)) {
    set_error("deflate lane of %llu bytes exceeds the 2 Gi sort limit", (unsigned long long)longest);
    return BB_ERROR;
  }
  size_t tmp = 0;
  BB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const uint16_t*)nullptr, (uint16_t*)nullptr,
                                              (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)longest, 0, 16,
                                              st));
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  int rc = sortws.reserve(2 * al(2 * total) + 2 * al(4 * total) + al(tmp) + al(8 * (nl + 1)) + 4096);
  if (rc) return rc;
  uint16_t* k0 = sortws.take<uint16_t>(total);
  uint16_t* k1 = sortws.take<uint16_t>(total);
  uint32_t* v0 = sortws.take<uint32_t>(total);
  uint32_t* v1 = sortws.take<uint32_t>(total);
  void* d_tmp = sortws.take<uint8_t>(tmp);
  uint64_t* d_lp = sortws.take<uint64_t>(nl + 1);
  (void)W;
  BB_CUDA_TRY(cudaMemcpyAsync(d_lp, lane_prefix.data(), 8 * (nl + 1), cudaMemcpyHostToDevice, st));
  T.mark("deflate.hash_sort");
  {
    const unsigned gx = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((longest + 256 * KS_KP - 1) / (256 * KS_KP), 4096));
    k_sort_keys<<<dim3(gx, nl), 256, 0, st>>>(d_lanes, d_lp, k0, v0);
    BB_LAUNCH_CHECK();
  }
  for (int i = 0; i < nl; i++) {
    const uint64_t o = lane_prefix[i], m = lane_prefix[i + 1] - o;
    if (!m) continue;
    size_t t2 = tmp;
    BB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(d_tmp, t2, k0 + o, k1 + o, v0 + o, v1 + o, (int)m, 0, 16, st));
    count_launch(2);
  }
  T.mark("deflate.profile");
  k_profile_sorted<<<dim3((unsigned)((longest + KS_T - 1) / KS_T), nl), KS_T, 0, st>>>(d_lanes, d_lp, k1, v1, d_prof,
                                                                                    with_bytes);
  BB_LAUNCH_CHECK();
  return BB_OK;
}

// ---------------------------------------------------------------------------
// K5: the lazy parse (deflate_slow) as a per-position state machine over profiles.
// The parse walks its segment forward, so profiles are fetched PR_CHUNK at a time
// (32-byte aligned vector loads into registers), with the following chunk
// already in flight, instead of one dependent 8-byte load per position; lanes
// are padded to 256 positions, so a chunk never leaves the lane's slice of the
// profile array.  The byte before each position rides in profile.y bits 24-31
// (K4 stores it), so emitting a literal needs no load of the input.
constexpr uint32_t PR_CHUNK = 4;
struct Parser {
  const uint2* prof;  // lane-relative
  uint64_t n;
  uint32_t p, L, avail, dist;
  uint32_t cb = 0xffffffffu;  // first position of the cached chunk (~0: none)
  uint4 a01, a23, b01, b23;   // chunks cb and cb + PR_CHUNK

  __device__ __forceinline__ void fetch(uint32_t q, uint4& x01, uint4& x23) {
    if (q < n) {
      const uint4* v = reinterpret_cast<const uint4*>(prof + q);
      x01 = __ldg(v);
      x23 = __ldg(v + 1);
    }
  }
  __device__ __forceinline__ uint2 prof_at(uint32_t q) {
    const uint32_t qb = q & ~(PR_CHUNK - 1);
    if (qb != cb) {
      if (qb == cb + PR_CHUNK)
        a01 = b01, a23 = b23;
      else
        fetch(qb, a01, a23);
      cb = qb;
      fetch(qb + PR_CHUNK, b01, b23);
    }
    const uint32_t k = q - cb;
    const uint4 h = k & 2 ? a23 : a01;
    return k & 1 ? make_uint2(h.z, h.w) : make_uint2(h.x, h.y);
  }

  // One loop-top iteration at p < n.  Returns a symbol or 0 (none).
  __device__ __forceinline__ uint32_t step() {
    uint32_t ml = MIN_MATCH - 1, md = 0, prev_byte = 0;
    if (L < MAX_LAZY) {
      const uint2 pr = prof_at(p);
      const uint32_t v = L >= GOOD_LENGTH ? pr.y : pr.x;
      const bool nil = (pr.x & PROF_AT_MAXDIST) && nil_head_at(p, n);
      const uint32_t len = v & 0x1ff;
      if (!nil && len > L) ml = len, md = (v >> 9) & 0x7fff;
      prev_byte = pr.y >> 24;
    }
    if (L >= MIN_MATCH && ml <= L) {
      uint32_t sym = SYM_MATCH | (L - MIN_MATCH) | ((dist - 1) << 8);
      p = p - 1 + L;
      L = MIN_MATCH - 1;
      avail = 0;
      dist = 0;
      return sym;
    }
    // (a literal is only emitted when L < MIN_MATCH, so the profile was read)
    uint32_t sym = 0;
    if (avail) sym = 0x40000000u | prev_byte;  // bit 30 marks "literal present"
    avail = 1;
    p++;
    L = ml;
    dist = md;
    return sym;
  }
  __device__ __forceinline__ uint32_t state() const { return pack_state(L, avail, dist); }
};

// strips the "present" marker of literal symbols
__device__ __forceinline__ uint32_t sym_clean(uint32_t s) { return s & ~0x40000000u; }

__global__ void k_parse_spec(const LaneDev* __restrict__ lanes, int nlanes,
                             const uint32_t* __restrict__ seg_lane, uint32_t nseg_total,
                             const uint2* __restrict__ prof, uint32_t* __restrict__ spec_syms,
                             uint2* __restrict__ state_map, SegExit* __restrict__ spec_exit,
                             uint32_t* __restrict__ spec_cnt, uint32_t* __restrict__ spec_post,
                             uint32_t sym_stride) {
  uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nseg_total) return;
  const LaneDev Ld = lanes[seg_lane[g]];
  const uint32_t k = g - Ld.seg0;
  const uint64_t s = (uint64_t)k * Ld.G;
  const uint64_t e = umin64(s + Ld.G, Ld.n);
  Parser P{prof + Ld.pbase, Ld.n, (uint32_t)s, MIN_MATCH - 1, 0, 0};
  uint32_t* out = spec_syms + (uint64_t)g * sym_stride;
  uint2* sm = state_map + (uint64_t)g * CONV_W;
  uint32_t cnt = 0, next_w = 0;
  // symbols leave four at a time as one 16-byte store (rows are 16-byte aligned)
  uint4 buf = make_uint4(0, 0, 0, 0);
  auto put = [&](uint32_t v) {
    const uint32_t j = cnt & 3;
    buf.x = j == 0 ? v : buf.x;
    buf.y = j == 1 ? v : buf.y;
    buf.z = j == 2 ? v : buf.z;
    buf.w = j == 3 ? v : buf.w;
    if (j == 3) *reinterpret_cast<uint4*>(out + cnt - 3) = buf;
    cnt++;
  };
  while (P.p < e) {
    uint32_t rel = P.p - (uint32_t)s;
    if (rel < CONV_W) {
      for (; next_w < rel; next_w++) sm[next_w] = make_uint2(0, 0);
      sm[rel] = make_uint2(P.state(), cnt);
      next_w = rel + 1;
    }
    uint32_t sym = P.step();
    if (sym) put(sym_clean(sym));
  }
  for (; next_w < CONV_W; next_w++) sm[next_w] = make_uint2(0, 0);
  uint32_t post = 0;
  if (k == Ld.nseg - 1 && P.p >= Ld.n && P.avail) {
    put(Ld.src[Ld.n - 1]);
    post = 1;
  }
  {
    const uint32_t j = cnt & 3, b0 = cnt - j;  // the partial last group
    if (j > 0) out[b0] = buf.x;
    if (j > 1) out[b0 + 1] = buf.y;
    if (j > 2) out[b0 + 2] = buf.z;
  }
  spec_exit[g] = SegExit{P.p, P.state()};
  spec_cnt[g] = cnt;
  spec_post[g] = post;
}

// One Jacobi round: every segment re-derives its result from its predecessor's
// current exit state.  A segment whose entry is unchanged is skipped.
// one fix-up round of segment g: re-parse from the predecessor's exit until the parse meets the
// speculative one (or the segment ends); *changed counts segments whose exit moved
__device__ __forceinline__ void parse_fixup_seg(uint32_t g, const LaneDev* __restrict__ lanes,
                                                const uint32_t* __restrict__ seg_lane, const uint2* __restrict__ prof,
                                                const uint2* __restrict__ state_map,
                                                const SegExit* __restrict__ spec_exit,
                                                const uint32_t* __restrict__ spec_cnt,
                                                const uint32_t* __restrict__ spec_post,
                                                const SegExit* exit_prev, SegExit* exit_next,
                                                SegExit* __restrict__ entry_used, uint32_t* __restrict__ fix_syms,
                                                uint32_t* __restrict__ fix_cnt, uint32_t* __restrict__ conv_idx,
                                                uint32_t* __restrict__ post_flag, uint32_t* changed,
                                                uint32_t sym_stride) {
  const LaneDev Ld = lanes[seg_lane[g]];
  const uint32_t k = g - Ld.seg0;
  if (k == 0) {
    exit_next[g] = exit_prev[g];
    return;
  }
  const SegExit entry = exit_prev[g - 1];
  const SegExit used = entry_used[g];
  if (entry.p == used.p && entry.state == used.state) {
    exit_next[g] = exit_prev[g];
    return;
  }
  entry_used[g] = entry;
  const uint64_t s = (uint64_t)k * Ld.G;
  const uint64_t e = umin64(s + Ld.G, Ld.n);
  Parser P{prof + Ld.pbase, Ld.n, entry.p, entry.state & 0x1ff, (entry.state >> 9) & 1,
           (entry.state >> 10) & 0x7fff};
  const uint2* sm = state_map + (uint64_t)g * CONV_W;
  uint32_t* out = fix_syms + (uint64_t)g * sym_stride;
  uint32_t cnt = 0;
  bool conv = false;
  uint32_t ci = 0;
  while (P.p < e) {
    uint32_t rel = P.p - (uint32_t)s;
    if (rel < CONV_W) {
      uint2 v = sm[rel];
      if (v.x == P.state()) {
        conv = true;
        ci = v.y;
        break;
      }
    }
    uint32_t sym = P.step();
    if (sym) out[cnt++] = sym_clean(sym);
  }
  SegExit ex;
  uint32_t post = 0;
  if (conv) {
    ex = spec_exit[g];
    post = spec_post[g];
  } else {
    ci = spec_cnt[g];  // no speculative tail
    if (k == Ld.nseg - 1 && P.p >= Ld.n && P.avail) {
      out[cnt++] = Ld.src[Ld.n - 1];
      post = 1;
    }
    ex = SegExit{P.p, P.state()};
  }
  fix_cnt[g] = cnt;
  conv_idx[g] = ci;
  post_flag[g] = post;
  exit_next[g] = ex;
  const SegExit old = exit_prev[g];
  if (old.p != ex.p || old.state != ex.state) atomicAdd(changed, 1u);
}

__global__ void k_parse_fixup(const LaneDev* __restrict__ lanes, const uint32_t* __restrict__ seg_lane,
                              uint32_t nseg_total, const uint2* __restrict__ prof,
                              const uint2* __restrict__ state_map, const SegExit* __restrict__ spec_exit,
                              const uint32_t* __restrict__ spec_cnt, const uint32_t* __restrict__ spec_post,
                              const SegExit* __restrict__ exit_prev, SegExit* __restrict__ exit_next,
                              SegExit* __restrict__ entry_used, uint32_t* __restrict__ fix_syms,
                              uint32_t* __restrict__ fix_cnt, uint32_t* __restrict__ conv_idx,
                              uint32_t* __restrict__ post_flag, uint32_t* __restrict__ changed,
                              uint32_t sym_stride) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nseg_total) return;
  parse_fixup_seg(g, lanes, seg_lane, prof, state_map, spec_exit, spec_cnt, spec_post, exit_prev, exit_next,
                  entry_used, fix_syms, fix_cnt, conv_idx, post_flag, changed, sym_stride);
}

// All fix-up rounds in one cooperative launch (opt-in, BB_FIXUP_COOP=1): a grid-wide barrier
// separates the rounds and the loop ends on the device when a round moves no exit.  Three
// rotating counters: round r counts into c[r % 3]; after its barrier every thread reads it and
// thread 0 clears c[(r + 2) % 3], whose last reader passed that same barrier.
__global__ void __launch_bounds__(128) k_parse_fixup_coop(
    const LaneDev* __restrict__ lanes, const uint32_t* __restrict__ seg_lane, uint32_t nseg_total,
    const uint2* __restrict__ prof, const uint2* __restrict__ state_map, const SegExit* __restrict__ spec_exit,
    const uint32_t* __restrict__ spec_cnt, const uint32_t* __restrict__ spec_post, SegExit* exit_a,
    SegExit* exit_b, SegExit* __restrict__ entry_used, uint32_t* __restrict__ fix_syms,
    uint32_t* __restrict__ fix_cnt, uint32_t* __restrict__ conv_idx, uint32_t* __restrict__ post_flag,
    volatile uint32_t* counters, uint32_t sym_stride, uint32_t max_rounds) {
  cg::grid_group grid = cg::this_grid();
  const SegExit* cur = exit_a;
  SegExit* nxt = exit_b;
  for (uint32_t r = 0; r < max_rounds; r++) {
    uint32_t* c = const_cast<uint32_t*>(counters) + (r % 3);
    for (uint64_t g = grid.thread_rank(); g < nseg_total; g += grid.size())
      parse_fixup_seg((uint32_t)g, lanes, seg_lane, prof, state_map, spec_exit, spec_cnt, spec_post, cur, nxt,
                      entry_used, fix_syms, fix_cnt, conv_idx, post_flag, c, sym_stride);
    grid.sync();
    if (grid.thread_rank() == 0) counters[(r + 2) % 3] = 0;
    if (counters[r % 3] == 0) return;
    const SegExit* t = nxt;
    nxt = const_cast<SegExit*>(cur);
    cur = t;
  }
  if (grid.thread_rank() == 0) counters[3] = 1;  // did not converge within max_rounds
}

// the fresh state each speculative parse assumed: segment k of a lane starts at k * G with
// prev_length = MIN_MATCH - 1, no pending literal (written on the device: no host round trip)
__global__ void k_fresh_entries(const LaneDev* __restrict__ lanes, const uint32_t* __restrict__ seg_lane,
                                uint32_t nseg_total, SegExit* __restrict__ entry_used) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nseg_total) return;
  const LaneDev Ld = lanes[seg_lane[g]];
  entry_used[g] = SegExit{(g - Ld.seg0) * Ld.G, 0x80000000u | (MIN_MATCH - 1)};
}

// ---------------------------------------------------------------------------
// K6a: per-lane symbol offsets of every segment (one CTA per lane)
struct LaneSyms {
  uint64_t total;  // symbols in the lane
  uint32_t post;   // last symbol is the post-loop literal
  uint32_t nblk;   // blocks
};

__global__ void __launch_bounds__(256) k_seg_scan(const LaneDev* __restrict__ lanes,
                                                 const uint32_t* __restrict__ spec_cnt,
                                                 const uint32_t* __restrict__ fix_cnt,
                                                 const uint32_t* __restrict__ conv_idx,
                                                 const uint32_t* __restrict__ post_flag,
                                                 const uint32_t* __restrict__ spec_post,
                                                 uint64_t* __restrict__ seg_off, LaneSyms* __restrict__ ls) {
  typedef cub::BlockScan<uint64_t, 256> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint64_t carry;
  const LaneDev Ld = lanes[blockIdx.x];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < Ld.nseg; base += 256) {
    uint32_t k = base + threadIdx.x;
    uint64_t c = 0;
    if (k < Ld.nseg) {
      uint32_t g = Ld.seg0 + k;
      c = (uint64_t)fix_cnt[g] + spec_cnt[g] - conv_idx[g];
    }
    uint64_t x, agg;
    Scan(tmp).ExclusiveSum(c, x, agg);
    if (k < Ld.nseg) seg_off[Ld.seg0 + k] = carry + x;
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    uint32_t gl = Ld.seg0 + Ld.nseg - 1;
    uint32_t post = post_flag[gl];
    LaneSyms r;
    r.total = carry;
    r.post = post;
    r.nblk = (uint32_t)((carry - post) / SYM_LIMIT + 1);
    ls[blockIdx.x] = r;
  }
}

// K6b: gather the final symbol stream (one warp per segment)
__global__ void k_compact(const LaneDev* __restrict__ lanes, const uint32_t* __restrict__ seg_lane,
                          uint32_t nseg_total, const uint32_t* __restrict__ spec_syms,
                          const uint32_t* __restrict__ spec_cnt, const uint32_t* __restrict__ fix_syms,
                          const uint32_t* __restrict__ fix_cnt, const uint32_t* __restrict__ conv_idx,
                          const uint64_t* __restrict__ seg_off, uint32_t* __restrict__ syms,
                          uint32_t sym_stride) {
  uint32_t g = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (g >= nseg_total) return;
  const int lane = threadIdx.x & 31;
  const LaneDev Ld = lanes[seg_lane[g]];
  uint32_t* dst = syms + Ld.sym_base + seg_off[g];
  uint32_t k = g - Ld.seg0;
  uint32_t fc = k ? fix_cnt[g] : 0;
  uint32_t ci = k ? conv_idx[g] : 0;
  const uint32_t* fs = fix_syms + (uint64_t)g * sym_stride;
  for (uint32_t i = lane; i < fc; i += 32) dst[i] = fs[i];
  const uint32_t* ss = spec_syms + (uint64_t)g * sym_stride;
  uint32_t sc = spec_cnt[g];
  for (uint32_t i = ci + lane; i < sc; i += 32) dst[fc + i - ci] = ss[i];
}

// ---------------------------------------------------------------------------
// K6c: per-block statistics and zlib's Huffman trees.
struct BlockInfo {
  uint64_t sym0;        // first symbol (lane-relative)
  uint32_t nsym;
  uint32_t stored_len;  // bytes covered
  uint32_t last_len;    // bytes covered by the final symbol
  uint32_t opt_lenb, static_lenb;
  uint32_t dyn_bits;    // full dynamic block incl. 3-bit type and EOB
  uint32_t static_bits; // full static block incl. 3-bit type and EOB
  uint32_t hdr_bits;    // dynamic tree description bits (after the 3-bit type)
  uint32_t valid;
};

// per block: lit/len codes (code | len << 16) [286] and dist codes [30]
struct BlockCodes {
  uint32_t l[L_CODES];
  uint32_t d[D_CODES];
};

// zlib trees.c state for one block.  The heap holds packed entries
// (freq << 32 | depth << 16 | node): zlib's smaller() order -- freq, then depth
// -- is the order of (entry >> 16), so each heap step is one 64-bit compare
// instead of four indirect loads.
template <int ELEMS>
struct TreeArr {
  uint16_t freq[ELEMS];
  uint16_t code[ELEMS];
  uint16_t dad[2 * ELEMS + 1];
  uint8_t len[2 * ELEMS + 2];  // +1: scan_tree guard slot (code lengths <= 15)
};

struct TreesState {
  TreeArr<L_CODES> lt;
  TreeArr<D_CODES> dt;
  TreeArr<BL_CODES> blt;
  alignas(16) uint32_t heap[HEAP_SIZE + 7];  // + grandson-load padding (t_down)
  uint16_t bl_count[16];
  uint64_t opt_len, static_len;
  int lmax, dmax, blmax;
};

// Heap entries pack (freq, depth, node) so one compare orders them as trees.c's
// smaller(): freq (15 bits: a block has <= 16384 symbols + 2 forced nodes) |
// depth (5 bits: a tree over <= 16386 counts is at most 21 deep) | node (10 bits).
__device__ __forceinline__ uint32_t t_entry(uint32_t freq, uint32_t depth, uint32_t node) {
  return (freq << 15) | (depth << 10) | node;
}
__device__ __forceinline__ uint32_t t_node(uint32_t e) { return e & 0x3ff; }
__device__ __forceinline__ uint32_t t_freq(uint32_t e) { return e >> 15; }
__device__ __forceinline__ uint32_t t_depth(uint32_t e) { return (e >> 10) & 0x1f; }

// trees.c pqdownheap with smaller(n, m) == key(n) <= key(m).  The walk down is one
// dependent shared-memory load per level; here the four grandsons (heap[4k .. 4k + 3],
// one 16-byte load) are fetched while the sons are compared, so each level's load was
// issued a level earlier.  (heap is padded: a grandson load may read past heap_len.)
// Used where few blocks run (K6 latency-bound: config1's 0.39 -> 0.30 ms); with many blocks
// per SM the extra loads cost shared-memory issue slots (config2 3.16 -> 3.28 ms), so the
// plain walk below serves that case.
__device__ __forceinline__ void t_down_pf(uint32_t* heap, int heap_len, int k) {
  const uint32_t v = heap[k];
  int j = k << 1;
  if (j <= heap_len) {
    uint2 sons = *reinterpret_cast<const uint2*>(heap + j);  // j even: 8-byte aligned
    uint4 gs = *reinterpret_cast<const uint4*>(heap + 2 * j);  // 2j = 4k: 16-byte aligned
    for (;;) {
      // key comparisons and the right-son sentinel as in t_down_plain
      const bool right = sons.y <= (sons.x | 0x3ffu);
      const uint32_t hj = right ? sons.y : sons.x;
      if (v <= (hj | 0x3ffu)) break;
      heap[k] = hj;
      k = j + right;
      j = k << 1;
      if (j > heap_len) break;
      sons = right ? make_uint2(gs.z, gs.w) : make_uint2(gs.x, gs.y);
      gs = *reinterpret_cast<const uint4*>(heap + 2 * j);
    }
  }
  heap[k] = v;
}
// (key(a) <= key(b) as a <= (b | 0x3ff): the node field never decides; heap[heap_len + 1] holds
// a sentinel above every key, so a missing right son is never taken -- t_build_tree keeps it)
__device__ __forceinline__ void t_down_plain(uint32_t* heap, int heap_len, int k) {
  const uint32_t v = heap[k];
  int j = k << 1;
  while (j <= heap_len) {
    const uint2 sons = *reinterpret_cast<const uint2*>(heap + j);
    const bool right = sons.y <= (sons.x | 0x3ffu);
    const uint32_t hj = right ? sons.y : sons.x;
    j += right;
    if (v <= (hj | 0x3ffu)) break;
    heap[k] = hj;
    k = j;
    j <<= 1;
  }
  heap[k] = v;
}
template <bool LAT>
__device__ __forceinline__ void t_down(uint32_t* heap, int heap_len, int k) {
  if (LAT) t_down_pf(heap, heap_len, k);
  else t_down_plain(heap, heap_len, k);
}

// trees.c build_tree + gen_bitlen + gen_codes (single thread)
// KIND: 0 lit/len, 1 dist, 2 bit-length
template <int KIND, bool LAT, int ELEMS>
__device__ int t_build_tree(TreesState* s, TreeArr<ELEMS>* t) {
  constexpr int max_length = KIND == 2 ? 7 : 15;
  constexpr int base = KIND == 0 ? 257 : 0;
  uint32_t* heap = s->heap;
  int n, max_code = -1, node;
  int heap_len = 0, heap_max = HEAP_SIZE;
  for (n = 0; n < ELEMS; n++) {
    if (t->freq[n] != 0) {
      heap[++heap_len] = t_entry(t->freq[n], 0, n);
      max_code = n;
    } else {
      t->len[n] = 0;
    }
  }
  while (heap_len < 2) {
    node = max_code < 2 ? ++max_code : 0;
    heap[++heap_len] = t_entry(1, 0, node);
    t->freq[node] = 1;
    s->opt_len--;
    if (KIND == 0) s->static_len -= c_z.sl_len[node];
    else if (KIND == 1) s->static_len -= 5;
  }
  heap[heap_len + 1] = 0xffffffffu;  // t_down_plain's right-son sentinel
  for (n = heap_len / 2; n >= 1; n--) t_down<LAT>(heap, heap_len, n);
  node = ELEMS;
  do {
    const uint32_t en = heap[1];
    heap[1] = heap[heap_len--];
    heap[heap_len + 1] = 0xffffffffu;
    t_down<LAT>(heap, heap_len, 1);
    const uint32_t em = heap[1];
    heap[--heap_max] = en;
    heap[--heap_max] = em;
    const uint32_t f = t_freq(en) + t_freq(em);
    const uint32_t d = max(t_depth(en), t_depth(em)) + 1;
    t->dad[t_node(en)] = t->dad[t_node(em)] = (uint16_t)node;
    heap[1] = t_entry(f & 0xffff, d, node);  // ush Freq, as in zlib
    node++;
    t_down<LAT>(heap, heap_len, 1);
  } while (heap_len >= 2);
  heap[--heap_max] = heap[1];

  int h, bits, overflow = 0;
  if (LAT) {
    // gen_bitlen (latency variant, few blocks).  The walk is serial through len[dad[n]]; the next entry's node and dad
    // are loaded an iteration ahead, and the sums and the length counts (16-bit fields of
    // four registers) stay in registers instead of read-modify-writes of shared memory.
    t->len[t_node(heap[heap_max])] = 0;
    uint64_t opt = s->opt_len, stat = s->static_len, blc[4] = {0, 0, 0, 0};
    h = heap_max + 1;
    uint32_t nn = h < (int)HEAP_SIZE ? t_node(heap[h]) : 0u;
    uint32_t dd = t->dad[nn];
    for (; h < (int)HEAP_SIZE; h++) {
      n = (int)nn;
      const uint32_t dad = dd;
      if (h + 1 < (int)HEAP_SIZE) {
        nn = t_node(heap[h + 1]);
        dd = t->dad[nn];
      }
      bits = t->len[dad] + 1;
      if (bits > max_length) bits = max_length, overflow++;
      t->len[n] = (uint8_t)bits;
      if (n > max_code) continue;
      const int q = bits >> 2;
      const uint64_t inc = 1ull << (16 * (bits & 3));
#pragma unroll
      for (int r = 0; r < 4; r++) blc[r] += q == r ? inc : 0ull;
      int xbits = 0;
      if (n >= base) xbits = KIND == 0 ? c_extra_lbits[n - base] : KIND == 1 ? c_extra_dbits[n - base] : c_extra_blbits[n - base];
      uint32_t f = t->freq[n];
      opt += (uint64_t)f * (uint32_t)(bits + xbits);
      if (KIND == 0) stat += (uint64_t)f * (uint32_t)(c_z.sl_len[n] + xbits);
      else if (KIND == 1) stat += (uint64_t)f * (uint32_t)(5 + xbits);
    }
    s->opt_len = opt;
    s->static_len = stat;
    for (bits = 0; bits <= 15; bits++) s->bl_count[bits] = (uint16_t)(blc[bits >> 2] >> (16 * (bits & 3)));
  } else {
    for (bits = 0; bits <= 15; bits++) s->bl_count[bits] = 0;
    t->len[t_node(heap[heap_max])] = 0;
    for (h = heap_max + 1; h < (int)HEAP_SIZE; h++) {
      n = t_node(heap[h]);
      bits = t->len[t->dad[n]] + 1;
      if (bits > max_length) bits = max_length, overflow++;
      t->len[n] = (uint8_t)bits;
      if (n > max_code) continue;
      s->bl_count[bits]++;
      int xbits = 0;
      if (n >= base) xbits = KIND == 0 ? c_extra_lbits[n - base] : KIND == 1 ? c_extra_dbits[n - base] : c_extra_blbits[n - base];
      uint32_t f = t->freq[n];
      s->opt_len += (uint64_t)f * (uint32_t)(bits + xbits);
      if (KIND == 0) s->static_len += (uint64_t)f * (uint32_t)(c_z.sl_len[n] + xbits);
      else if (KIND == 1) s->static_len += (uint64_t)f * (uint32_t)(5 + xbits);
    }
  }
  if (overflow) {
    do {
      bits = max_length - 1;
      while (s->bl_count[bits] == 0) bits--;
      s->bl_count[bits]--;
      s->bl_count[bits + 1] += 2;
      s->bl_count[max_length]--;
      overflow -= 2;
    } while (overflow > 0);
    for (bits = max_length; bits != 0; bits--) {
      n = s->bl_count[bits];
      while (n != 0) {
        int m = t_node(heap[--h]);
        if (m > max_code) continue;
        if ((uint32_t)t->len[m] != (uint32_t)bits) {
          s->opt_len += ((uint64_t)bits - t->len[m]) * t->freq[m];
          t->len[m] = (uint8_t)bits;
        }
        n--;
      }
    }
  }
  // gen_codes
  uint16_t next_code[16];
  uint32_t c = 0;
  for (bits = 1; bits <= 15; bits++) {
    c = (c + s->bl_count[bits - 1]) << 1;
    next_code[bits] = (uint16_t)c;
  }
  for (n = 0; n <= max_code; n++) {
    int l = t->len[n];
    if (l == 0) continue;
    t->code[n] = (uint16_t)(__brev((uint32_t)next_code[l]++) >> (32 - l));
  }
  return max_code;
}

template <int ELEMS>
__device__ void t_scan_tree(TreesState* s, TreeArr<ELEMS>* t, int max_code) {
  int prevlen = -1, curlen, nextlen = t->len[0], count = 0, max_count = 7, min_count = 4;
  if (nextlen == 0) max_count = 138, min_count = 3;
  t->len[max_code + 1] = 0xff;
  for (int n = 0; n <= max_code; n++) {
    curlen = nextlen;
    nextlen = t->len[n + 1];
    if (++count < max_count && curlen == nextlen) {
      continue;
    } else if (count < min_count) {
      s->blt.freq[curlen] += (uint16_t)count;
    } else if (curlen != 0) {
      if (curlen != prevlen) s->blt.freq[curlen]++;
      s->blt.freq[16]++;
    } else if (count <= 10) {
      s->blt.freq[17]++;
    } else {
      s->blt.freq[18]++;
    }
    count = 0;
    prevlen = curlen;
    if (nextlen == 0) max_count = 138, min_count = 3;
    else if (curlen == nextlen) max_count = 6, min_count = 3;
    else max_count = 7, min_count = 4;
  }
}

// little-endian bit writer into a block's header buffer
struct HdrWriter {
  uint32_t* w;
  uint32_t bits;
  __device__ void put(uint32_t v, uint32_t len) {
    if (!len) return;
    uint32_t i = bits >> 5, o = bits & 31;
    w[i] |= v << o;
    if (o + len > 32) w[i + 1] |= v >> (32 - o);
    bits += len;
  }
};

template <int ELEMS>
__device__ void t_send_tree(TreesState* s, TreeArr<ELEMS>* t, int max_code, HdrWriter& hw) {
  int prevlen = -1, curlen, nextlen = t->len[0], count = 0, max_count = 7, min_count = 4;
  if (nextlen == 0) max_count = 138, min_count = 3;
  TreeArr<BL_CODES>* bl = &s->blt;
  for (int n = 0; n <= max_code; n++) {
    curlen = nextlen;
    nextlen = t->len[n + 1];
    if (++count < max_count && curlen == nextlen) {
      continue;
    } else if (count < min_count) {
      do {
        hw.put(bl->code[curlen], bl->len[curlen]);
      } while (--count != 0);
    } else if (curlen != 0) {
      if (curlen != prevlen) {
        hw.put(bl->code[curlen], bl->len[curlen]);
        count--;
      }
      hw.put(bl->code[16], bl->len[16]);
      hw.put((uint32_t)(count - 3), 2);
    } else if (count <= 10) {
      hw.put(bl->code[17], bl->len[17]);
      hw.put((uint32_t)(count - 3), 3);
    } else {
      hw.put(bl->code[18], bl->len[18]);
      hw.put((uint32_t)(count - 11), 7);
    }
    count = 0;
    prevlen = curlen;
    if (nextlen == 0) max_count = 138, min_count = 3;
    else if (curlen == nextlen) max_count = 6, min_count = 3;
    else max_count = 7, min_count = 4;
  }
}

#ifndef BK_THREADS_OVR
constexpr int BK_THREADS = 32;  // one warp per block: measured 3.1 ms vs 4.8 ms with 64
#else
constexpr int BK_THREADS = BK_THREADS_OVR;
#endif

// NT threads per block: one warp when blocks are plentiful (register-limited occupancy);
// 256 threads with per-warp histograms when a call has few blocks (small lanes: the
// histogram of a block's 16383 symbols is then the latency of the whole stage)
template <int NT>
__global__ void __launch_bounds__(NT) k_blocks(const LaneDev* __restrict__ lanes,
                                                       const uint32_t* __restrict__ blk_lane,
                                                       uint32_t nblk_slots, const LaneSyms* __restrict__ ls,
                                                       const uint32_t* __restrict__ syms,
                                                       BlockInfo* __restrict__ info,
                                                       BlockCodes* __restrict__ codes,
                                                       uint32_t* __restrict__ hdr) {
  __shared__ TreesState S;
  __shared__ uint32_t hw_buf[HDR_BYTES / 4];
  __shared__ uint32_t s_len_sum, s_last_len, s_hdr_bits, s_stored;
  // symbol counts as packed u16 pairs (a block has <= 16383 symbols)
  constexpr int NW = NT / 32;
  __shared__ uint32_t h_l2w[NW][(L_CODES + 1) / 2], h_d2w[NW][(D_CODES + 1) / 2];
  uint32_t* h_l2 = h_l2w[threadIdx.x >> 5];  // this warp's histogram (merged into warp 0's below)
  uint32_t* h_d2 = h_d2w[threadIdx.x >> 5];
  auto h_l = [&](int i) -> uint32_t { return (h_l2w[0][i >> 1] >> (16 * (i & 1))) & 0xffff; };
  auto h_d = [&](int i) -> uint32_t { return (h_d2w[0][i >> 1] >> (16 * (i & 1))) & 0xffff; };
  uint32_t slot = blockIdx.x;
  if (slot >= nblk_slots) return;
  const uint32_t li = blk_lane[slot];
  const LaneDev Ld = lanes[li];
  const uint32_t b = slot - Ld.blk0;
  const LaneSyms L = ls[li];
  if (b >= L.nblk) {
    if (threadIdx.x == 0) info[slot].valid = 0;
    return;
  }
  const uint64_t s0 = (uint64_t)b * SYM_LIMIT;
  const uint64_t s1 = (b == L.nblk - 1) ? L.total : s0 + SYM_LIMIT;
  const uint32_t nsym = (uint32_t)(s1 - s0);
  // init (init_block: END_BLOCK freq 1)
  for (int i = threadIdx.x; i < (int)BL_CODES; i += blockDim.x) S.blt.freq[i] = 0;
  for (int i = threadIdx.x; i < NW * (int)(L_CODES + 1) / 2; i += blockDim.x) (&h_l2w[0][0])[i] = 0;
  for (int i = threadIdx.x; i < NW * (int)(D_CODES + 1) / 2; i += blockDim.x) (&h_d2w[0][0])[i] = 0;
  for (int i = threadIdx.x; i < (int)(HDR_BYTES / 4); i += blockDim.x) hw_buf[i] = 0;
  if (threadIdx.x == 0) {
    s_len_sum = 0;
    s_last_len = 0;
  }
  __syncthreads();
  const uint32_t* sy = syms + Ld.sym_base + s0;
  uint32_t local = 0;
  auto count = [&](uint32_t v) {
    if (v & SYM_MATCH) {
      uint32_t lc = v & 0xff, dist = (v >> 8) & 0x7fff;
      local += lc + 3;
      const uint32_t li = c_z.length_code[lc] + 257, di = d_code(dist);
      atomicAdd(&h_l2[li >> 1], 1u << (16 * (li & 1)));
      atomicAdd(&h_d2[di >> 1], 1u << (16 * (di & 1)));
    } else {
      local += 1;
      const uint32_t li = v & 0xff;
      atomicAdd(&h_l2[li >> 1], 1u << (16 * (li & 1)));
    }
  };
  {
    // four independent loads in flight per thread (the symbol stream comes from DRAM)
    uint32_t i = threadIdx.x;
    for (; i + 3 * NT < nsym; i += 4 * NT) {
      const uint32_t v0 = __ldg(sy + i), v1 = __ldg(sy + i + NT), v2 = __ldg(sy + i + 2 * NT),
                     v3 = __ldg(sy + i + 3 * NT);
      count(v0), count(v1), count(v2), count(v3);
    }
    for (; i < nsym; i += NT) count(__ldg(sy + i));
    if (threadIdx.x == 0 && nsym) s_last_len = sym_len(__ldg(sy + nsym - 1));
  }
  // reduce stored length
  for (int o = 16; o; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&s_len_sum, local);
  __syncthreads();
  if (NW > 1) {  // merge the per-warp counts (packed u16 pairs: a block has <= 16383 symbols)
    for (int i = threadIdx.x; i < (int)(L_CODES + 1) / 2; i += blockDim.x) {
      uint32_t v = 0;
      for (int w = 1; w < NW; w++) v += h_l2w[w][i];
      h_l2w[0][i] += v;
    }
    for (int i = threadIdx.x; i < (int)(D_CODES + 1) / 2; i += blockDim.x) {
      uint32_t v = 0;
      for (int w = 1; w < NW; w++) v += h_d2w[w][i];
      h_d2w[0][i] += v;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < (int)L_CODES; i += blockDim.x) S.lt.freq[i] = (uint16_t)(h_l(i) + (i == 256));
  for (int i = threadIdx.x; i < (int)D_CODES; i += blockDim.x) S.dt.freq[i] = (uint16_t)h_d(i);
  __syncthreads();
  if (threadIdx.x == 0) {
    S.opt_len = 0;
    S.static_len = 0;
    S.lmax = t_build_tree<0, (NT > 32)>(&S, &S.lt);
    S.dmax = t_build_tree<1, (NT > 32)>(&S, &S.dt);
    t_scan_tree(&S, &S.lt, S.lmax);
    t_scan_tree(&S, &S.dt, S.dmax);
    t_build_tree<2, (NT > 32)>(&S, &S.blt);
    int max_blindex;
    for (max_blindex = BL_CODES - 1; max_blindex >= 3; max_blindex--)
      if (S.blt.len[c_bl_order[max_blindex]] != 0) break;
    S.opt_len += 3 * ((uint64_t)max_blindex + 1) + 5 + 5 + 4;
    S.blmax = max_blindex;
    uint64_t opt_lenb = (S.opt_len + 3 + 7) >> 3;
    uint64_t static_lenb = (S.static_len + 3 + 7) >> 3;
    // A block k_layout will certainly store (_tr_flush_block's rule, with the block start provably
    // still in the window: <= 32000 bytes and >= 262 symbols, hence bytes, after it -- see k_layout's
    // buf_ok) needs no tree description, code tables or size sums (the mantissa planes' blocks).
    const bool stored = s_len_sum <= 32000 && L.total - s1 >= 262 &&
                        (uint64_t)s_len_sum + 4 <= umin64(opt_lenb, static_lenb);
    HdrWriter hw{hw_buf, 0};
    if (!stored) {  // dynamic header (send_all_trees)
      hw.put((uint32_t)(S.lmax + 1 - 257), 5);
      hw.put((uint32_t)(S.dmax + 1 - 1), 5);
      hw.put((uint32_t)(max_blindex + 1 - 4), 4);
      for (int r = 0; r < max_blindex + 1; r++) hw.put(S.blt.len[c_bl_order[r]], 3);
      t_send_tree(&S, &S.lt, S.lmax, hw);
      t_send_tree(&S, &S.dt, S.dmax, hw);
    }
    BlockInfo bi;
    bi.sym0 = s0;
    bi.nsym = nsym;
    bi.stored_len = s_len_sum;
    bi.last_len = s_last_len;
    bi.opt_lenb = (uint32_t)umin64(opt_lenb, 0xffffffffu);
    bi.static_lenb = (uint32_t)umin64(static_lenb, 0xffffffffu);
    bi.hdr_bits = hw.bits;
    bi.dyn_bits = bi.static_bits = 0;
    bi.valid = 1;
    info[slot] = bi;
    s_hdr_bits = hw.bits;
    s_stored = stored;
  }
  __syncthreads();
  if (s_stored) return;
  // codes to global; exact bit sizes: sum over codes of freq * (len + extra)
  BlockCodes* bc = codes + slot;
  // (freq of internal/forced nodes is irrelevant: only real symbols are counted)
  __shared__ unsigned long long dyn_sum, sta_sum;
  if (threadIdx.x == 0) dyn_sum = sta_sum = 0;
  __syncthreads();
  unsigned long long dsum = 0, ssum = 0;
  for (int i = threadIdx.x; i < (int)L_CODES; i += blockDim.x) {
    bc->l[i] = (uint32_t)S.lt.code[i] | ((uint32_t)S.lt.len[i] << 16);
  }
  for (int i = threadIdx.x; i < (int)D_CODES; i += blockDim.x) {
    bc->d[i] = (uint32_t)S.dt.code[i] | ((uint32_t)S.dt.len[i] << 16);
  }
  // exact sizes from the symbol histograms (the real counts h_l / h_d, so the
  // frequency-1 nodes build_tree forces into sparse trees are not counted)
  for (int i = threadIdx.x; i < (int)L_CODES; i += blockDim.x) {
    const uint32_t f = h_l(i);
    if (!f) continue;
    const uint32_t x = i >= 257 ? c_extra_lbits[i - 257] : 0;
    dsum += (unsigned long long)f * (S.lt.len[i] + x);
    ssum += (unsigned long long)f * (c_z.sl_len[i] + x);
  }
  for (int i = threadIdx.x; i < (int)D_CODES; i += blockDim.x) {
    const uint32_t f = h_d(i);
    if (!f) continue;
    const uint32_t x = c_extra_dbits[i];
    dsum += (unsigned long long)f * (S.dt.len[i] + x);
    ssum += (unsigned long long)f * (5 + x);
  }
  for (int o = 16; o; o >>= 1) {
    dsum += __shfl_down_sync(0xffffffffu, dsum, o);
    ssum += __shfl_down_sync(0xffffffffu, ssum, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&dyn_sum, dsum);
    atomicAdd(&sta_sum, ssum);
  }
  uint32_t* hb = hdr + (uint64_t)slot * (HDR_BYTES / 4);
  for (int i = threadIdx.x; i < (int)(HDR_BYTES / 4); i += blockDim.x) hb[i] = hw_buf[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t hbits = s_hdr_bits;
    info[slot].dyn_bits = (uint32_t)(3 + hbits + dyn_sum + S.lt.len[256]);
    info[slot].static_bits = (uint32_t)(3 + sta_sum + 7);
  }
}

// ---------------------------------------------------------------------------
// K6d: per-lane layout: _tr_flush_block's decision + bit offsets.  One warp per
// lane; block records are fetched 32 at a time and broadcast by shuffle.
struct BlockPlan {
  uint64_t bit_off;     // lane-blob-relative bit offset of the block's 3-bit header
  uint64_t byte_start;  // input position of the block's first byte
  uint32_t type;        // 0 stored, 1 static, 2 dynamic
  uint32_t last;
};

__global__ void k_layout(const LaneDev* __restrict__ lanes, int nlanes, const LaneSyms* __restrict__ ls,
                         const BlockInfo* __restrict__ info, BlockPlan* __restrict__ plan,
                         uint64_t* __restrict__ blob_len) {
  int li = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (li >= nlanes) return;
  const int lane = threadIdx.x & 31;
  const LaneDev Ld = lanes[li];
  const uint32_t nb = ls[li].nblk;
  uint64_t bit = 16;  // after the 2-byte zlib header
  uint64_t pos = 0;
  for (uint32_t base = 0; base < nb; base += 32) {
    uint32_t b = base + lane;
    BlockInfo bi = {};
    if (b < nb) bi = info[Ld.blk0 + b];
    uint32_t cnt = min(32u, nb - base);
    uint32_t my_type = 0, my_last = 0;
    uint64_t my_bit = 0, my_pos = 0;
    for (uint32_t i = 0; i < cnt; i++) {
      uint32_t stored_len = __shfl_sync(0xffffffffu, bi.stored_len, i);
      uint32_t last_len = __shfl_sync(0xffffffffu, bi.last_len, i);
      uint32_t opt_lenb = __shfl_sync(0xffffffffu, bi.opt_lenb, i);
      uint32_t static_lenb = __shfl_sync(0xffffffffu, bi.static_lenb, i);
      uint32_t dyn_bits = __shfl_sync(0xffffffffu, bi.dyn_bits, i);
      uint32_t static_bits = __shfl_sync(0xffffffffu, bi.static_bits, i);
      const bool last = base + i == nb - 1;
      // slides done by fill_window at or before the flush's loop top
      uint64_t tf = last ? Ld.n : pos + stored_len - last_len + 1;
      bool buf_ok = pos >= (uint64_t)WSIZE * slides_at(tf, Ld.n);
      uint64_t olb = opt_lenb;
      if ((uint64_t)static_lenb <= olb) olb = static_lenb;
      uint32_t type;
      uint64_t sz;
      if ((uint64_t)stored_len + 4 <= olb && buf_ok) {
        type = 0;
        uint64_t after_hdr = bit + 3;
        sz = ((after_hdr + 7) & ~uint64_t(7)) - bit + 32 + 8ull * stored_len;
      } else if ((uint64_t)static_lenb == olb) {
        type = 1;
        sz = static_bits;
      } else {
        type = 2;
        sz = dyn_bits;
      }
      if (lane == (int)i) {
        my_type = type;
        my_last = last;
        my_bit = bit;
        my_pos = pos;
      }
      bit += sz;
      pos += stored_len;
    }
    if (b < nb) plan[Ld.blk0 + b] = BlockPlan{my_bit, my_pos, my_type, my_last};
  }
  if (lane == 0) blob_len[li] = ((bit + 7) >> 3) + 4;
}

// ---------------------------------------------------------------------------
// Placement: lane blob pointers inside their containers; capacity checks.
struct ContainerDev {
  uint8_t* dst;
  uint64_t cap;
  uint64_t count;
  int split;  // 1 split, 0 raw, -1 bare blob (no BBC1 header)
  int lane0;  // first lane (slot 0); slot 1 = lane0 + 1 when split
};

__global__ void k_place(const ContainerDev* __restrict__ cons, int ncons, const uint64_t* __restrict__ blob_len,
                        uint8_t** __restrict__ lane_out, uint64_t* __restrict__ con_len,
                        int* __restrict__ con_status) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncons) return;
  ContainerDev C = cons[c];
  uint64_t hdr = C.split < 0 ? 0 : BB_CONTAINER_HEADER;
  uint64_t hl = blob_len[C.lane0];
  uint64_t ll = C.split == 1 ? blob_len[C.lane0 + 1] : 0;
  uint64_t total = hdr + hl + ll;
  con_len[c] = total;
  bool ok = total <= C.cap;
  con_status[c] = ok ? BB_OK : BB_INVALID_ARG;
  lane_out[C.lane0] = ok ? C.dst + hdr : nullptr;
  if (C.split == 1) lane_out[C.lane0 + 1] = ok ? C.dst + hdr + hl : nullptr;
}

// ---------------------------------------------------------------------------
// K7: bit packing.  One CTA per block; symbols in chunks of 2048 (8 per
// thread): bit lengths -> block scan -> shared-memory staging with atomicOr ->
// complete words stored; the block's shared edge words merged by k_edges.
constexpr int EM_THREADS = 256, EM_PER = 8, EM_CHUNK = EM_THREADS * EM_PER;
constexpr int EM_WORDS = (EM_CHUNK * 48) / 32 + 4;

__device__ __forceinline__ void sym_bits(uint32_t v, const uint32_t* lcodes, const uint32_t* dcodes,
                                         bool stat, uint64_t& bits, uint32_t& len) {
  if (v & SYM_MATCH) {
    uint32_t lc = v & 0xff, dist = (v >> 8) & 0x7fff;
    uint32_t code = c_z.length_code[lc];
    uint32_t lcd, lln;
    if (stat) lcd = c_z.sl_code[code + 257], lln = c_z.sl_len[code + 257];
    else lcd = lcodes[code + 257] & 0xffff, lln = lcodes[code + 257] >> 16;
    bits = lcd;
    len = lln;
    uint32_t xl = c_extra_lbits[code];
    if (xl) {
      bits |= (uint64_t)(lc - c_z.base_length[code]) << len;
      len += xl;
    }
    uint32_t dc = d_code(dist);
    uint32_t dcd, dln;
    if (stat) dcd = c_z.sd_code[dc], dln = 5;
    else dcd = dcodes[dc] & 0xffff, dln = dcodes[dc] >> 16;
    bits |= (uint64_t)dcd << len;
    len += dln;
    uint32_t xd = c_extra_dbits[dc];
    if (xd) {
      bits |= (uint64_t)(dist - c_z.base_dist[dc]) << len;
      len += xd;
    }
  } else {
    uint32_t c = v & 0xff;
    if (stat) bits = c_z.sl_code[c], len = c_z.sl_len[c];
    else bits = lcodes[c] & 0xffff, len = lcodes[c] >> 16;
  }
}

// Global writes of K7 are plain 32-bit stores of words a block owns entirely.  The block's first
// word (when it starts mid-word, it holds the previous block's tail) and its last word (when it
// ends mid-word) are not stored: their block-owned bits go to edge[2 * slot + {0, 1}] as
// (word index relative to the lane's word base, value), and k_edges ORs the contributions that
// land on the same word and stores each word once.  Nothing is pre-zeroed and no global atomics
// are issued, so when the container lives in the next GPU's HBM (fused hand-off) every container
// byte crosses NVLink once.
constexpr uint32_t EDGE_NONE = 0xffffffffu;

__global__ void __launch_bounds__(EM_THREADS) k_emit(const LaneDev* __restrict__ lanes,
                                                     const uint32_t* __restrict__ blk_lane, uint32_t nblk_slots,
                                                     const LaneSyms* __restrict__ ls,
                                                     const BlockInfo* __restrict__ info,
                                                     const BlockPlan* __restrict__ plan,
                                                     const BlockCodes* __restrict__ codes,
                                                     const uint32_t* __restrict__ hdr,
                                                     const uint32_t* __restrict__ syms,
                                                     uint8_t* const* __restrict__ lane_out,
                                                     uint2* __restrict__ edge) {
  typedef cub::BlockScan<uint32_t, EM_THREADS> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint32_t stage[EM_WORDS];
  __shared__ uint32_t s_l[L_CODES], s_d[D_CODES];
  __shared__ uint32_t s_carry;  // the block's partial word left by the previous piece
  __shared__ uint2 s_lo;        // the block's first-word contribution
  const uint32_t slot = blockIdx.x;
  if (slot >= nblk_slots) return;
  const uint32_t li = blk_lane[slot];
  const LaneDev Ld = lanes[li];
  const uint32_t b = slot - Ld.blk0;
  if (b >= ls[li].nblk) return;
  uint8_t* out = lane_out[li];
  if (!out) return;
  const BlockInfo bi = info[slot];
  const BlockPlan pl = plan[slot];
  // word-aligned base for the lane blob
  uintptr_t a = reinterpret_cast<uintptr_t>(out);
  uint32_t* wbase = reinterpret_cast<uint32_t*>(a & ~uintptr_t(3));
  const uint64_t bit0 = 8ull * (a & 3) + pl.bit_off;
  const uint64_t wf = bit0 >> 5;
  const bool first_shared = (bit0 & 31) != 0;
  const uint32_t hdr3 = (pl.type << 1) | pl.last;
  if (pl.type == 0) {
    // stored: 3 header bits, pad to a byte, LEN, NLEN, raw bytes; bytes [B, E) relative to wbase
    const uint64_t B = (bit0 + 3 + 7) >> 3;
    const uint32_t len = bi.stored_len;
    const uint32_t hdr4 = (len & 0xffff) | ((~len & 0xffff) << 16);
    const uint8_t* src = Ld.src + pl.byte_start;
    const uint64_t E = B + 4 + len;
    const uint64_t wl = (E - 1) >> 2;
    const bool last_shared = (E & 3) != 0;
    const uintptr_t src_end = reinterpret_cast<uintptr_t>(src) + len;
    for (uint64_t wi = wf + threadIdx.x; wi <= wl; wi += blockDim.x) {
      uint32_t v = 0;
      bool done = false;
      if (4 * wi >= B + 4 && 4 * wi + 4 <= E) {  // interior: four input bytes, two aligned loads
        const uintptr_t ua = reinterpret_cast<uintptr_t>(src) + (4 * wi - B - 4);
        const uintptr_t base = ua & ~uintptr_t(3);
        if (base + 8 <= src_end) {
          const uint32_t lo = __ldg(reinterpret_cast<const uint32_t*>(base));
          const uint32_t hi = __ldg(reinterpret_cast<const uint32_t*>(base) + 1);
          v = __funnelshift_r(lo, hi, 8 * (uint32_t)(ua & 3));
          done = true;
        }
      }
      if (!done) {
        for (int k = 0; k < 4; k++) {
          const uint64_t ob = 4 * wi + k;
          if (ob < B || ob >= E) continue;
          const uint64_t r = ob - B;
          const uint32_t byte_v = r < 4 ? (hdr4 >> (8 * r)) & 0xff : src[r - 4];
          v |= byte_v << (8 * k);
        }
      }
      // the 3 header bits (then zero padding up to B); they straddle into word wf + 1 from bit 30 on
      if (wi == wf) v |= hdr3 << (bit0 & 31);
      if (wi == wf + 1 && (bit0 & 31) > 29) v |= hdr3 >> (32 - (bit0 & 31));
      const bool is_lo = wi == wf && first_shared, is_hi = wi == wl && last_shared;
      if (is_lo) edge[2 * slot] = make_uint2((uint32_t)wi, v);
      else if (is_hi) edge[2 * slot + 1] = make_uint2((uint32_t)wi, v);
      else wbase[wi] = v;
    }
    if (threadIdx.x == 0) {
      if (!first_shared) edge[2 * slot] = make_uint2(EDGE_NONE, 0);
      if (!last_shared || (wl == wf && first_shared)) edge[2 * slot + 1] = make_uint2(EDGE_NONE, 0);
    }
    return;
  }
  const bool stat = pl.type == 1;
  const BlockCodes* bc = codes + slot;
  for (int i = threadIdx.x; i < (int)L_CODES; i += blockDim.x) s_l[i] = bc->l[i];
  for (int i = threadIdx.x; i < (int)D_CODES; i += blockDim.x) s_d[i] = bc->d[i];
  if (threadIdx.x == 0) {
    s_carry = 0;
    s_lo = make_uint2(EDGE_NONE, 0);
  }
  // writes staged words [0, nwords) of a piece starting at absolute bit cbit (piece_bits long):
  // complete words are stored (the shared first word becomes the lo contribution), a partial last
  // word becomes the carry for the next piece
  auto flush = [&](uint64_t cbit, uint32_t piece_bits) {
    const uint32_t sh = (uint32_t)(cbit & 31);
    const uint32_t nwords = (sh + piece_bits + 31) >> 5;
    const bool partial_end = ((sh + piece_bits) & 31) != 0;
    for (uint32_t i = threadIdx.x; i < nwords; i += blockDim.x) {
      const uint64_t aw = (cbit >> 5) + i;
      if (i == nwords - 1 && partial_end) s_carry = stage[i];
      else if (aw == wf && first_shared) s_lo = make_uint2((uint32_t)aw, stage[i]);
      else wbase[aw] = stage[i];
    }
  };
  uint64_t bit = bit0;
  __syncthreads();
  {
    // piece 0: the block header and (dynamic) the tree description, staged like a symbol chunk
    const uint32_t hbits = stat ? 0u : bi.hdr_bits;
    const uint32_t sh = (uint32_t)(bit & 31);
    const uint32_t nwords = (sh + 3 + hbits + 31) >> 5;
    for (uint32_t i = threadIdx.x; i < nwords + 1; i += blockDim.x) stage[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicOr(&stage[0], hdr3 << sh);
      if (sh > 29) atomicOr(&stage[1], hdr3 >> (32 - sh));  // the header straddles a word
    }
    const uint32_t* hb = hdr + (uint64_t)slot * (HDR_BYTES / 4);
    for (uint32_t i = threadIdx.x; i * 32 < hbits; i += blockDim.x) {
      const uint32_t l = min(32u, hbits - i * 32);
      uint64_t v = hb[i];
      if (l < 32) v &= (1ull << l) - 1;
      const uint32_t o = sh + 3 + 32 * i, wi = o >> 5, ob = o & 31;
      atomicOr(&stage[wi], (uint32_t)(v << ob));
      if (ob + l > 32) atomicOr(&stage[wi + 1], (uint32_t)(v >> (32 - ob)));
    }
    __syncthreads();
    flush(bit, 3 + hbits);
    bit += 3 + hbits;
    __syncthreads();
  }
  const uint32_t* sy = syms + Ld.sym_base + bi.sym0;
  const uint32_t total = bi.nsym + 1;  // + END_BLOCK
  const uint32_t eob_code = stat ? c_z.sl_code[256] : (s_l[256] & 0xffff);
  const uint32_t eob_len = stat ? 7 : (s_l[256] >> 16);
  for (uint32_t c0 = 0; c0 < total; c0 += EM_CHUNK) {
    uint64_t vb[EM_PER];
    uint32_t vl[EM_PER];
    uint32_t tlen = 0;
#pragma unroll
    for (int k = 0; k < EM_PER; k++) {
      uint32_t i = c0 + threadIdx.x * EM_PER + k;
      vb[k] = 0;
      vl[k] = 0;
      if (i < bi.nsym) {
        sym_bits(sy[i], s_l, s_d, stat, vb[k], vl[k]);
      } else if (i == bi.nsym) {
        vb[k] = eob_code;
        vl[k] = eob_len;
      }
      tlen += vl[k];
    }
    uint32_t toff, chunk_bits;
    Scan(tmp).ExclusiveSum(tlen, toff, chunk_bits);
    const uint64_t cbit = bit;  // chunk start (absolute, rel. wbase)
    const uint32_t sh = (uint32_t)(cbit & 31);
    const uint32_t nwords = (sh + chunk_bits + 31) >> 5;
    for (uint32_t i = threadIdx.x; i < nwords; i += blockDim.x) stage[i] = (i == 0 && sh) ? s_carry : 0u;
    __syncthreads();
    uint32_t o = sh + toff;
#pragma unroll
    for (int k = 0; k < EM_PER; k++) {
      if (vl[k]) {
        uint32_t wi = o >> 5, ob = o & 31;
        atomicOr(&stage[wi], (uint32_t)(vb[k] << ob));
        if (ob + vl[k] > 32) atomicOr(&stage[wi + 1], (uint32_t)(vb[k] >> (32 - ob)));
        if (ob + vl[k] > 64) atomicOr(&stage[wi + 2], (uint32_t)(vb[k] >> (64 - ob)));
        o += vl[k];
      }
    }
    __syncthreads();
    flush(cbit, chunk_bits);
    bit += chunk_bits;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    // the block's last word: partial iff the block ends mid-word (then it is the carry)
    uint2 hi = make_uint2(EDGE_NONE, 0);
    uint2 lo = s_lo;
    if (bit & 31) {
      const uint64_t wl = (bit - 1) >> 5;
      if (wl == wf && first_shared) lo = make_uint2((uint32_t)wl, s_carry);
      else hi = make_uint2((uint32_t)wl, s_carry);
    }
    edge[2 * slot] = lo;
    edge[2 * slot + 1] = hi;
  }
}

// one thread per edge contribution; the first contribution of each word ORs the run of
// contributions to that word (blocks are contiguous, so they are adjacent in slot order) and
// stores it
__global__ void k_edges(const LaneDev* __restrict__ lanes, const uint32_t* __restrict__ blk_lane,
                        uint32_t nblk_slots, const LaneSyms* __restrict__ ls, uint8_t* const* __restrict__ lane_out,
                        const uint2* __restrict__ edge) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t slot = t >> 1;
  if (slot >= nblk_slots) return;
  const uint32_t li = blk_lane[slot];
  const LaneDev Ld = lanes[li];
  const uint32_t nb = ls[li].nblk;
  if (slot - Ld.blk0 >= nb) return;
  uint8_t* out = lane_out[li];
  if (!out) return;
  const uint2 me = edge[t];
  if (me.x == EDGE_NONE) return;
  const uint32_t t0 = 2 * Ld.blk0, t1 = 2 * (Ld.blk0 + nb);  // this lane's contributions
  for (uint32_t u = t; u-- > t0;) {  // an earlier contribution to the same word owns it
    const uint32_t x = edge[u].x;
    if (x == EDGE_NONE) continue;
    if (x == me.x) return;
    break;
  }
  uint32_t v = me.y;
  for (uint32_t u = t + 1; u < t1; u++) {
    const uint2 c = edge[u];
    if (c.x == EDGE_NONE) continue;
    if (c.x != me.x) break;
    v |= c.y;
  }
  uint32_t* wbase = reinterpret_cast<uint32_t*>(reinterpret_cast<uintptr_t>(out) & ~uintptr_t(3));
  wbase[me.x] = v;
}

// ---------------------------------------------------------------------------
// Adler-32: (A, B, m) per piece with A = sum x, B = sum (m - j) x_j over a
// piece of m bytes; concatenation: A = A1 + A2, B = B1 + B2 + m2 * A1.
constexpr uint32_t MOD = 65521;
constexpr int AD_THREADS = 256, AD_BYTES = 256;  // 64 KiB per CTA
constexpr uint64_t AD_CHUNK = (uint64_t)AD_THREADS * AD_BYTES;

struct Adl {
  uint32_t A, B;
  uint64_t m;
};

__device__ __forceinline__ Adl adl_cat(Adl l, Adl r) {
  Adl o;
  o.A = (l.A + r.A) % MOD;
  o.B = (uint32_t)(((uint64_t)l.B + r.B + (r.m % MOD) * l.A) % MOD);
  o.m = l.m + r.m;
  return o;
}

__device__ Adl adl_warp(Adl v) {
  // ordered reduction: lane i holds piece i; result in lane 0
  for (int off = 1; off < 32; off <<= 1) {
    Adl r;
    r.A = __shfl_down_sync(0xffffffffu, v.A, off);
    r.B = __shfl_down_sync(0xffffffffu, v.B, off);
    r.m = __shfl_down_sync(0xffffffffu, v.m, off);
    if ((threadIdx.x & 31) + off < 32 && ((threadIdx.x & 31) & (2 * off - 1)) == 0) v = adl_cat(v, r);
  }
  return v;
}

__global__ void __launch_bounds__(AD_THREADS) k_adler_chunks(const LaneDev* __restrict__ lanes,
                                                             const WorkItem* __restrict__ work,
                                                             Adl* __restrict__ partial) {
  __shared__ Adl wres[AD_THREADS / 32];
  const WorkItem w = work[blockIdx.x];
  const LaneDev Ld = lanes[w.lane];
  const uint64_t s = (uint64_t)w.start;  // chunk index within the lane
  const uint64_t c0 = s * AD_CHUNK + (uint64_t)threadIdx.x * AD_BYTES;
  uint32_t A = 0, B = 0;
  uint64_t m = 0;
  if (c0 < Ld.n) {
    uint64_t c1 = umin64(c0 + AD_BYTES, Ld.n);
    m = c1 - c0;
    const uint8_t* p = Ld.src + c0;
    uint32_t i = 0;
    if (m == AD_BYTES) {
      for (; i < AD_BYTES; i += 16) {
        uint32_t v[4];
        gather16(p + i, v);
        // sum x_k and sum k x_k over the 16 bytes: B += sum (m - i - k) x_k
        const uint32_t sx = __dp4a(v[0], 0x01010101u, __dp4a(v[1], 0x01010101u, __dp4a(v[2], 0x01010101u, __dp4a(v[3], 0x01010101u, 0u))));
        const uint32_t kx = __dp4a(v[0], 0x03020100u, __dp4a(v[1], 0x07060504u, __dp4a(v[2], 0x0b0a0908u, __dp4a(v[3], 0x0f0e0d0cu, 0u))));
        A += sx;
        B += (uint64_t)(m - i) * sx - kx;
      }
    } else {
      for (; i < m; i++) {
        uint32_t x = p[i];
        A += x;
        B += (uint32_t)(m - i) * x;
      }
    }
    A %= MOD;
    B %= MOD;
  }
  Adl v{A, B, m};
  v = adl_warp(v);
  if ((threadIdx.x & 31) == 0) wres[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    Adl u = threadIdx.x < AD_THREADS / 32 ? wres[threadIdx.x] : Adl{0, 0, 0};
    u = adl_warp(u);
    if (threadIdx.x == 0) partial[blockIdx.x] = u;
  }
}

// per lane: ordered reduction of chunk partials, zlib header + trailer
__global__ void k_adler_final(const LaneDev* __restrict__ lanes, int nlanes, const uint32_t* __restrict__ chunk0,
                              const Adl* __restrict__ partial, uint8_t* const* __restrict__ lane_out,
                              const uint64_t* __restrict__ blob_len) {
  int li = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (li >= nlanes) return;
  const int lane = threadIdx.x & 31;
  const LaneDev Ld = lanes[li];
  const uint32_t nch = (uint32_t)((Ld.n + AD_CHUNK - 1) / AD_CHUNK);
  Adl acc{0, 0, 0};
  for (uint32_t base = 0; base < nch; base += 32) {
    Adl v = base + lane < nch ? partial[chunk0[li] + base + lane] : Adl{0, 0, 0};
    v = adl_warp(v);
    acc = adl_cat(acc, Adl{__shfl_sync(0xffffffffu, v.A, 0), __shfl_sync(0xffffffffu, v.B, 0),
                           __shfl_sync(0xffffffffu, v.m, 0)});
  }
  if (lane != 0) return;
  uint8_t* out = lane_out[li];
  if (!out) return;
  uint32_t a = (1 + acc.A) % MOD;
  uint32_t b = (uint32_t)((Ld.n % MOD + acc.B) % MOD);
  uint32_t ad = (b << 16) | a;
  // zlib header 78 9C and the big-endian Adler-32 trailer, as byte stores (they share words with the
  // blocks' edge words and the container header, all written by earlier kernels)
  out[0] = 0x78;
  out[1] = 0x9c;
  uint8_t* tail = out + blob_len[li] - 4;
  tail[0] = (uint8_t)(ad >> 24);
  tail[1] = (uint8_t)(ad >> 16);
  tail[2] = (uint8_t)(ad >> 8);
  tail[3] = (uint8_t)ad;
}

__global__ void k_container_header(const ContainerDev* __restrict__ cons, int ncons,
                                   const uint64_t* __restrict__ blob_len, const int* __restrict__ con_status) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncons) return;
  ContainerDev C = cons[c];
  if (C.split < 0 || con_status[c] != BB_OK) return;
  uint64_t hl = blob_len[C.lane0], ll = C.split == 1 ? blob_len[C.lane0 + 1] : 0;
  uint8_t h[BB_CONTAINER_HEADER];
  h[0] = 'B', h[1] = 'B', h[2] = 'C', h[3] = '1', h[4] = 1, h[5] = BB_BACKEND_DEFLATE;
  h[6] = C.split ? 1 : 0;
  for (int i = 0; i < 8; i++) {
    h[7 + i] = (uint8_t)(C.count >> (8 * i));
    h[15 + i] = (uint8_t)(hl >> (8 * i));
    h[23 + i] = (uint8_t)(ll >> (8 * i));
  }
  for (int i = 0; i < BB_CONTAINER_HEADER; i++) C.dst[i] = h[i];
}

}  // namespace


// K3 launcher (key generation, CUB onesweep radix sort, link scatter)
// ---------------------------------------------------------------------------
// host orchestration

struct DeflateEngine {
  Workspace ws;
  Workspace sortws;  // K3's per-segment final head tables
  bool tables_ready = false;
  uint64_t* h_pinned = nullptr;  // small pinned scratch for results
  size_t h_pinned_cap = 0;
};

DeflateEngine* deflate_engine_create() { return new DeflateEngine(); }

void deflate_engine_destroy(DeflateEngine* e) {
  if (!e) return;
  if (e->h_pinned) cudaFreeHost(e->h_pinned);
  delete e;
}

static int pinned(DeflateEngine* e, size_t bytes) {
  if (bytes <= e->h_pinned_cap) return BB_OK;
  if (e->h_pinned) cudaFreeHost(e->h_pinned);
  e->h_pinned = nullptr;
  size_t want = std::max<size_t>(bytes, 1 << 16);
  BB_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&e->h_pinned), want, cudaHostAllocDefault));
  e->h_pinned_cap = want;
  return BB_OK;
}

int deflate_containers(DeflateEngine* e, const std::vector<LaneJob>& jobs,
                       const std::vector<ContainerJob>& containers, cudaStream_t st, uint64_t* container_len,
                       int* container_status) {
  if (!e->tables_ready) {
    ZTables t = make_tables();
    BB_CUDA_TRY(cudaMemcpyToSymbol(c_z, &t, sizeof t));
    BB_CUDA_TRY(cudaFuncSetAttribute(k_hash_prev6, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    BB_CUDA_TRY(cudaFuncSetAttribute(k_hash_prev7, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  BB_CUDA_TRY(cudaFuncSetAttribute(k_hash_prev8, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    BB_CUDA_TRY(cudaFuncSetAttribute(k_profile3, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * PF_WIN + 16));
    BB_CUDA_TRY(cudaFuncSetAttribute(k_gram4, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * PF_WIN + 16));
    BB_CUDA_TRY(cudaFuncSetAttribute(k_profile4, cudaFuncAttributeMaxDynamicSharedMemorySize, PF2_SMEM + 16));
    e->tables_ready = true;
  }
  const int nl = (int)jobs.size();
  const int nc = (int)containers.size();
  if (nl == 0) return BB_OK;
  // lanes ordered by container/slot so slot 1 == lane0 + 1
  std::vector<int> order(nl);
  for (int i = 0; i < nl; i++) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    if (jobs[a].container != jobs[b].container) return jobs[a].container < jobs[b].container;
    return jobs[a].slot < jobs[b].slot;
  });
  std::vector<LaneDev> L(nl);
  std::vector<ContainerDev> C(nc);
  for (int c = 0; c < nc; c++) {
    C[c] = ContainerDev{containers[c].dst, containers[c].cap, containers[c].element_count,
                        containers[c].split, -1};
  }
  std::vector<WorkItem> hp_work, pf_work, pf2_work, ad_work;
  std::vector<uint32_t> seg_lane, blk_lane, ad_chunk0(nl);
  uint64_t pos_total = 0, sym_total = 0;
  uint32_t seg_total = 0, blk_total = 0;
  uint32_t maxG = 0;
  for (int i = 0; i < nl; i++) {
    const LaneJob& j = jobs[order[i]];
    if (j.n >= (1ull << 32) - 1) {
      set_error("deflate lane of %llu bytes exceeds 4 GiB - 2", (unsigned long long)j.n);
      return BB_ERROR;
    }
    LaneDev d;
    d.src = j.src;
    d.n = j.n;
    d.pbase = pos_total;
#ifndef K5_G_BIG
#define K5_G_BIG 4096
#endif
#ifndef K5_G_SMALL
#define K5_G_SMALL 128  // config1: parse 0.192 -> 0.116 ms (64: 0.092 ms but more fix-up, 2.431 vs 2.376 ms per round trip)
#endif
    d.G = j.n <= (1u << 20) ? K5_G_SMALL : j.n <= (4u << 20) ? 1024 : K5_G_BIG;  // small lanes: more, shorter parse segments
    d.seg0 = seg_total;
    d.nseg = (uint32_t)std::max<uint64_t>(1, (j.n + d.G - 1) / d.G);
    d.blk0 = blk_total;
    d.nblk_max = (uint32_t)(j.n / SYM_LIMIT + 2);
    d.sym_base = sym_total;
    d.container = j.container;
    d.slot = j.slot;
    if (j.slot == 0) C[j.container].lane0 = i;
    L[i] = d;
    for (uint64_t s = 0; s < j.n; s += HP_SEG) hp_work.push_back(WorkItem{(uint32_t)i, (uint32_t)s});
    for (uint64_t s = 0; s < j.n; s += PF_SEG) pf_work.push_back(WorkItem{(uint32_t)i, (uint32_t)s});
    for (uint64_t s = 0; s < j.n; s += PF2_SEG) pf2_work.push_back(WorkItem{(uint32_t)i, (uint32_t)s});
    ad_chunk0[i] = (uint32_t)ad_work.size();
    for (uint64_t s = 0; s * AD_CHUNK < j.n; s++) ad_work.push_back(WorkItem{(uint32_t)i, (uint32_t)s});
    for (uint32_t k = 0; k < d.nseg; k++) seg_lane.push_back((uint32_t)i);
    for (uint32_t k = 0; k < d.nblk_max; k++) blk_lane.push_back((uint32_t)i);
    pos_total += (j.n + 255) & ~uint64_t(255);
    sym_total += j.n + 256;
    seg_total += d.nseg;
    blk_total += d.nblk_max;
    maxG = std::max(maxG, d.G);
  }
  const uint32_t sym_stride = (maxG + 1 + 3) & ~3u;  // 16-byte aligned segment rows (K5 vector stores)
  std::vector<uint64_t> lane_prefix(nl + 1, 0);
  for (int i = 0; i < nl; i++) lane_prefix[i + 1] = lane_prefix[i] + L[i].n;
  const uint64_t npos_exact = lane_prefix[nl];
  // workspace layout
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t need = 0;
  need += al(sizeof(LaneDev) * nl) + al(sizeof(ContainerDev) * nc);
  need += al(sizeof(WorkItem) * (hp_work.size() + pf_work.size() + pf2_work.size() + ad_work.size() + 4));
  need += 2 * al(4 * pos_total) + al(32ull * nl);  // K4G's g3 / g4, the walk selection
  need += al(4 * seg_lane.size()) + al(4 * blk_lane.size()) + al(4 * nl);
  need += al(2 * pos_total) + al(8 * pos_total);
  need += 2 * al(4ull * seg_total * sym_stride);            // spec + fixup symbols
  need += al(8ull * seg_total * CONV_W);                   // state map
  need += 5 * al(sizeof(SegExit) * seg_total) + 6 * al(4ull * seg_total) + al(8ull * seg_total);
  need += al(4 * sym_total);
  need += al(sizeof(LaneSyms) * nl) + al(sizeof(BlockInfo) * blk_total) + al(sizeof(BlockCodes) * blk_total);
  need += al(HDR_BYTES * (size_t)blk_total) + al(sizeof(BlockPlan) * blk_total) + al(16ull * blk_total);
  need += al(8 * nl) + al(sizeof(uint8_t*) * nl) + al(8 * nc) + al(4 * nc) + al(sizeof(Adl) * ad_work.size() + 16);
  need += 64 * 256 + 2 * al(8 * (nl + 1)) + al(4 * nl) + al(sizeof(WorkItem) * (pos_total / HP4_SEG + nl + 1));
  int rc = e->ws.reserve(need);
  if (rc) return rc;
  Workspace& W = e->ws;
  LaneDev* d_lanes = W.take<LaneDev>(nl);
  ContainerDev* d_cons = W.take<ContainerDev>(nc);
  WorkItem* d_hp = W.take<WorkItem>(hp_work.size() + 1);
  WorkItem* d_pf = W.take<WorkItem>(pf_work.size() + 1);
  WorkItem* d_pf2 = W.take<WorkItem>(pf2_work.size() + 1);
  uint32_t* d_g3 = W.take<uint32_t>(pos_total);
  uint32_t* d_g4 = W.take<uint32_t>(pos_total);
  unsigned long long* d_k4stat = W.take<unsigned long long>(4 * nl);
  WorkItem* d_ad = W.take<WorkItem>(ad_work.size() + 1);
  uint32_t* d_seg_lane = W.take<uint32_t>(seg_lane.size());
  uint32_t* d_blk_lane = W.take<uint32_t>(blk_lane.size());
  uint32_t* d_ad_chunk0 = W.take<uint32_t>(nl);
  uint16_t* d_pd = W.take<uint16_t>(pos_total);
  uint2* d_prof = W.take<uint2>(pos_total);
  uint32_t* d_spec_syms = W.take<uint32_t>((size_t)seg_total * sym_stride);
  uint32_t* d_fix_syms = W.take<uint32_t>((size_t)seg_total * sym_stride);
  uint2* d_state_map = W.take<uint2>((size_t)seg_total * CONV_W);
  SegExit* d_spec_exit = W.take<SegExit>(seg_total);
  SegExit* d_exit_a = W.take<SegExit>(seg_total);
  SegExit* d_exit_b = W.take<SegExit>(seg_total);
  SegExit* d_entry_used = W.take<SegExit>(seg_total);
  uint32_t* d_spec_cnt = W.take<uint32_t>(seg_total);
  uint32_t* d_spec_post = W.take<uint32_t>(seg_total);
  uint32_t* d_fix_cnt = W.take<uint32_t>(seg_total);
  uint32_t* d_conv_idx = W.take<uint32_t>(seg_total);
  uint32_t* d_post_flag = W.take<uint32_t>(seg_total);
  uint32_t* d_changed = W.take<uint32_t>(4);
  uint64_t* d_seg_off = W.take<uint64_t>(seg_total);
  uint32_t* d_syms = W.take<uint32_t>(sym_total);
  LaneSyms* d_ls = W.take<LaneSyms>(nl);
  BlockInfo* d_info = W.take<BlockInfo>(blk_total);
  BlockCodes* d_codes = W.take<BlockCodes>(blk_total);
  uint32_t* d_hdr = W.take<uint32_t>((size_t)blk_total * (HDR_BYTES / 4));
  BlockPlan* d_plan = W.take<BlockPlan>(blk_total);
  uint2* d_edge = W.take<uint2>(2ull * blk_total);
  uint64_t* d_blob_len = W.take<uint64_t>(nl);
  uint8_t** d_lane_out = W.take<uint8_t*>(nl);
  uint64_t* d_con_len = W.take<uint64_t>(nc);
  int* d_con_status = W.take<int>(nc);
  Adl* d_adl = W.take<Adl>(ad_work.size() + 1);

  StageTimer T(st);
  T.mark("deflate.upload");
  BB_CUDA_TRY(cudaMemcpyAsync(d_lanes, L.data(), sizeof(LaneDev) * nl, cudaMemcpyHostToDevice, st));
  BB_CUDA_TRY(cudaMemcpyAsync(d_cons, C.data(), sizeof(ContainerDev) * nc, cudaMemcpyHostToDevice, st));
  if (!hp_work.empty())
    BB_CUDA_TRY(cudaMemcpyAsync(d_hp, hp_work.data(), sizeof(WorkItem) * hp_work.size(), cudaMemcpyHostToDevice, st));
  if (!pf_work.empty() && getenv("BB_K4_SORTED") != nullptr)
    BB_CUDA_TRY(cudaMemcpyAsync(d_pf, pf_work.data(), sizeof(WorkItem) * pf_work.size(), cudaMemcpyHostToDevice, st));
  if (!ad_work.empty())
    BB_CUDA_TRY(cudaMemcpyAsync(d_ad, ad_work.data(), sizeof(WorkItem) * ad_work.size(), cudaMemcpyHostToDevice, st));
  BB_CUDA_TRY(cudaMemcpyAsync(d_seg_lane, seg_lane.data(), 4 * seg_lane.size(), cudaMemcpyHostToDevice, st));
  BB_CUDA_TRY(cudaMemcpyAsync(d_blk_lane, blk_lane.data(), 4 * blk_lane.size(), cudaMemcpyHostToDevice, st));
  BB_CUDA_TRY(cudaMemcpyAsync(d_ad_chunk0, ad_chunk0.data(), 4 * nl, cudaMemcpyHostToDevice, st));

  // K3, K4
  // default: K3 hash-chain links + K4 lock-step chain walk.  BB_K4_SORTED=1 selects the
  // bucket-sorted variant (K3S + K4S): bit-identical, but slower on config2 (sort 13.2 ms + walk
  // 43.5 ms vs 5.6 + 35.0 ms per step, profiles/r2_ncu_summary.md)
  static const bool k4_sorted = getenv("BB_K4_SORTED") != nullptr;
  if (!k4_sorted) {
    T.mark("deflate.hash_prev");
    if (npos_exact) {
      rc = hash_prev_two_phase(e->sortws, W, d_lanes, nl, lane_prefix, d_pd, st);
      if (rc) return rc;
    }
    // Per lane: K4's full lock-step chain walk, or K4G (first 3- / 4-gram candidates, then
    // the 4-gram subsequence walk) where sampled chains say it is cheaper; both bit-identical.
    // BB_K4_CLASSIC=1 / BB_K4G=1 force one walk for every lane.
    const bool k4_classic = getenv("BB_K4_CLASSIC") != nullptr;  // read per call (tests switch them)
    const bool k4_force_g = getenv("BB_K4G") != nullptr;
    std::vector<char> use_g(nl, 0);
    if (!k4_classic && !pf_work.empty()) {
      bool any_big = false;
      for (int i = 0; i < nl; i++) any_big = any_big || L[i].n >= K4G_MIN_LANE;
      if (k4_force_g) {
        std::fill(use_g.begin(), use_g.end(), 1);
      } else if (any_big) {
        T.mark("deflate.k4_select");
        BB_CUDA_TRY(cudaMemsetAsync(d_k4stat, 0, 32ull * nl, st));
        k_k4_sample<<<dim3(K4S_CTAS, nl), 256, 0, st>>>(d_lanes, d_pd, d_k4stat);
        BB_LAUNCH_CHECK();
        rc = pinned(e, 32ull * nl);
        if (rc) return rc;
        BB_CUDA_TRY(cudaMemcpyAsync(e->h_pinned, d_k4stat, 32ull * nl, cudaMemcpyDeviceToHost, st));
        BB_CUDA_TRY(cudaStreamSynchronize(st));
        static const bool k4_debug = getenv("BB_K4_DEBUG") != nullptr;
        for (int i = 0; i < nl; i++) {
          const uint64_t* S = e->h_pinned + 4 * i;
          use_g[i] = S[3] && S[0] >= S[1] + S[2] + K4G_MARGIN * S[3];
          if (k4_debug && S[3])
            fprintf(stderr, "k4 lane %d n=%llu L=%.2f S4=%.2f H4=%.2f -> %s\n", i, (unsigned long long)L[i].n,
                    (double)S[0] / S[3], (double)S[1] / S[3], (double)S[2] / S[3], use_g[i] ? "K4G" : "classic");
        }
      }
    }
    for (int i = 0; i < nl; i++) g_k4_positions[use_g[i] ? 1 : 0] += L[i].n;
    std::vector<WorkItem> w_classic, w_gram, w_prof4;
    for (const WorkItem& w : pf_work) (use_g[w.lane] ? w_gram : w_classic).push_back(w);
    for (const WorkItem& w : pf2_work)
      if (use_g[w.lane]) w_prof4.push_back(w);
    std::vector<WorkItem> both(w_classic);
    both.insert(both.end(), w_gram.begin(), w_gram.end());
    if (!both.empty())
      BB_CUDA_TRY(cudaMemcpyAsync(d_pf, both.data(), sizeof(WorkItem) * both.size(), cudaMemcpyHostToDevice, st));
    if (!w_prof4.empty())
      BB_CUDA_TRY(
          cudaMemcpyAsync(d_pf2, w_prof4.data(), sizeof(WorkItem) * w_prof4.size(), cudaMemcpyHostToDevice, st));
    T.mark("deflate.profile");
    if (!w_classic.empty()) {
      k_profile3<<<(unsigned)w_classic.size(), PF_THREADS, 4 * PF_WIN + 16, st>>>(d_lanes, d_pf, d_pd, d_prof, 1);
      BB_LAUNCH_CHECK();
    }
    if (!w_gram.empty()) {
      T.mark("deflate.gram");
      k_gram4<<<(unsigned)w_gram.size(), PF_THREADS, 4 * PF_WIN + 16, st>>>(d_lanes, d_pf + w_classic.size(), d_pd,
                                                                           d_g3, d_g4);
      BB_LAUNCH_CHECK();
      T.mark("deflate.profile4");
      k_profile4<<<(unsigned)w_prof4.size(), PF_THREADS, PF2_SMEM + 16, st>>>(d_lanes, d_pf2, d_g3, d_g4, d_prof, 1);
      BB_LAUNCH_CHECK();
    }
  } else if (npos_exact) {
    rc = profile_sorted(e->sortws, W, d_lanes, nl, lane_prefix, d_prof, 1, T, st);
    if (rc) return rc;
  }
  // K5: speculative parse, then fix-up rounds until no exit state changes
  T.mark("deflate.parse_spec");
#ifndef K5_PT
#define K5_PT 128
#endif
  const unsigned pt = K5_PT, pg = (seg_total + pt - 1) / pt;
  k_parse_spec<<<pg, pt, 0, st>>>(d_lanes, nl, d_seg_lane, seg_total, d_prof, d_spec_syms, d_state_map,
                                  d_spec_exit, d_spec_cnt, d_spec_post, sym_stride);
  BB_LAUNCH_CHECK();
  // entry_used = the fresh state each speculative parse assumed
  k_fresh_entries<<<(seg_total + 255) / 256, 256, 0, st>>>(d_lanes, d_seg_lane, seg_total, d_entry_used);
  BB_LAUNCH_CHECK();
  BB_CUDA_TRY(cudaMemcpyAsync(d_exit_a, d_spec_exit, sizeof(SegExit) * seg_total, cudaMemcpyDeviceToDevice, st));
  BB_CUDA_TRY(cudaMemsetAsync(d_fix_cnt, 0, 4ull * seg_total, st));
  BB_CUDA_TRY(cudaMemsetAsync(d_conv_idx, 0, 4ull * seg_total, st));
  BB_CUDA_TRY(cudaMemcpyAsync(d_post_flag, d_spec_post, 4ull * seg_total, cudaMemcpyDeviceToDevice, st));
  if ((rc = pinned(e, 64 + 16ull * nc))) return rc;
  T.mark("deflate.parse_fixup");
  {
    // BB_FIXUP_COOP=1: all rounds in one cooperative launch (no host round trip per round).  Not the
    // default: measured equal (config1 2.38 vs 2.39 ms, config2 unchanged), and two cooperative grids
    // launched concurrently on one device by different host threads (the plugin e2e, a 1-GPU stage
    // runner) could each end up partly resident and wait on each other at the grid barrier.
    static const bool host_loop = getenv("BB_FIXUP_COOP") == nullptr;
    int coop_blocks = 0;
    int dev = 0;
    BB_CUDA_TRY(cudaGetDevice(&dev));
    if (!host_loop) {
      static int per_sm_dev[64] = {};  // occupancy of the cooperative kernel, queried once per device
      if (dev >= 0 && dev < 64 && per_sm_dev[dev] == 0) {
        int per_sm = 0;
        BB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_parse_fixup_coop, 128, 0));
        per_sm_dev[dev] = std::max(per_sm, 1);
      }
      const int per_sm = dev >= 0 && dev < 64 ? per_sm_dev[dev] : 1;
      coop_blocks = std::min<int>(per_sm * kNumSMs, (int)((seg_total + 127) / 128));
    }
    if (coop_blocks > 0) {
      BB_CUDA_TRY(cudaMemsetAsync(d_changed, 0, 16, st));
      const uint32_t max_rounds = seg_total + 3;
      uint32_t seg_total_u = seg_total;
      volatile uint32_t* counters = d_changed;
      void* args[] = {(void*)&d_lanes, (void*)&d_seg_lane, (void*)&seg_total_u, (void*)&d_prof,
                      (void*)&d_state_map, (void*)&d_spec_exit, (void*)&d_spec_cnt, (void*)&d_spec_post,
                      (void*)&d_exit_a, (void*)&d_exit_b, (void*)&d_entry_used, (void*)&d_fix_syms,
                      (void*)&d_fix_cnt, (void*)&d_conv_idx, (void*)&d_post_flag, (void*)&counters,
                      (void*)&sym_stride, (void*)&max_rounds};
      BB_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_parse_fixup_coop, dim3(coop_blocks), dim3(128), args,
                                              0, st));
      count_launch();
    } else {
      BB_CUDA_TRY(cudaMemsetAsync(d_changed, 0, 16, st));  // counters[3]: the coop path's non-convergence flag
      SegExit *cur = d_exit_a, *nxt = d_exit_b;
      for (int round = 0;; round += 2) {
        BB_CUDA_TRY(cudaMemsetAsync(d_changed, 0, 8, st));
        for (int r = 0; r < 2; r++) {
          k_parse_fixup<<<pg, pt, 0, st>>>(d_lanes, d_seg_lane, seg_total, d_prof, d_state_map, d_spec_exit,
                                           d_spec_cnt, d_spec_post, cur, nxt, d_entry_used, d_fix_syms, d_fix_cnt,
                                           d_conv_idx, d_post_flag, d_changed + r, sym_stride);
          BB_LAUNCH_CHECK();
          std::swap(cur, nxt);
        }
        BB_CUDA_TRY(cudaMemcpyAsync(e->h_pinned, d_changed + 1, 4, cudaMemcpyDeviceToHost, st));
        BB_CUDA_TRY(cudaStreamSynchronize(st));
        uint32_t changed = *reinterpret_cast<uint32_t*>(e->h_pinned);
        if (changed == 0) break;
        if (round > (int)seg_total + 2) {
          set_error("deflate parse fix-up did not converge");
          return BB_ERROR;
        }
      }
    }
  }
  // K6
  T.mark("deflate.compact");
  k_seg_scan<<<nl, 256, 0, st>>>(d_lanes, d_spec_cnt, d_fix_cnt, d_conv_idx, d_post_flag, d_spec_post, d_seg_off, d_ls);
  BB_LAUNCH_CHECK();
  k_compact<<<(seg_total + 7) / 8, 256, 0, st>>>(d_lanes, d_seg_lane, seg_total, d_spec_syms, d_spec_cnt, d_fix_syms,
                                                 d_fix_cnt, d_conv_idx, d_seg_off, d_syms, sym_stride);
  BB_LAUNCH_CHECK();
  T.mark("deflate.blocks_trees");
  BB_CUDA_TRY(cudaMemsetAsync(d_hdr, 0, (size_t)blk_total * HDR_BYTES, st));
  if (blk_total < 4u * kNumSMs)
    k_blocks<256><<<blk_total, 256, 0, st>>>(d_lanes, d_blk_lane, blk_total, d_ls, d_syms, d_info, d_codes, d_hdr);
  else
    k_blocks<BK_THREADS><<<blk_total, BK_THREADS, 0, st>>>(d_lanes, d_blk_lane, blk_total, d_ls, d_syms, d_info,
                                                           d_codes, d_hdr);
  BB_LAUNCH_CHECK();
  T.mark("deflate.layout");
  k_layout<<<(nl + 3) / 4, 128, 0, st>>>(d_lanes, nl, d_ls, d_info, d_plan, d_blob_len);
  BB_LAUNCH_CHECK();
  k_place<<<(nc + 127) / 128, 128, 0, st>>>(d_cons, nc, d_blob_len, d_lane_out, d_con_len, d_con_status);
  BB_LAUNCH_CHECK();
  T.mark("deflate.emit");
  k_emit<<<blk_total, EM_THREADS, 0, st>>>(d_lanes, d_blk_lane, blk_total, d_ls, d_info, d_plan, d_codes, d_hdr,
                                           d_syms, d_lane_out, d_edge);
  BB_LAUNCH_CHECK();
  k_edges<<<(2 * blk_total + 255) / 256, 256, 0, st>>>(d_lanes, d_blk_lane, blk_total, d_ls, d_lane_out, d_edge);
  BB_LAUNCH_CHECK();
  T.mark("deflate.adler_finalize");
  if (!ad_work.empty()) {
    k_adler_chunks<<<(unsigned)ad_work.size(), AD_THREADS, 0, st>>>(d_lanes, d_ad, d_adl);
    BB_LAUNCH_CHECK();
  }
  k_adler_final<<<(nl + 3) / 4, 128, 0, st>>>(d_lanes, nl, d_ad_chunk0, d_adl, d_lane_out, d_blob_len);
  BB_LAUNCH_CHECK();
  k_container_header<<<(nc + 127) / 128, 128, 0, st>>>(d_cons, nc, d_blob_len, d_con_status);
  BB_LAUNCH_CHECK();
  BB_CUDA_TRY(cudaMemcpyAsync(e->h_pinned, d_con_len, 8ull * nc, cudaMemcpyDeviceToHost, st));
  BB_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<char*>(e->h_pinned) + 8ull * nc, d_con_status, 4ull * nc,
                              cudaMemcpyDeviceToHost, st));
  uint32_t* h_nonconv = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(e->h_pinned) + 12ull * nc);
  BB_CUDA_TRY(cudaMemcpyAsync(h_nonconv, d_changed + 3, 4, cudaMemcpyDeviceToHost, st));
  BB_CUDA_TRY(cudaStreamSynchronize(st));
  T.finish();
  if (*h_nonconv) {
    set_error("deflate parse fix-up did not converge");
    return BB_ERROR;
  }
  const int* hs = reinterpret_cast<const int*>(reinterpret_cast<char*>(e->h_pinned) + 8ull * nc);
  for (int c = 0; c < nc; c++) {
    container_len[c] = e->h_pinned[c];
    container_status[c] = hs[c];
  }
  return BB_OK;
}

}  // namespace bb

#ifdef PF_STATS
extern "C" BB_API void bb_debug_pf_stats(unsigned long long* out4, int reset) {
  cudaMemcpyFromSymbol(out4, bb::g_pf_stats, sizeof(unsigned long long) * 4);
  if (reset) {
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(bb::g_pf_stats, z, sizeof z);
  }
}
#endif

// Test hook: K3S + K4S alone on one lane (profiles without the parse's byte), for the
// comparison with the oracle's orc_match_profile.
// Test / bench hook: cumulative lane positions whose profiles came from the classic walk
// (out[0]) and from K4G (out[1]) -- the coverage of each K4 kernel for the roofline accounting
extern "C" BB_API void bb_debug_k4_positions(uint64_t* out2) {
  out2[0] = bb::g_k4_positions[0].load();
  out2[1] = bb::g_k4_positions[1].load();
}

extern "C" BB_API int bb_debug_profile_sorted(const uint8_t* d_in, size_t n, uint32_t* d_prof, void* stream) {
  using namespace bb;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!n) return BB_OK;
  LaneDev d{};
  d.src = d_in;
  d.n = n;
  LaneDev* dl;
  BB_CUDA_TRY(cudaMalloc(&dl, sizeof d));
  BB_CUDA_TRY(cudaMemcpy(dl, &d, sizeof d, cudaMemcpyHostToDevice));
  Workspace sw, w2;
  std::vector<uint64_t> lp{0, n};
  struct NoTimer {
    void mark(const char*) {}
  } nt;
  int rc = profile_sorted(sw, w2, dl, 1, lp, reinterpret_cast<uint2*>(d_prof), 0, nt, st);
  if (rc) return rc;
  BB_CUDA_TRY(cudaStreamSynchronize(st));
  cudaFree(dl);
  return BB_OK;
}

// ---------------------------------------------------------------------------
// Test hooks (not part of include/bbcodec.h): run K3 / K4 alone on one lane so
// tests can compare them with the oracle's orc_hash_prev / orc_match_profile.
extern "C" BB_API int bb_debug_hash_prev_profile(const uint8_t* d_in, size_t n, uint16_t* d_pd,
                                                 uint32_t* d_prof, void* stream) {
  using namespace bb;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ZTables t = make_tables();
  BB_CUDA_TRY(cudaMemcpyToSymbol(c_z, &t, sizeof t));
  BB_CUDA_TRY(cudaFuncSetAttribute(k_hash_prev6, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  BB_CUDA_TRY(cudaFuncSetAttribute(k_hash_prev7, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  BB_CUDA_TRY(cudaFuncSetAttribute(k_hash_prev8, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  BB_CUDA_TRY(cudaFuncSetAttribute(k_profile3, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * PF_WIN + 16));
  BB_CUDA_TRY(cudaFuncSetAttribute(k_gram4, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * PF_WIN + 16));
  BB_CUDA_TRY(cudaFuncSetAttribute(k_profile4, cudaFuncAttributeMaxDynamicSharedMemorySize, PF2_SMEM + 16));
  LaneDev d{};
  d.src = d_in;
  d.n = n;
  std::vector<WorkItem> hp, pf, pf2;
  for (uint64_t s = 0; s < n; s += HP_SEG) hp.push_back(WorkItem{0, (uint32_t)s});
  for (uint64_t s = 0; s < n; s += PF_SEG) pf.push_back(WorkItem{0, (uint32_t)s});
  for (uint64_t s = 0; s < n; s += PF2_SEG) pf2.push_back(WorkItem{0, (uint32_t)s});
  LaneDev* dl;
  WorkItem *dh, *dp, *dp2;
  uint32_t* dg = nullptr;
  BB_CUDA_TRY(cudaMalloc(&dl, sizeof d));
  BB_CUDA_TRY(cudaMalloc(&dh, sizeof(WorkItem) * (hp.size() + 1)));
  BB_CUDA_TRY(cudaMalloc(&dp, sizeof(WorkItem) * (pf.size() + 1)));
  BB_CUDA_TRY(cudaMalloc(&dp2, sizeof(WorkItem) * (pf2.size() + 1)));
  BB_CUDA_TRY(cudaMalloc(&dg, 8 * (n + 1)));
  BB_CUDA_TRY(cudaMemcpy(dl, &d, sizeof d, cudaMemcpyHostToDevice));
  if (!hp.empty()) BB_CUDA_TRY(cudaMemcpy(dh, hp.data(), sizeof(WorkItem) * hp.size(), cudaMemcpyHostToDevice));
  if (!pf.empty()) BB_CUDA_TRY(cudaMemcpy(dp, pf.data(), sizeof(WorkItem) * pf.size(), cudaMemcpyHostToDevice));
  if (!pf2.empty()) BB_CUDA_TRY(cudaMemcpy(dp2, pf2.data(), sizeof(WorkItem) * pf2.size(), cudaMemcpyHostToDevice));
  if (n) {
    Workspace sw, w2;
    int rc = w2.reserve(4096 + 16 * (n / HP4_SEG + 2));
    if (rc) return rc;
    std::vector<uint64_t> lp{0, n};
    rc = hash_prev_two_phase(sw, w2, dl, 1, lp, d_pd, st);
    if (rc) return rc;
    BB_CUDA_TRY(cudaStreamSynchronize(st));
  }
  if (!pf.empty() && d_prof) {
    const bool k4_classic = getenv("BB_K4_CLASSIC") != nullptr;  // per call: tests check both walks
    if (k4_classic) {
      k_profile3<<<(unsigned)pf.size(), PF_THREADS, 4 * PF_WIN + 16, st>>>(dl, dp, d_pd,
                                                                        reinterpret_cast<uint2*>(d_prof), 0);
    } else {
      k_gram4<<<(unsigned)pf.size(), PF_THREADS, 4 * PF_WIN + 16, st>>>(dl, dp, d_pd, dg, dg + n);
      BB_LAUNCH_CHECK();
      k_profile4<<<(unsigned)pf2.size(), PF_THREADS, PF2_SMEM + 16, st>>>(dl, dp2, dg, dg + n,
                                                                         reinterpret_cast<uint2*>(d_prof), 0);
    }
    BB_LAUNCH_CHECK();
  }
  BB_CUDA_TRY(cudaStreamSynchronize(st));
  cudaFree(dl);
  cudaFree(dh);
  cudaFree(dp);
  cudaFree(dp2);
  cudaFree(dg);
  return BB_OK;
}
