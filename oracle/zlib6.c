/* ORACLE / TEST INFRASTRUCTURE ONLY -- see oracle/bboracle.h.
 *
 * CPU restatement of zlib 1.3 compress2(dest, &len, src, n, Z_DEFAULT_COMPRESSION)
 * as called by the reference deflate backend (reference proj/src/codec.cpp:17-25).
 * zlib is a third-party dependency that is not vendored under /root/reference;
 * the pinned build is the system zlib1g 1:1.3.dfsg-3.1ubuntu2.2 (vanilla madler
 * zlib 1.3 on amd64, zlibCompileFlags 0xa9).  This file restates its published
 * algorithm for level 6 (deflate.c: lm_init, fill_window, deflate_slow,
 * longest_match; trees.c: _tr_tally, _tr_flush_block, build_tree, gen_bitlen,
 * gen_codes, scan_tree, send_tree, build_bl_tree, send_all_trees,
 * compress_block, _tr_stored_block; adler32.c) with absolute input positions
 * instead of zlib's sliding 64 KiB window.  The window slide is still tracked
 * because it changes exactly two observable things:
 *   1. stored-block eligibility (zlib passes buf == NULL when block_start < 0);
 *   2. a chain head at relative position 0 after a slide reads as NIL.
 * Bytes beyond the end of input never change the chosen parse (longest_match
 * caps at lookahead and stops at nice_match = min(128, lookahead)), so LCPs are
 * simply bounded by the remaining input here.
 *
 * orc_zlib_compress()           -- the sequential zlib-shaped restatement.
 * orc_zlib_compress_profiled()  -- identical bytes through the decomposition the
 *                                  GPU uses: hash-prev distances (K3), per-position
 *                                  match profiles for chain budgets 128 and 32
 *                                  (K4), the lazy parse as an O(1)/position state
 *                                  machine over profiles (K5), then the same
 *                                  block coder.  Both are pinned against libz.
 */
#include <stdlib.h>
#include <string.h>

#include "bboracle.h"

#define L_CODES 286
#define D_CODES 30
#define BL_CODES 19
#define HEAP_SIZE (2 * L_CODES + 1)
#define MAX_BITS 15
#define MAX_BL_BITS 7
#define END_BLOCK 256
#define LITERALS 256
#define LENGTH_CODES 29
#define REP_3_6 16
#define REPZ_3_10 17
#define REPZ_11_138 18

/* level 6 configuration_table entry {good, lazy, nice, chain} */
#define GOOD_LENGTH 8
#define MAX_LAZY 16
#define NICE_LENGTH 128
#define MAX_CHAIN 128
#define MIN_MATCH 3
#define MAX_MATCH 258
#define WSIZE 32768u
#define MAX_DIST (WSIZE - (MAX_MATCH + MIN_MATCH + 1)) /* 32506 */
#define MIN_LOOKAHEAD (MAX_MATCH + MIN_MATCH + 1)       /* 262 */
#define WINDOW_SIZE (2u * WSIZE)
#define TOO_FAR 4096
#define SYM_LIMIT 16383 /* lit_bufsize - 1, lit_bufsize = 1 << (8 + 6) */
#define HASH_BITS 15
#define HASH_MASK ((1u << HASH_BITS) - 1)

static const int extra_lbits[LENGTH_CODES] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2,
                                              2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
static const int extra_dbits[D_CODES] = {0, 0, 0, 0, 1, 1, 2, 2,  3,  3,  4,  4,  5,  5,  6,
                                         6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
static const int extra_blbits[BL_CODES] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 2, 3, 7};
static const unsigned char bl_order[BL_CODES] = {16, 17, 18, 0, 8,  7, 9,  6, 10, 5,
                                                 11, 4,  12, 3, 13, 2, 14, 1, 15};

static unsigned char length_code[256];
static unsigned char dist_code[512];
static int base_length[LENGTH_CODES];
static int base_dist[D_CODES];
static unsigned short static_ltree_len[L_CODES + 2], static_ltree_code[L_CODES + 2];
static unsigned short static_dtree_len[D_CODES], static_dtree_code[D_CODES];

static unsigned bi_reverse(unsigned code, int len) {
  unsigned res = 0;
  do {
    res |= code & 1;
    code >>= 1, res <<= 1;
  } while (--len > 0);
  return res >> 1;
}

/* trees.c gen_codes */
static void gen_codes(const unsigned short* len, unsigned short* code, int max_code,
                      const unsigned short* bl_count) {
  unsigned short next_code[MAX_BITS + 1];
  unsigned c = 0;
  for (int bits = 1; bits <= MAX_BITS; bits++) {
    c = (c + bl_count[bits - 1]) << 1;
    next_code[bits] = (unsigned short)c;
  }
  for (int n = 0; n <= max_code; n++) {
    int l = len[n];
    if (l == 0) continue;
    code[n] = (unsigned short)bi_reverse(next_code[l]++, l);
  }
}

/* trees.c tr_static_init */
static void tables_init(void) {
  static int done = 0;
  if (done) return;
  int length = 0, code, n, dist;
  for (code = 0; code < LENGTH_CODES - 1; code++) {
    base_length[code] = length;
    for (n = 0; n < (1 << extra_lbits[code]); n++) length_code[length++] = (unsigned char)code;
  }
  length_code[length - 1] = (unsigned char)code; /* 258 -> code 285 */
  base_length[LENGTH_CODES - 1] = 0;
  dist = 0;
  for (code = 0; code < 16; code++) {
    base_dist[code] = dist;
    for (n = 0; n < (1 << extra_dbits[code]); n++) dist_code[dist++] = (unsigned char)code;
  }
  dist >>= 7;
  for (; code < D_CODES; code++) {
    base_dist[code] = dist << 7;
    for (n = 0; n < (1 << (extra_dbits[code] - 7)); n++) dist_code[256 + dist++] = (unsigned char)code;
  }
  unsigned short bl_count[MAX_BITS + 1] = {0};
  for (n = 0; n <= 143; n++) static_ltree_len[n] = 8, bl_count[8]++;
  for (; n <= 255; n++) static_ltree_len[n] = 9, bl_count[9]++;
  for (; n <= 279; n++) static_ltree_len[n] = 7, bl_count[7]++;
  for (; n <= 287; n++) static_ltree_len[n] = 8, bl_count[8]++;
  gen_codes(static_ltree_len, static_ltree_code, L_CODES + 1, bl_count);
  for (n = 0; n < D_CODES; n++) {
    static_dtree_len[n] = 5;
    static_dtree_code[n] = (unsigned short)bi_reverse((unsigned)n, 5);
  }
  done = 1;
}

static unsigned d_code(unsigned dist) { return dist < 256 ? dist_code[dist] : dist_code[256 + (dist >> 7)]; }

/* ------------------------------------------------------------------------- */
/* adler32.c                                                                  */
uint32_t orc_adler32(uint32_t adler, const uint8_t* buf, size_t n) {
  uint64_t a = adler & 0xffff, b = adler >> 16;
  while (n) {
    size_t k = n < 5552 ? n : 5552; /* NMAX */
    n -= k;
    while (k--) {
      a += *buf++;
      b += a;
    }
    a %= 65521;
    b %= 65521;
  }
  return (uint32_t)((b << 16) | a);
}

/* ------------------------------------------------------------------------- */
/* Bit writer (trees.c send_bits / bi_windup / put_short, LSB first)          */
typedef struct {
  uint8_t* out;
  size_t cap, pos;
  uint64_t bb;
  int bc;
  int overflow;
} bitw;

static void put_byte(bitw* w, unsigned v) {
  if (w->pos < w->cap)
    w->out[w->pos] = (uint8_t)v;
  else
    w->overflow = 1;
  w->pos++;
}
static void send_bits(bitw* w, unsigned value, int length) {
  w->bb |= (uint64_t)value << w->bc;
  w->bc += length;
  while (w->bc >= 8) {
    put_byte(w, (unsigned)(w->bb & 0xff));
    w->bb >>= 8;
    w->bc -= 8;
  }
}
static void bi_windup(bitw* w) {
  if (w->bc > 0) put_byte(w, (unsigned)(w->bb & 0xff));
  w->bb = 0;
  w->bc = 0;
}

/* ------------------------------------------------------------------------- */
/* Tree state (deflate_state subset)                                          */
typedef struct {
  unsigned short freq[HEAP_SIZE];
  unsigned short code[HEAP_SIZE];
  unsigned short dad[HEAP_SIZE];
  unsigned short len[HEAP_SIZE + 1]; /* +1: scan_tree guard slot */
} tree_t;

typedef struct {
  const unsigned short* static_len;
  const int* extra_bits;
  int extra_base;
  int elems;
  int max_length;
} static_desc;

static const static_desc l_sdesc = {static_ltree_len, extra_lbits, LITERALS + 1, L_CODES, MAX_BITS};
static const static_desc d_sdesc = {static_dtree_len, extra_dbits, 0, D_CODES, MAX_BITS};
static const static_desc bl_sdesc = {NULL, extra_blbits, 0, BL_CODES, MAX_BL_BITS};

typedef struct {
  tree_t* tree;
  int max_code;
  const static_desc* sd;
} tree_desc;

typedef struct {
  tree_t lt, dt, blt;
  tree_desc l_desc, d_desc, bl_desc;
  int heap[2 * L_CODES + 1];
  int heap_len, heap_max;
  unsigned char depth[2 * L_CODES + 1];
  unsigned short bl_count[MAX_BITS + 1];
  uint64_t opt_len, static_len;
  unsigned short sym_dist[SYM_LIMIT + 1];
  unsigned char sym_lc[SYM_LIMIT + 1];
  unsigned sym_next;
  bitw w;
} dstate;

static void init_block(dstate* s) {
  for (int n = 0; n < L_CODES; n++) s->lt.freq[n] = 0;
  for (int n = 0; n < D_CODES; n++) s->dt.freq[n] = 0;
  for (int n = 0; n < BL_CODES; n++) s->blt.freq[n] = 0;
  s->lt.freq[END_BLOCK] = 1;
  s->opt_len = s->static_len = 0;
  s->sym_next = 0;
}

#define SMALLEST 1
static int smaller(const tree_t* t, int n, int m, const unsigned char* depth) {
  return t->freq[n] < t->freq[m] || (t->freq[n] == t->freq[m] && depth[n] <= depth[m]);
}

static void pqdownheap(dstate* s, const tree_t* t, int k) {
  int v = s->heap[k];
  int j = k << 1;
  while (j <= s->heap_len) {
    if (j < s->heap_len && smaller(t, s->heap[j + 1], s->heap[j], s->depth)) j++;
    if (smaller(t, v, s->heap[j], s->depth)) break;
    s->heap[k] = s->heap[j];
    k = j;
    j <<= 1;
  }
  s->heap[k] = v;
}

static void gen_bitlen(dstate* s, tree_desc* desc) {
  tree_t* t = desc->tree;
  int max_code = desc->max_code;
  const unsigned short* stree = desc->sd->static_len;
  const int* extra = desc->sd->extra_bits;
  int base = desc->sd->extra_base;
  int max_length = desc->sd->max_length;
  int h, n, m, bits, xbits, overflow = 0;
  for (bits = 0; bits <= MAX_BITS; bits++) s->bl_count[bits] = 0;
  t->len[s->heap[s->heap_max]] = 0; /* root */
  for (h = s->heap_max + 1; h < HEAP_SIZE; h++) {
    n = s->heap[h];
    bits = t->len[t->dad[n]] + 1;
    if (bits > max_length) bits = max_length, overflow++;
    t->len[n] = (unsigned short)bits;
    if (n > max_code) continue; /* not a leaf */
    s->bl_count[bits]++;
    xbits = 0;
    if (n >= base) xbits = extra[n - base];
    unsigned f = t->freq[n];
    s->opt_len += (uint64_t)f * (unsigned)(bits + xbits);
    if (stree) s->static_len += (uint64_t)f * (unsigned)(stree[n] + xbits);
  }
  if (overflow == 0) return;
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
      m = s->heap[--h];
      if (m > max_code) continue;
      if ((unsigned)t->len[m] != (unsigned)bits) {
        s->opt_len += ((uint64_t)bits - t->len[m]) * t->freq[m];
        t->len[m] = (unsigned short)bits;
      }
      n--;
    }
  }
}

static void build_tree(dstate* s, tree_desc* desc) {
  tree_t* t = desc->tree;
  const unsigned short* stree = desc->sd->static_len;
  int elems = desc->sd->elems;
  int n, m, max_code = -1, node;
  s->heap_len = 0, s->heap_max = HEAP_SIZE;
  for (n = 0; n < elems; n++) {
    if (t->freq[n] != 0) {
      s->heap[++(s->heap_len)] = max_code = n;
      s->depth[n] = 0;
    } else {
      t->len[n] = 0;
    }
  }
  while (s->heap_len < 2) {
    node = s->heap[++(s->heap_len)] = (max_code < 2 ? ++max_code : 0);
    t->freq[node] = 1;
    s->depth[node] = 0;
    s->opt_len--;
    if (stree) s->static_len -= stree[node];
  }
  desc->max_code = max_code;
  for (n = s->heap_len / 2; n >= 1; n--) pqdownheap(s, t, n);
  node = elems;
  do {
    n = s->heap[SMALLEST];
    s->heap[SMALLEST] = s->heap[s->heap_len--];
    pqdownheap(s, t, SMALLEST);
    m = s->heap[SMALLEST];
    s->heap[--(s->heap_max)] = n;
    s->heap[--(s->heap_max)] = m;
    t->freq[node] = (unsigned short)(t->freq[n] + t->freq[m]);
    s->depth[node] = (unsigned char)((s->depth[n] >= s->depth[m] ? s->depth[n] : s->depth[m]) + 1);
    t->dad[n] = t->dad[m] = (unsigned short)node;
    s->heap[SMALLEST] = node++;
    pqdownheap(s, t, SMALLEST);
  } while (s->heap_len >= 2);
  s->heap[--(s->heap_max)] = s->heap[SMALLEST];
  gen_bitlen(s, desc);
  gen_codes(t->len, t->code, max_code, s->bl_count);
}

static void scan_tree(dstate* s, tree_t* t, int max_code) {
  int n, prevlen = -1, curlen, nextlen = t->len[0], count = 0, max_count = 7, min_count = 4;
  if (nextlen == 0) max_count = 138, min_count = 3;
  t->len[max_code + 1] = (unsigned short)0xffff; /* guard */
  for (n = 0; n <= max_code; n++) {
    curlen = nextlen;
    nextlen = t->len[n + 1];
    if (++count < max_count && curlen == nextlen) {
      continue;
    } else if (count < min_count) {
      s->blt.freq[curlen] += (unsigned short)count;
    } else if (curlen != 0) {
      if (curlen != prevlen) s->blt.freq[curlen]++;
      s->blt.freq[REP_3_6]++;
    } else if (count <= 10) {
      s->blt.freq[REPZ_3_10]++;
    } else {
      s->blt.freq[REPZ_11_138]++;
    }
    count = 0;
    prevlen = curlen;
    if (nextlen == 0)
      max_count = 138, min_count = 3;
    else if (curlen == nextlen)
      max_count = 6, min_count = 3;
    else
      max_count = 7, min_count = 4;
  }
}

#define SEND_CODE(s, c, t) send_bits(&(s)->w, (t)->code[c], (t)->len[c])

static void send_tree(dstate* s, tree_t* t, int max_code) {
  int n, prevlen = -1, curlen, nextlen = t->len[0], count = 0, max_count = 7, min_count = 4;
  if (nextlen == 0) max_count = 138, min_count = 3;
  for (n = 0; n <= max_code; n++) {
    curlen = nextlen;
    nextlen = t->len[n + 1];
    if (++count < max_count && curlen == nextlen) {
      continue;
    } else if (count < min_count) {
      do {
        SEND_CODE(s, curlen, &s->blt);
      } while (--count != 0);
    } else if (curlen != 0) {
      if (curlen != prevlen) {
        SEND_CODE(s, curlen, &s->blt);
        count--;
      }
      SEND_CODE(s, REP_3_6, &s->blt);
      send_bits(&s->w, (unsigned)(count - 3), 2);
    } else if (count <= 10) {
      SEND_CODE(s, REPZ_3_10, &s->blt);
      send_bits(&s->w, (unsigned)(count - 3), 3);
    } else {
      SEND_CODE(s, REPZ_11_138, &s->blt);
      send_bits(&s->w, (unsigned)(count - 11), 7);
    }
    count = 0;
    prevlen = curlen;
    if (nextlen == 0)
      max_count = 138, min_count = 3;
    else if (curlen == nextlen)
      max_count = 6, min_count = 3;
    else
      max_count = 7, min_count = 4;
  }
}

static int build_bl_tree(dstate* s) {
  int max_blindex;
  scan_tree(s, &s->lt, s->l_desc.max_code);
  scan_tree(s, &s->dt, s->d_desc.max_code);
  build_tree(s, &s->bl_desc);
  for (max_blindex = BL_CODES - 1; max_blindex >= 3; max_blindex--)
    if (s->blt.len[bl_order[max_blindex]] != 0) break;
  s->opt_len += 3 * ((uint64_t)max_blindex + 1) + 5 + 5 + 4;
  return max_blindex;
}

static void send_all_trees(dstate* s, int lcodes, int dcodes, int blcodes) {
  send_bits(&s->w, (unsigned)(lcodes - 257), 5);
  send_bits(&s->w, (unsigned)(dcodes - 1), 5);
  send_bits(&s->w, (unsigned)(blcodes - 4), 4);
  for (int rank = 0; rank < blcodes; rank++) send_bits(&s->w, s->blt.len[bl_order[rank]], 3);
  send_tree(s, &s->lt, lcodes - 1);
  send_tree(s, &s->dt, dcodes - 1);
}

static void compress_block(dstate* s, const unsigned short* lcode, const unsigned short* llen,
                           const unsigned short* dcode, const unsigned short* dlen) {
  for (unsigned sx = 0; sx < s->sym_next; sx++) {
    unsigned dist = s->sym_dist[sx];
    int lc = s->sym_lc[sx];
    if (dist == 0) {
      send_bits(&s->w, lcode[lc], llen[lc]);
    } else {
      unsigned code = length_code[lc];
      send_bits(&s->w, lcode[code + LITERALS + 1], llen[code + LITERALS + 1]);
      int extra = extra_lbits[code];
      if (extra != 0) send_bits(&s->w, (unsigned)(lc - base_length[code]), extra);
      dist--;
      code = d_code(dist);
      send_bits(&s->w, dcode[code], dlen[code]);
      extra = extra_dbits[code];
      if (extra != 0) send_bits(&s->w, dist - (unsigned)base_dist[code], extra);
    }
  }
  send_bits(&s->w, lcode[END_BLOCK], llen[END_BLOCK]);
}

/* _tr_tally: returns 1 when the symbol buffer is full (sym_next == sym_end) */
static int tally(dstate* s, unsigned dist, unsigned lc) {
  s->sym_dist[s->sym_next] = (unsigned short)dist;
  s->sym_lc[s->sym_next] = (unsigned char)lc;
  s->sym_next++;
  if (dist == 0) {
    s->lt.freq[lc]++;
  } else {
    dist--;
    s->lt.freq[length_code[lc] + LITERALS + 1]++;
    s->dt.freq[d_code(dist)]++;
  }
  return s->sym_next == SYM_LIMIT;
}

/* _tr_flush_block.  buf_ok == 0 where zlib passes buf == NULL (block_start < 0). */
static void flush_block(dstate* s, const uint8_t* buf, int buf_ok, uint64_t stored_len, int last) {
  uint64_t opt_lenb, static_lenb;
  build_tree(s, &s->l_desc);
  build_tree(s, &s->d_desc);
  int max_blindex = build_bl_tree(s);
  opt_lenb = (s->opt_len + 3 + 7) >> 3;
  static_lenb = (s->static_len + 3 + 7) >> 3;
  if (static_lenb <= opt_lenb) opt_lenb = static_lenb;
  if (stored_len + 4 <= opt_lenb && buf_ok) {
    send_bits(&s->w, (0u << 1) + (unsigned)last, 3);
    bi_windup(&s->w);
    put_byte(&s->w, (unsigned)(stored_len & 0xff));
    put_byte(&s->w, (unsigned)((stored_len >> 8) & 0xff));
    put_byte(&s->w, (unsigned)(~stored_len & 0xff));
    put_byte(&s->w, (unsigned)((~stored_len >> 8) & 0xff));
    for (uint64_t i = 0; i < stored_len; i++) put_byte(&s->w, buf[i]);
  } else if (static_lenb == opt_lenb) {
    send_bits(&s->w, (1u << 1) + (unsigned)last, 3);
    compress_block(s, static_ltree_code, static_ltree_len, static_dtree_code, static_dtree_len);
  } else {
    send_bits(&s->w, (2u << 1) + (unsigned)last, 3);
    send_all_trees(s, s->l_desc.max_code + 1, s->d_desc.max_code + 1, max_blindex + 1);
    compress_block(s, s->lt.code, s->lt.len, s->dt.code, s->dt.len);
  }
  init_block(s);
  if (last) bi_windup(&s->w);
}

static dstate* dstate_new(uint8_t* out, size_t cap) {
  tables_init();
  dstate* s = (dstate*)calloc(1, sizeof(dstate));
  s->l_desc.tree = &s->lt;
  s->l_desc.sd = &l_sdesc;
  s->d_desc.tree = &s->dt;
  s->d_desc.sd = &d_sdesc;
  s->bl_desc.tree = &s->blt;
  s->bl_desc.sd = &bl_sdesc;
  s->w.out = out;
  s->w.cap = cap;
  init_block(s);
  return s;
}

size_t orc_compress_bound(size_t n) { return n + (n >> 12) + (n >> 14) + (n >> 25) + 13; }

static unsigned hash3(const uint8_t* in, size_t p) {
  return (((unsigned)in[p] << 10) ^ ((unsigned)in[p + 1] << 5) ^ in[p + 2]) & HASH_MASK;
}

/* Window bookkeeping shared by both encoders: fill_window() runs at the loop
 * top whenever lookahead < MIN_LOOKAHEAD and slides when strstart (relative)
 * >= wsize + MAX_DIST.  Returns the lookahead after the fill. */
static size_t window_top(size_t p, size_t n, uint64_t* slides) {
  uint64_t base = (uint64_t)WSIZE * *slides;
  uint64_t wend = base + WINDOW_SIZE;
  if (wend > n) wend = n;
  if (wend - p < MIN_LOOKAHEAD) {
    if (p - base >= WSIZE + MAX_DIST) {
      (*slides)++;
      base += WSIZE;
      wend = base + WINDOW_SIZE;
      if (wend > n) wend = n;
    }
  }
  return (size_t)(wend - p);
}

static int finish_stream(dstate* s, const uint8_t* in, size_t n, size_t* out_len) {
  uint32_t ad = orc_adler32(1, in, n);
  put_byte(&s->w, ad >> 24);
  put_byte(&s->w, (ad >> 16) & 0xff);
  put_byte(&s->w, (ad >> 8) & 0xff);
  put_byte(&s->w, ad & 0xff);
  int rc = s->w.overflow ? -1 : 0;
  *out_len = s->w.pos;
  free(s);
  return rc;
}

#define FLUSH(last_)                                                                       \
  do {                                                                                     \
    int ok_ = block_start >= (uint64_t)WSIZE * slides;                                     \
    flush_block(s, in + block_start, ok_, (uint64_t)(p - block_start), (last_));           \
    block_start = p;                                                                       \
  } while (0)

/* deflate.c deflate_slow() + longest_match(), level 6, absolute positions. */
int orc_zlib_compress(const uint8_t* in, size_t n, uint8_t* out, size_t cap, size_t* out_len) {
  dstate* s = dstate_new(out, cap);
  int32_t* head = (int32_t*)malloc(sizeof(int32_t) * (HASH_MASK + 1));
  int32_t* prev = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
  for (unsigned i = 0; i <= HASH_MASK; i++) head[i] = -1;
  put_byte(&s->w, 0x78);
  put_byte(&s->w, 0x9c);

  size_t p = 0, block_start = 0;
  uint64_t slides = 0;
  unsigned prev_length = MIN_MATCH - 1, match_length = MIN_MATCH - 1;
  size_t prev_match = 0, match_start = 0;
  int match_available = 0;
  for (;;) {
    size_t lookahead = window_top(p, n, &slides);
    if (lookahead == 0) break;
    uint64_t base = (uint64_t)WSIZE * slides;
    int64_t hash_head = -1; /* NIL */
    if (lookahead >= MIN_MATCH) {
      unsigned h = hash3(in, p);
      hash_head = head[h];
      prev[p] = head[h];
      head[h] = (int32_t)p;
      /* a head at relative position <= 0 was cleared to NIL by slide_hash */
      if (hash_head >= 0 && (uint64_t)hash_head <= base) hash_head = -1;
      if (hash_head == 0) hash_head = -1; /* absolute 0 == NIL before any slide */
    }
    prev_length = match_length, prev_match = match_start;
    match_length = MIN_MATCH - 1;
    if (hash_head >= 0 && prev_length < MAX_LAZY && p - (size_t)hash_head <= MAX_DIST) {
      /* longest_match(s, hash_head) */
      unsigned chain = MAX_CHAIN;
      unsigned best_len = prev_length;
      unsigned nice = NICE_LENGTH;
      uint64_t rel = p - base;
      uint64_t limit = rel > MAX_DIST ? p - MAX_DIST : base; /* NIL in relative terms */
      if (prev_length >= GOOD_LENGTH) chain >>= 2;
      if (nice > lookahead) nice = (unsigned)lookahead;
      unsigned maxl = lookahead < MAX_MATCH ? (unsigned)lookahead : MAX_MATCH;
      int64_t cur = hash_head;
      do {
        const uint8_t* a = in + p;
        const uint8_t* b = in + cur;
        unsigned len = 0;
        while (len < maxl && a[len] == b[len]) len++;
        if (len > best_len) {
          match_start = (size_t)cur;
          best_len = len;
          if (len >= nice) break;
        }
        cur = prev[cur];
      } while (cur >= 0 && (uint64_t)cur > limit && --chain != 0);
      match_length = best_len <= lookahead ? best_len : (unsigned)lookahead;
      if (match_length == MIN_MATCH && p - match_start > TOO_FAR) match_length = MIN_MATCH - 1;
    }
    if (prev_length >= MIN_MATCH && match_length <= prev_length) {
      size_t max_insert = p + lookahead - MIN_MATCH;
      int bflush = tally(s, (unsigned)(p - 1 - prev_match), prev_length - MIN_MATCH);
      unsigned k = prev_length - 2;
      do {
        if (++p <= max_insert) {
          unsigned h = hash3(in, p);
          prev[p] = head[h];
          head[h] = (int32_t)p;
        }
      } while (--k != 0);
      match_available = 0;
      match_length = MIN_MATCH - 1;
      p++;
      if (bflush) FLUSH(0);
    } else if (match_available) {
      int bflush = tally(s, 0, in[p - 1]);
      if (bflush) FLUSH(0);
      p++;
    } else {
      match_available = 1;
      p++;
    }
  }
  if (match_available) tally(s, 0, in[p - 1]);
  FLUSH(1);
  free(head);
  free(prev);
  return finish_stream(s, in, n, out_len);
}

/* ------------------------------------------------------------------------- */
/* The GPU decomposition, on the CPU.                                         */

void orc_hash_prev(const uint8_t* in, size_t n, uint16_t* pd) {
  int64_t* head = (int64_t*)malloc(sizeof(int64_t) * (HASH_MASK + 1));
  for (unsigned i = 0; i <= HASH_MASK; i++) head[i] = -1;
  for (size_t q = 0; q < n; q++) {
    pd[q] = 0;
    if (q + MIN_MATCH > n) continue;
    unsigned h = hash3(in, q);
    if (head[h] >= 0 && q - (size_t)head[h] < WSIZE) pd[q] = (uint16_t)(q - (size_t)head[h]);
    head[h] = (int64_t)q;
  }
  free(head);
}

#define PROF_LEN(x) ((x)&0x1ffu)
#define PROF_DIST(x) (((x) >> 9) & 0x7fffu)
#define PROF_AT_MAXDIST 0x80000000u

/* K4: for every position, the chain walk of longest_match() with best_len
 * starting below any real match, recorded after 32 and after 128 candidates.
 * The first maximum (ties keep the earlier = nearer candidate) over the walk
 * truncated at the first candidate reaching nice_match is exactly what
 * longest_match returns for any prev_length below that maximum. */
static void profile_one(const uint8_t* in, size_t n, const uint16_t* pd, size_t p, uint32_t* out) {
  out[0] = out[1] = 0;
  if (p + MIN_MATCH > n || pd[p] == 0) return;
  size_t first = p - pd[p];
  if (pd[p] > MAX_DIST || first == 0) return; /* too far / absolute 0 is NIL */
  size_t lookahead = n - p;
  unsigned nice = lookahead < NICE_LENGTH ? (unsigned)lookahead : NICE_LENGTH;
  unsigned maxl = lookahead < MAX_MATCH ? (unsigned)lookahead : MAX_MATCH;
  size_t limit = p > MAX_DIST ? p - MAX_DIST : 0;
  unsigned best = MIN_MATCH - 1, bestd = 0;
  uint32_t flag = pd[p] == MAX_DIST ? PROF_AT_MAXDIST : 0;
  size_t cur = first;
  unsigned count = 0;
  for (;;) {
    unsigned len = 0;
    while (len < maxl && in[p + len] == in[cur + len]) len++;
    count++;
    if (len > best) {
      best = len;
      bestd = (unsigned)(p - cur);
      if (len >= nice) {
        if (count <= 32) out[1] = best | (bestd << 9);
        break;
      }
    }
    if (count == 32) out[1] = best > 2 ? (best | (bestd << 9)) : 0;
    if (count == MAX_CHAIN) break;
    if (pd[cur] == 0) break;
    size_t nxt = cur - pd[cur];
    if (nxt <= limit) break;
    cur = nxt;
  }
  if (count < 32) out[1] = best > 2 ? (best | (bestd << 9)) : 0;
  out[0] = best > 2 ? (best | (bestd << 9)) : 0;
  /* TOO_FAR: a length-3 match more than 4096 back is dropped */
  if (PROF_LEN(out[0]) == MIN_MATCH && PROF_DIST(out[0]) > TOO_FAR) out[0] = 0;
  if (PROF_LEN(out[1]) == MIN_MATCH && PROF_DIST(out[1]) > TOO_FAR) out[1] = 0;
  out[0] |= flag;
  out[1] |= flag;
}

void orc_match_profile(const uint8_t* in, size_t n, uint32_t* prof) {
  uint16_t* pd = (uint16_t*)malloc(sizeof(uint16_t) * (n ? n : 1));
  orc_hash_prev(in, n, pd);
  for (size_t p = 0; p < n; p++) profile_one(in, n, pd, p, prof + 2 * p);
  free(pd);
}

int orc_zlib_compress_profiled(const uint8_t* in, size_t n, uint8_t* out, size_t cap,
                               size_t* out_len) {
  uint32_t* prof = (uint32_t*)malloc(sizeof(uint32_t) * 2 * (n ? n : 1));
  orc_match_profile(in, n, prof);
  dstate* s = dstate_new(out, cap);
  put_byte(&s->w, 0x78);
  put_byte(&s->w, 0x9c);
  size_t p = 0, block_start = 0;
  uint64_t slides = 0;
  unsigned L = MIN_MATCH - 1; /* prev_length */
  unsigned pdist = 0;         /* prev match distance */
  int avail = 0;
  for (;;) {
    size_t lookahead = window_top(p, n, &slides);
    if (lookahead == 0) break;
    unsigned ml = MIN_MATCH - 1, md = 0;
    if (L < MAX_LAZY) {
      uint32_t pr = prof[2 * p + (L >= GOOD_LENGTH ? 1 : 0)];
      /* a first candidate exactly MAX_DIST back sits at relative 0 right after a
       * slide at strstart == wsize + MAX_DIST (only possible near the end) */
      int nil = (pr & PROF_AT_MAXDIST) && p - (uint64_t)WSIZE * slides == MAX_DIST;
      if (!nil && PROF_LEN(pr) > L) ml = PROF_LEN(pr), md = PROF_DIST(pr);
    }
    if (L >= MIN_MATCH && ml <= L) {
      int bflush = tally(s, pdist, L - MIN_MATCH);
      p = p - 1 + L;
      L = MIN_MATCH - 1;
      avail = 0;
      if (bflush) FLUSH(0);
    } else if (avail) {
      int bflush = tally(s, 0, in[p - 1]);
      if (bflush) FLUSH(0);
      p++;
      L = ml, pdist = md;
    } else {
      avail = 1;
      p++;
      L = ml, pdist = md;
    }
  }
  if (avail) tally(s, 0, in[p - 1]);
  FLUSH(1);
  free(prof);
  return finish_stream(s, in, n, out_len);
}
