/* ORACLE / TEST INFRASTRUCTURE ONLY -- see oracle/bboracle.h.
 *
 * CPU restatement of zlib 1.3 uncompress() as called by the reference deflate
 * backend's decode (reference proj/src/codec.cpp:27-38).  zlib (third-party,
 * not vendored; pinned zlib1g 1:1.3.dfsg-3.1ubuntu2.2) accepts a stream iff:
 *   - the 2-byte header passes (CMF*256+FLG) % 31 == 0, CM == 8, CINFO <= 7,
 *     FDICT clear (inflate.c HEAD; FDICT -> Z_NEED_DICT -> Z_DATA_ERROR);
 *   - every block is valid (inflate.c TYPE/STORED/TABLE/LENLENS/CODELENS/LEN/
 *     DIST and inftrees.c inflate_table's over-subscribed / incomplete rules);
 *   - the big-endian Adler-32 trailer matches (inflate.c CHECK);
 *   - the output fits destLen (uncompress2: destLen == 0 is served by a 1-byte
 *     scratch buffer, so a stream of <= 1 byte "succeeds" with 0 bytes).
 * Bytes after the trailer are ignored.  Every failure is one status here,
 * because the reference maps all of them to CorruptContainer.
 */
#include <stdlib.h>
#include <string.h>

#include "bboracle.h"

typedef struct {
  const uint8_t* in;
  size_t n, pos; /* byte position of next unread byte */
  uint64_t hold;
  int bits;
} bitr;

/* returns 0 if not enough input */
static int need(bitr* r, int k) {
  while (r->bits < k) {
    if (r->pos >= r->n) return 0;
    r->hold |= (uint64_t)r->in[r->pos++] << r->bits;
    r->bits += 8;
  }
  return 1;
}
static unsigned take(bitr* r, int k) {
  unsigned v = (unsigned)(r->hold & ((1ull << k) - 1));
  r->hold >>= k;
  r->bits -= k;
  return v;
}

/* canonical Huffman decoding table: for every length, first code / count /
 * symbols in order (puff-style), plus zlib's validity rules. */
typedef struct {
  short count[16];
  short symbol[320];
  int max; /* longest length present, 0 = no codes */
} huff;

enum { T_CODES, T_LENS, T_DISTS };

/* inftrees.c inflate_table validity: over-subscribed -> error; incomplete ->
 * error unless (type != CODES and max length == 1); no codes -> OK. */
static int build(huff* h, const unsigned short* lens, int n, int type) {
  short offs[16];
  memset(h->count, 0, sizeof(h->count));
  for (int s = 0; s < n; s++) h->count[lens[s]]++;
  int max = 15;
  while (max >= 1 && h->count[max] == 0) max--;
  h->max = max;
  if (max == 0) return 0;
  int left = 1;
  for (int len = 1; len <= 15; len++) {
    left <<= 1;
    left -= h->count[len];
    if (left < 0) return -1;
  }
  if (left > 0 && (type == T_CODES || max != 1)) return -1;
  offs[1] = 0;
  for (int len = 1; len < 15; len++) offs[len + 1] = (short)(offs[len] + h->count[len]);
  for (int s = 0; s < n; s++)
    if (lens[s] != 0) h->symbol[offs[lens[s]]++] = (short)s;
  return 0;
}

/* decode one symbol; -1 = invalid code (incomplete / empty table), -2 = input */
static int decode(bitr* r, const huff* h) {
  int code = 0, first = 0, index = 0;
  if (h->max == 0) {
    /* zlib's empty table: any 1-bit pattern is an invalid code */
    if (!need(r, 1)) return -2;
    return -1;
  }
  for (int len = 1; len <= 15; len++) {
    if (!need(r, 1)) return -2;
    code |= (int)take(r, 1);
    int count = h->count[len];
    if (code - count < first) return h->symbol[index + (code - first)];
    index += count;
    first += count;
    first <<= 1;
    code <<= 1;
    if (len >= h->max) return -1; /* code beyond the longest length: unassigned */
  }
  return -1;
}

static const unsigned short lbase[29] = {3,  4,  5,  6,  7,  8,  9,  10,  11,  13,  15,  17,  19,  23, 27,
                                         31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
static const unsigned short lext[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2,
                                        2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
static const unsigned short dbase[30] = {1,    2,    3,    4,    5,    7,     9,     13,    17,  25,
                                         33,   49,   65,   97,   129,  193,   257,   385,   513, 769,
                                         1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
static const unsigned short dext[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6,
                                        6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};

typedef struct {
  uint8_t* out;
  size_t lim;   /* bytes we may write (destLen, or 1 when destLen == 0) */
  size_t total; /* bytes produced */
  uint8_t scratch;
} sink;

static int put(sink* s, uint8_t b) {
  if (s->total >= s->lim) return -1;
  s->out[s->total++] = b;
  return 0;
}

static int codes(bitr* r, sink* s, const huff* lh, const huff* dh) {
  for (;;) {
    int sym = decode(r, lh);
    if (sym < 0) return -1;
    if (sym < 256) {
      if (put(s, (uint8_t)sym)) return -1;
    } else if (sym == 256) {
      return 0;
    } else {
      sym -= 257;
      if (sym >= 29) return -1; /* invalid literal/length code (286, 287) */
      if (!need(r, lext[sym])) return -1;
      unsigned len = lbase[sym] + take(r, lext[sym]);
      int ds = decode(r, dh);
      if (ds < 0 || ds >= 30) return -1; /* invalid distance code */
      if (!need(r, dext[ds])) return -1;
      size_t dist = dbase[ds] + take(r, dext[ds]);
      if (dist > s->total) return -1; /* invalid distance too far back */
      while (len--) {
        if (put(s, s->out[s->total - dist])) return -1;
      }
    }
  }
}

int orc_zlib_uncompress(const uint8_t* in, size_t n, uint8_t* out, size_t cap, size_t* out_len) {
  sink s;
  s.out = cap ? out : &s.scratch;
  s.lim = cap ? cap : 1;
  s.total = 0;
  bitr r = {in, n, 0, 0, 0};
  *out_len = 0;
  if (n < 2) return -5;
  unsigned cmf = in[0], flg = in[1];
  r.pos = 2;
  if (((cmf << 8) + flg) % 31 != 0) return -3;
  if ((cmf & 0x0f) != 8) return -3;
  if ((cmf >> 4) + 8 > 15) return -3;
  if (flg & 0x20) return -3;
  static const unsigned char order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
  int last;
  do {
    if (!need(&r, 3)) return -5;
    last = (int)take(&r, 1);
    unsigned type = take(&r, 2);
    if (type == 0) {
      /* stored: discard to byte boundary */
      take(&r, r.bits & 7);
      if (!need(&r, 32)) return -5;
      unsigned len = take(&r, 16), nlen = take(&r, 16);
      if (len != (~nlen & 0xffff)) return -3;
      /* remaining whole bytes in hold (bits is a multiple of 8) then raw input */
      while (len && r.bits) {
        if (put(&s, (uint8_t)take(&r, 8))) return -5;
        len--;
      }
      if (r.pos + len > n) return -5;
      for (unsigned i = 0; i < len; i++)
        if (put(&s, in[r.pos + i])) return -5;
      r.pos += len;
    } else if (type == 1) {
      static huff fl, fd;
      static int init = 0;
      if (!init) {
        unsigned short lens[288];
        int i;
        for (i = 0; i < 144; i++) lens[i] = 8;
        for (; i < 256; i++) lens[i] = 9;
        for (; i < 280; i++) lens[i] = 7;
        for (; i < 288; i++) lens[i] = 8;
        build(&fl, lens, 288, T_LENS);
        for (i = 0; i < 32; i++) lens[i] = 5;
        build(&fd, lens, 32, T_DISTS);
        init = 1;
      }
      if (codes(&r, &s, &fl, &fd)) return -3;
    } else if (type == 2) {
      if (!need(&r, 14)) return -5;
      int nlen = (int)take(&r, 5) + 257, ndist = (int)take(&r, 5) + 1, ncode = (int)take(&r, 4) + 4;
      if (nlen > 286 || ndist > 30) return -3;
      unsigned short lens[320];
      memset(lens, 0, sizeof(lens));
      for (int i = 0; i < ncode; i++) {
        if (!need(&r, 3)) return -5;
        lens[order[i]] = (unsigned short)take(&r, 3);
      }
      huff ch, lh, dh;
      if (build(&ch, lens, 19, T_CODES)) return -3;
      int have = 0;
      memset(lens, 0, sizeof(lens));
      while (have < nlen + ndist) {
        int sym;
        if (ch.max == 0) {
          /* zlib's empty code-length table decodes every 1-bit pattern as 0 */
          if (!need(&r, 1)) return -5;
          take(&r, 1);
          sym = 0;
        } else {
          sym = decode(&r, &ch);
          if (sym == -2) return -5;
          if (sym < 0) return -3;
        }
        if (sym < 16) {
          lens[have++] = (unsigned short)sym;
        } else {
          unsigned len = 0, copy;
          if (sym == 16) {
            if (have == 0) return -3;
            len = lens[have - 1];
            if (!need(&r, 2)) return -5;
            copy = 3 + take(&r, 2);
          } else if (sym == 17) {
            if (!need(&r, 3)) return -5;
            copy = 3 + take(&r, 3);
          } else {
            if (!need(&r, 7)) return -5;
            copy = 11 + take(&r, 7);
          }
          if (have + (int)copy > nlen + ndist) return -3;
          while (copy--) lens[have++] = (unsigned short)len;
        }
      }
      if (lens[256] == 0) return -3;
      if (build(&lh, lens, nlen, T_LENS)) return -3;
      if (build(&dh, lens + nlen, ndist, T_DISTS)) return -3;
      if (codes(&r, &s, &lh, &dh)) return -3;
    } else {
      return -3;
    }
  } while (!last);
  /* CHECK: byte-align, then the big-endian Adler-32 of the output */
  take(&r, r.bits & 7);
  if (!need(&r, 32)) return -5;
  unsigned b0 = take(&r, 8), b1 = take(&r, 8), b2 = take(&r, 8), b3 = take(&r, 8);
  uint32_t want = (b0 << 24) | (b1 << 16) | (b2 << 8) | b3;
  if (want != orc_adler32(1, s.out, s.total)) return -3;
  *out_len = cap ? s.total : 0;
  return 0;
}
