/* ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product path.
 *
 * CPU restatement of the reference's hot-path arithmetic:
 *   - BBC1 container, byte split/merge, entropy      (reference proj/src/codec.cpp)
 *   - synthetic activations (fp16, + frozen bf16)     (reference proj/src/synth.cpp)
 *   - the deflate backend = zlib 1.3 compress2(level 6) / uncompress
 *     (third-party, NOT vendored under /root/reference: system package zlib1g
 *      1:1.3.dfsg-3.1ubuntu2.2, ZLIB_VERSION "1.3"; call sites reference
 *      proj/src/codec.cpp:17-38).  zlib's published algorithm (deflate.c
 *      deflate_slow/longest_match/fill_window, trees.c, adler32.c, inflate.c)
 *      is restated in oracle/zlib6.c and oracle/inflate.c.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the
 * reference itself (oracle/_ref/libbeeplan_ref.so, compiled from the reference
 * sources by oracle/Makefile and linked with the pinned libz.so.1.3) and against
 * the committed golden vectors in tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
 * reference) may load this library.
 */
#ifndef BB_ORACLE_H
#define BB_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* zlib-exact level-6 deflate (compress2 semantics). Returns 0 or -1 (cap). */
size_t orc_compress_bound(size_t n);
int orc_zlib_compress(const uint8_t* in, size_t n, uint8_t* out, size_t cap, size_t* out_len);
/* Same output, computed through the GPU pipeline's decomposition:
 * per-position match profiles -> lazy parse -> 16383-symbol blocks. */
int orc_zlib_compress_profiled(const uint8_t* in, size_t n, uint8_t* out, size_t cap,
                               size_t* out_len);
/* Per-position match profile (K4 of the GPU pipeline), two u32 per position:
 * prof[2p] for chain budget 128, prof[2p+1] for budget 32.  Layout:
 * bits 0-8 len (0 = no usable match), 9-23 dist, 31 = first candidate at 32506. */
void orc_match_profile(const uint8_t* in, size_t n, uint32_t* prof);
/* Previous-same-hash distance per position (K3): 0 = none within 32767. */
void orc_hash_prev(const uint8_t* in, size_t n, uint16_t* pd);

/* uncompress() semantics: 0 = Z_OK with *out_len bytes, <0 = zlib error code.
 * cap is the caller's destLen (0 allowed: zlib then accepts <=1 byte). */
int orc_zlib_uncompress(const uint8_t* in, size_t n, uint8_t* out, size_t cap, size_t* out_len);

uint32_t orc_adler32(uint32_t adler, const uint8_t* buf, size_t n);

/* BBC1 codec (reference proj/src/codec.cpp). Status codes = bb_status. */
size_t orc_container_bound(size_t n, int backend, int split);
int orc_compress(const uint8_t* in, size_t n, int backend, int split, uint8_t* out, size_t cap,
                 size_t* out_len);
int orc_decompress(const uint8_t* in, size_t n, uint8_t* out, size_t cap, size_t* out_len);
int orc_split(const uint8_t* in, size_t n, uint8_t* high, uint8_t* low);
void orc_merge(const uint8_t* high, const uint8_t* low, size_t count, uint8_t* out);
double orc_entropy(const uint8_t* in, size_t n);

/* Synthetic activations (reference proj/src/synth.cpp:66-94) and the frozen
 * bf16 variant (same Box-Muller stream, bf16 round-to-nearest-even). */
void orc_synth_fp16(size_t elements, uint64_t seed, uint8_t* out);
void orc_synth_bf16(size_t elements, uint64_t seed, uint8_t* out);
uint16_t orc_fp16_from_float(float v);
uint16_t orc_bf16_from_float(float v);

#ifdef __cplusplus
}
#endif
#endif
