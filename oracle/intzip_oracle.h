/*
 * intzip_oracle.h — CPU restatement of the reference's hot-path algorithms.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 decoder;
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  The product (paper_1209_2137_b200/) never links or calls it.
 *
 * Every function restates one reference function (file:line under
 * /root/reference/proj/core).  Pinned against the reference's own
 * known-answer tests (tests/test_oracle_golden.py) and against the reference
 * compiled from its sources (oracle/_ref, tests/test_oracle_vs_ref.py).
 * Status codes are izg_status values from include/intzip_b200.h.
 */
#ifndef INTZIP_ORACLE_H
#define INTZIP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* bitpack.cpp:287-291 */
uint32_t orc_max_bitwidth(const uint32_t* values, size_t n);
/* bitpack.h:18-23 layout; bitpack.cpp:122-161 / 324-328 (unpack) and
 * 87-120 / 318-322 (masked pack) */
void orc_unpack_vertical128(const uint32_t* words, uint32_t b, uint32_t* out);
void orc_pack_vertical128(const uint32_t* values, uint32_t b, uint32_t* out);
/* bitpack.h:12-16 scalar layout; unpack_scalar32 (bitpack.cpp:305-309) */
void orc_unpack_scalar32(const uint32_t* words, uint32_t b, uint32_t* out);

/* delta.cpp:18-89 (D1, D4); D2/DM are extensions (izg_delta).
 * encode returns 0, or 1 when the input decreases (delta.cpp:13) and
 * allow_wrap == 0. */
void orc_delta_decode(int delta, uint32_t* values, size_t n);
int orc_delta_encode(int delta, uint32_t* values, size_t n, int allow_wrap);

/* codec_basic.cpp:16-51 */
size_t orc_vbyte_encode(const uint32_t* values, size_t n, uint8_t* out);
int orc_vbyte_decode(const uint8_t* bytes, size_t nbytes, uint32_t* out,
                     size_t count, size_t* consumed);

/* codec_patched.cpp:15-48 */
void orc_histogram_of_widths(const uint32_t* values, size_t n, uint32_t* counts33);
uint64_t orc_fastpfor_cost_bits(const uint32_t* counts33, uint32_t block_len,
                                uint32_t b);
void orc_fastpfor_choose_width(const uint32_t* counts33, uint32_t block_len,
                               uint32_t* b, uint32_t* maxbits);

/* Codec::encode_deltas / decode_deltas for izg_codec
 * (codec_binpack.cpp:70-119, codec_patched.cpp:219-417).  Decode also covers
 * IZG_BP32 (codec_binpack.cpp:43-60), IZG_FASTPFOR and IZG_SIMPLEPFOR
 * (codec_patched.cpp:292-417, scalar_arrays / simple8b storage); encode only
 * the two SIMD codecs.
 * encode returns words written (out must hold orc_encode_bound words) or
 * (size_t)-1 on a count error; decode returns an izg_status. */
size_t orc_encode_bound(int codec, size_t count);
size_t orc_encode_deltas(int codec, const uint32_t* deltas, size_t count,
                         uint32_t* out);
int orc_decode_deltas(int codec, const uint32_t* words, size_t nwords,
                      uint32_t* out, size_t count, size_t* consumed);

/* One chunk of encode_array / decode_array (codec.cpp:14-69).
 * orc_encode_chunk: n values (1..65536) -> payload words (returns count, or
 * (size_t)-1 when the input decreases and allow_wrap == 0; with allow_wrap
 * the deltas are taken mod 2^32, which decode_array accepts).
 * orc_decode_chunk: returns an izg_status. */
size_t orc_encode_chunk(int codec, int delta, const uint32_t* values, uint32_t n,
                        uint32_t* out, int allow_wrap);
int orc_decode_chunk(int codec, int delta, const uint32_t* payload,
                     size_t nwords, uint32_t n, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif
