/*
 * intzip_oracle.c — CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see intzip_oracle.h).  Written for clarity, not
 * speed: bit-by-bit packing, straight loops, the reference's check order.
 * File:line citations are under /root/reference/proj/core/.
 */
#include "intzip_oracle.h"

#include <string.h>

#include "../include/intzip_b200.h"

/* ---- bit packing ------------------------------------------------------ */

/* bitpack.cpp:287-291: bit_width of the OR of all values. */
uint32_t orc_max_bitwidth(const uint32_t* values, size_t n) {
  uint32_t acc = 0, w = 0;
  for (size_t i = 0; i < n; ++i) acc |= values[i];
  while (acc) { ++w; acc >>= 1; }
  return w;
}

/* Vertical layout, bitpack.h:12-23: value t lives in lane t%4 at lane slot
 * t/4, i.e. at bits [slot*b, slot*b+b) of that lane's scalar bit string; bit
 * p of a lane string is bit p%32 of lane word p/32, and lane word i of lane j
 * is stream word 4i+j.  Restates unpack128<B> (bitpack.cpp:122-161). */
void orc_unpack_vertical128(const uint32_t* words, uint32_t b, uint32_t* out) {
  for (uint32_t t = 0; t < 128; ++t) {
    const uint32_t lane = t % 4, slot = t / 4;
    uint32_t v = 0;
    for (uint32_t k = 0; k < b; ++k) {
      const uint32_t p = slot * b + k;
      const uint32_t word = words[4 * (p / 32) + lane];
      v |= ((word >> (p % 32)) & 1u) << k;
    }
    out[t] = v;
  }
}

/* pack128<B> with masking (bitpack.cpp:87-120, 318-322): v mod 2^b. */
/* bitpack.h:12-16 scalar layout, unpack_scalar32 (bitpack.cpp:305-309):
 * value i at bits [i*b, i*b+b) of the b-word stream, low bits first. */
void orc_unpack_scalar32(const uint32_t* words, uint32_t b, uint32_t* out) {
  for (uint32_t i = 0; i < 32; ++i) {
    uint64_t v = 0;
    for (uint32_t k = 0; k < b; ++k) {
      const uint32_t bit = i * b + k;
      v |= (uint64_t)((words[bit / 32] >> (bit % 32)) & 1u) << k;
    }
    out[i] = (uint32_t)v;
  }
}

void orc_pack_vertical128(const uint32_t* values, uint32_t b, uint32_t* out) {
  memset(out, 0, sizeof(uint32_t) * 4 * b);
  for (uint32_t t = 0; t < 128; ++t) {
    const uint32_t lane = t % 4, slot = t / 4;
    for (uint32_t k = 0; k < b; ++k) {
      if ((values[t] >> k) & 1u) {
        const uint32_t p = slot * b + k;
        out[4 * (p / 32) + lane] |= 1u << (p % 32);
      }
    }
  }
}

/* ---- differential coding --------------------------------------------- */

/* delta_decode_scalar / delta_decode_stride4 (delta.cpp:25-75), wrapping;
 * D2 / DM are extensions (see izg_delta). */
void orc_delta_decode(int delta, uint32_t* v, size_t n) {
  switch (delta) {
    case IZG_DELTA_D1:
      for (size_t i = 1; i < n; ++i) v[i] += v[i - 1];
      break;
    case IZG_DELTA_D4:
      for (size_t i = 4; i < n; ++i) v[i] += v[i - 4];
      break;
    case IZG_DELTA_D2:
      for (size_t i = 2; i < n; ++i) v[i] += v[i - 2];
      break;
    case IZG_DELTA_DM: {
      uint32_t last = 0; /* x_{4k-1}, x_{-1} = 0 */
      for (size_t base = 0; base < n; base += 4) {
        const size_t end = base + 4 < n ? base + 4 : n;
        for (size_t i = base; i < end; ++i) v[i] += last;
        last = v[end - 1];
      }
      break;
    }
    default:
      break;
  }
}

/* delta_encode_scalar / _stride4 (delta.cpp:18-23, 53-58): downward in place,
 * reject a decrease (delta.cpp:13) unless allow_wrap. */
int orc_delta_encode(int delta, uint32_t* v, size_t n, int allow_wrap) {
  size_t i;
  switch (delta) {
    case IZG_DELTA_D1:
      for (i = n; i-- > 1;) {
        if (!allow_wrap && v[i] < v[i - 1]) return 1;
        v[i] -= v[i - 1];
      }
      break;
    case IZG_DELTA_D4:
      for (i = n; i-- > 4;) {
        if (!allow_wrap && v[i] < v[i - 4]) return 1;
        v[i] -= v[i - 4];
      }
      break;
    case IZG_DELTA_D2:
      for (i = n; i-- > 2;) {
        if (!allow_wrap && v[i] < v[i - 2]) return 1;
        v[i] -= v[i - 2];
      }
      break;
    case IZG_DELTA_DM: {
      /* x_{4k+j} - x_{4k-1}; walk vectors downward so bases are still raw. */
      size_t nvec = (n + 3) / 4;
      for (size_t k = nvec; k-- > 1;) {
        const uint32_t base = v[4 * k - 1];
        const size_t end = 4 * k + 4 < n ? 4 * k + 4 : n;
        for (i = 4 * k; i < end; ++i) {
          if (!allow_wrap && v[i] < base) return 1;
          v[i] -= base;
        }
      }
      break;
    }
    default:
      break;
  }
  return 0;
}

/* ---- Variable Byte (codec_basic.cpp:16-51) ------------------------------ */

size_t orc_vbyte_encode(const uint32_t* values, size_t n, uint8_t* out) {
  size_t pos = 0;
  for (size_t i = 0; i < n; ++i) {
    uint32_t v = values[i];
    while (v >= 128) {
      out[pos++] = (uint8_t)(v & 0x7F);
      v >>= 7;
    }
    out[pos++] = (uint8_t)(v | 0x80);
  }
  return pos;
}

int orc_vbyte_decode(const uint8_t* bytes, size_t nbytes, uint32_t* out,
                     size_t count, size_t* consumed) {
  size_t pos = 0;
  for (size_t i = 0; i < count; ++i) {
    uint32_t v = 0, shift = 0;
    for (;;) {
      if (pos >= nbytes) return IZG_E_VBYTE_TRUNCATED;
      const uint8_t b = bytes[pos++];
      if (b & 0x80) {
        if (shift == 28 && (b & 0x70)) return IZG_E_VBYTE_OVERFLOW;
        v |= (uint32_t)(b & 0x7F) << shift;
        break;
      }
      if (shift == 28) return IZG_E_VBYTE_TOO_LONG;
      v |= (uint32_t)b << shift;
      shift += 7;
    }
    out[i] = v;
  }
  *consumed = pos;
  return IZG_OK;
}

/* ---- FastPFOR width choice (codec_patched.cpp:15-48) ------------------- */

void orc_histogram_of_widths(const uint32_t* values, size_t n, uint32_t* counts33) {
  memset(counts33, 0, 33 * sizeof(uint32_t));
  for (size_t i = 0; i < n; ++i) counts33[orc_max_bitwidth(&values[i], 1)]++;
}

static uint32_t hist_maxbits(const uint32_t* h) {
  uint32_t m = 0;
  for (uint32_t w = 0; w <= 32; ++w)
    if (h[w]) m = w;
  return m;
}

uint64_t orc_fastpfor_cost_bits(const uint32_t* h, uint32_t block_len, uint32_t b) {
  const uint32_t maxbits = hist_maxbits(h);
  uint64_t exceptions = 0;
  for (uint32_t w = b + 1; w <= 32; ++w) exceptions += h[w];
  uint64_t cost = (uint64_t)b * block_len;
  if (exceptions > 0) cost += (uint64_t)(8 + maxbits - b) * exceptions;
  return cost;
}

void orc_fastpfor_choose_width(const uint32_t* h, uint32_t block_len,
                               uint32_t* b_out, uint32_t* maxbits_out) {
  const uint32_t maxbits = hist_maxbits(h);
  uint32_t best_b = 0;
  uint64_t best = ~(uint64_t)0;
  for (uint32_t b = 0; b <= maxbits; ++b) {
    const uint64_t cost = orc_fastpfor_cost_bits(h, block_len, b);
    if (cost <= best) { /* ties go to the larger width (codec_patched.cpp:42) */
      best = cost;
      best_b = b;
    }
  }
  *b_out = best_b;
  *maxbits_out = maxbits;
}

/* ---- codecs ------------------------------------------------------------- */

size_t orc_encode_bound(int codec, size_t count) {
  const size_t blocks = count / 128;
  if (codec == IZG_SIMDBP128) return 4 * ((blocks + 15) / 16) + 128 * blocks + 4;
  /* header + packed + L + byte array + bitset + 32 arrays (count, pad, data) */
  return 2 + 128 * blocks + (blocks * 131 + 3) / 4 + 1 + 32 * 5 +
         128 * (blocks + 32) + 16;
}

/* SimdBp128Codec::encode_deltas (codec_binpack.cpp:70-92). */
static size_t bp128_encode(const uint32_t* d, size_t count, uint32_t* out) {
  size_t pos = 0;
  for (size_t base = 0; base < count; base += 16 * 128) {
    size_t groups = (count - base) / 128;
    if (groups > 16) groups = 16;
    uint8_t widths[16] = {0};
    for (size_t g = 0; g < groups; ++g)
      widths[g] = (uint8_t)orc_max_bitwidth(d + base + 128 * g, 128);
    for (int w = 0; w < 4; ++w)
      out[pos++] = (uint32_t)widths[4 * w] | (uint32_t)widths[4 * w + 1] << 8 |
                   (uint32_t)widths[4 * w + 2] << 16 | (uint32_t)widths[4 * w + 3] << 24;
    for (size_t g = 0; g < groups; ++g) {
      orc_pack_vertical128(d + base + 128 * g, widths[g], out + pos);
      pos += 4 * (size_t)widths[g];
    }
  }
  return pos;
}

/* SimdBp128Codec::decode_deltas (codec_binpack.cpp:94-119). */
static int bp128_decode(const uint32_t* words, size_t nwords, uint32_t* out,
                        size_t count, size_t* consumed) {
  size_t pos = 0;
  for (size_t base = 0; base < count; base += 16 * 128) {
    size_t groups = (count - base) / 128;
    if (groups > 16) groups = 16;
    if (pos + 4 > nwords) return IZG_E_BP_TRUNC_DESC;
    uint32_t widths[16];
    for (size_t g = 0; g < 16; ++g) widths[g] = (words[pos + g / 4] >> (8 * (g % 4))) & 0xFF;
    pos += 4;
    for (size_t g = 0; g < groups; ++g) {
      if (widths[g] > 32) return IZG_E_BP_WIDTH;
      if (pos + 4 * (size_t)widths[g] > nwords) return IZG_E_BP_TRUNC_PAYLOAD;
      orc_unpack_vertical128(words + pos, widths[g], out + base + 128 * g);
      pos += 4 * (size_t)widths[g];
    }
  }
  *consumed = pos;
  return IZG_OK;
}

/* Bp32Codec::decode_deltas (codec_binpack.cpp:43-60): per 128 integers one
 * descriptor word (byte g = width of scalar group g), then 4 groups. */
static int bp32_decode(const uint32_t* words, size_t nwords, uint32_t* out, size_t count,
                       size_t* consumed) {
  size_t pos = 0;
  for (size_t base = 0; base < count; base += 128) {
    if (pos >= nwords) return IZG_E_BP32_TRUNC_DESC;
    const uint32_t desc = words[pos++];
    for (int g = 0; g < 4; ++g) {
      const uint32_t w = (desc >> (8 * g)) & 0xFF;
      if (w > 32) return IZG_E_BP32_WIDTH;
      if (pos + w > nwords) return IZG_E_BP32_TRUNC_PAYLOAD;
      orc_unpack_scalar32(words + pos, w, out + base + 32 * g);
      pos += w;
    }
  }
  *consumed = pos;
  return IZG_OK;
}

/* simple8b_decode, 32-bit overload (codec_basic.cpp:256-300, table
 * codec_basic.h:45-60): 64-bit words, low half first; selector = low 4 bits;
 * values truncated to 32 bits; returns words consumed or (size_t)-1 when the
 * stream ends before `count` values. */
static const uint32_t kS8Cap[16] = {240, 120, 60, 30, 20, 15, 12, 10, 8, 7, 6, 5, 4, 3, 2, 1};
static const uint32_t kS8Bits[16] = {0, 0, 1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 15, 20, 30, 60};
static size_t simple8b_decode(const uint32_t* words, size_t nwords, uint32_t* out,
                              size_t count) {
  size_t pos = 0, done = 0;
  while (done < count) {
    if (pos + 2 > nwords) return (size_t)-1;
    const uint64_t word = words[pos] | ((uint64_t)words[pos + 1] << 32);
    pos += 2;
    const uint32_t sel = (uint32_t)(word & 0xF), bits = kS8Bits[sel];
    size_t take = count - done < kS8Cap[sel] ? count - done : kS8Cap[sel];
    for (size_t k = 0; k < take; ++k) {
      uint64_t v = 0;
      if (bits) v = (word >> (4 + k * bits)) & ((bits == 64 ? 0 : (1ull << bits)) - 1);
      out[done + k] = (uint32_t)v;
    }
    done += take;
  }
  return pos;
}

/* FastPforCodec::encode_deltas, vertical_arrays storage
 * (codec_patched.cpp:219-290). */
static size_t fastpfor_encode(const uint32_t* d, size_t count, uint32_t* out) {
  if (count == 0) return 0;
  size_t pos = 0;
  const size_t blocks = count / 128;
  out[pos++] = 0; /* patched below */
  uint8_t byte_array[65536 / 128 * 131];
  size_t nba = 0;
  static uint32_t width_arrays[33][65536 + 128];
  size_t nwa[33] = {0};
  for (size_t k = 0; k < blocks; ++k) {
    const uint32_t* v = d + 128 * k;
    uint32_t hist[33], b, maxbits;
    orc_histogram_of_widths(v, 128, hist);
    orc_fastpfor_choose_width(hist, 128, &b, &maxbits);
    byte_array[nba++] = (uint8_t)b;
    byte_array[nba++] = (uint8_t)maxbits;
    if (maxbits > b) {
      uint8_t positions[128];
      uint32_t c = 0;
      for (uint32_t i = 0; i < 128; ++i)
        if (v[i] >> b) positions[c++] = (uint8_t)i;
      byte_array[nba++] = (uint8_t)c;
      memcpy(byte_array + nba, positions, c);
      nba += c;
      for (uint32_t e = 0; e < c; ++e)
        width_arrays[maxbits - b][nwa[maxbits - b]++] = v[positions[e]] >> b;
    }
    orc_pack_vertical128(v, b, out + pos);
    pos += 4 * (size_t)b;
  }
  out[0] = (uint32_t)pos;
  out[pos++] = (uint32_t)nba;
  const size_t ba_words = (nba + 3) / 4;
  memset(out + pos, 0, ba_words * 4);
  memcpy(out + pos, byte_array, nba);
  pos += ba_words;
  uint32_t bitset = 0;
  for (uint32_t w = 1; w <= 32; ++w)
    if (nwa[w]) bitset |= 1u << (w - 1);
  out[pos++] = bitset;
  for (uint32_t w = 1; w <= 32; ++w) {
    if (!nwa[w]) continue;
    out[pos++] = (uint32_t)nwa[w];
    while (pos % 4 != 0) out[pos++] = 0; /* 16-byte alignment in the page */
    const size_t padded = (nwa[w] + 127) / 128 * 128;
    for (size_t i = nwa[w]; i < padded; ++i) width_arrays[w][i] = 0;
    for (size_t g = 0; g < padded / 128; ++g) {
      orc_pack_vertical128(width_arrays[w] + 128 * g, w, out + pos);
      pos += 4 * (size_t)w;
    }
  }
  return pos;
}

/* FastPforCodec::decode_deltas (codec_patched.cpp:292-417) for the three
 * patch storages (codec_patched.cpp:195-199): storage 0 = vertical_arrays
 * (simdfastpfor), 1 = scalar_arrays (fastpfor), 2 = simple8b (simplepfor).
 * Checks in the reference's order. */
static int fastpfor_decode(int storage, const uint32_t* words, size_t nwords, uint32_t* out,
                           size_t count, size_t* consumed) {
  if (count == 0) { *consumed = 0; return IZG_OK; }
  const size_t blocks = count / 128;
  if (nwords == 0) return IZG_E_FP_TRUNC_PAGE;
  const size_t ba_offset = words[0];
  if (ba_offset < 1 || ba_offset >= nwords) return IZG_E_FP_BA_OFFSET;
  const size_t ba_len = words[ba_offset];
  const size_t ba_words = (ba_len + 3) / 4;
  if (ba_offset + 1 + ba_words > nwords) return IZG_E_FP_TRUNC_BA;
  const uint8_t* bytes = (const uint8_t*)(words + ba_offset + 1);

  uint8_t mb[512], mmax[512], mc[512];
  size_t mpos[512];
  size_t bpos = 0;
  for (size_t k = 0; k < blocks; ++k) {
    if (bpos + 2 > ba_len) return IZG_E_FP_TRUNC_META;
    mb[k] = bytes[bpos];
    mmax[k] = bytes[bpos + 1];
    mc[k] = 0;
    bpos += 2;
    if (mb[k] > 32 || mmax[k] > 32 || mb[k] > mmax[k]) return IZG_E_FP_WIDTHS;
    if (mmax[k] > mb[k]) {
      if (bpos >= ba_len) return IZG_E_FP_TRUNC_META;
      mc[k] = bytes[bpos++];
      if (mc[k] == 0) return IZG_E_FP_EMPTY_EXC;
      if (bpos + mc[k] > ba_len) return IZG_E_FP_TRUNC_POS;
      mpos[k] = bpos;
      for (uint32_t i = 0; i < mc[k]; ++i)
        if (bytes[bpos + i] >= 128) return IZG_E_FP_POS_RANGE;
      bpos += mc[k];
    }
  }
  if (bpos != ba_len) return IZG_E_FP_BA_LEN;

  /* Exception highs (codec_patched.cpp:338-379).  Arrays: bitset, then per
   * width its count and its groups (vertical: 16 B-aligned groups of 128;
   * scalar: groups of 32); values are extracted on demand below instead of
   * bulk-unpacked, with identical results.  Simple-8b: one stream of all
   * highs in block order. */
  size_t pos = ba_offset + 1 + ba_words;
  size_t arr_base[33] = {0}, arr_n[33] = {0};
  static uint32_t s8_highs[512 * 255];
  if (storage == 2) {
    size_t total = 0;
    for (size_t k = 0; k < blocks; ++k) total += mc[k];
    const size_t used = simple8b_decode(words + pos, nwords - pos, s8_highs, total);
    if (used == (size_t)-1) return IZG_E_S8_EXHAUSTED;
    pos += used;
  } else {
    if (pos >= nwords) return IZG_E_FP_NO_BITSET;
    const uint32_t bitset = words[pos++];
    for (uint32_t w = 1; w <= 32; ++w) {
      if (!(bitset & (1u << (w - 1)))) continue;
      if (pos >= nwords) return IZG_E_FP_TRUNC_EXC;
      const uint32_t n = words[pos++];
      const size_t group = storage == 0 ? 128 : 32;
      if (storage == 0)
        while (pos % 4 != 0) ++pos;
      const size_t padded = ((size_t)n + group - 1) / group * group;
      const size_t nw = padded / group * (group / 32) * (size_t)w;
      if (pos + nw > nwords) return IZG_E_FP_TRUNC_EXC;
      arr_base[w] = pos;
      arr_n[w] = n;
      pos += nw;
    }
  }

  size_t packed = 1, s8_cursor = 0;
  size_t cursors[33] = {0};
  for (size_t k = 0; k < blocks; ++k) {
    if (packed + 4 * (size_t)mb[k] > ba_offset) return IZG_E_FP_OVERRUN;
    uint32_t* o = out + 128 * k;
    if (storage == 0) {
      orc_unpack_vertical128(words + packed, mb[k], o);
    } else {
      for (int g = 0; g < 4; ++g)
        orc_unpack_scalar32(words + packed + (size_t)mb[k] * g, mb[k], o + 32 * g);
    }
    packed += 4 * (size_t)mb[k];
    if (mc[k]) {
      const uint32_t w = mmax[k] - mb[k];
      for (uint32_t i = 0; i < mc[k]; ++i) {
        uint32_t high;
        if (storage == 2) {
          high = s8_highs[s8_cursor++];
        } else {
          if (cursors[w] >= arr_n[w]) return IZG_E_FP_EXHAUSTED;
          const size_t r = cursors[w]++;
          uint32_t group[128];
          if (storage == 0) {
            orc_unpack_vertical128(words + arr_base[w] + (r / 128) * 4 * w, w, group);
            high = group[r % 128];
          } else {
            orc_unpack_scalar32(words + arr_base[w] + (r / 32) * w, w, group);
            high = group[r % 32];
          }
        }
        o[bytes[mpos[k] + i]] |= high << mb[k];
      }
    }
  }
  if (packed != ba_offset) return IZG_E_FP_PACKED_SIZE;
  *consumed = pos;
  return IZG_OK;
}

size_t orc_encode_deltas(int codec, const uint32_t* deltas, size_t count, uint32_t* out) {
  if (count % 128 != 0 || codec > IZG_SIMDFASTPFOR) return (size_t)-1;
  if (codec == IZG_SIMDBP128) return bp128_encode(deltas, count, out);
  if (count > 65536) return (size_t)-1;
  return fastpfor_encode(deltas, count, out);
}

int orc_decode_deltas(int codec, const uint32_t* words, size_t nwords,
                      uint32_t* out, size_t count, size_t* consumed) {
  if (count % 128 != 0) return IZG_E_COUNT_MULTIPLE;
  if (codec == IZG_SIMDBP128) return bp128_decode(words, nwords, out, count, consumed);
  if (codec == IZG_BP32) return bp32_decode(words, nwords, out, count, consumed);
  if (count > 65536) return IZG_E_PAGE_TOO_LARGE;
  const int storage = codec == IZG_SIMDFASTPFOR ? 0 : codec == IZG_FASTPFOR ? 1 : 2;
  return fastpfor_decode(storage, words, nwords, out, count, consumed);
}

/* ---- pipeline, one chunk (codec.cpp:14-69) ------------------------------ */

size_t orc_encode_chunk(int codec, int delta, const uint32_t* values, uint32_t n,
                        uint32_t* out, int allow_wrap) {
  static uint32_t scratch[65536];
  static uint8_t rem[127 * 5 + 4];
  memcpy(scratch, values, (size_t)n * 4);
  if (orc_delta_encode(delta, scratch, n, allow_wrap)) return (size_t)-1;
  const size_t core = (size_t)n / 128 * 128;
  size_t pos = orc_encode_deltas(codec, scratch, core, out);
  if (core < n) {
    const size_t nb = orc_vbyte_encode(scratch + core, n - core, rem);
    const size_t nw = (nb + 3) / 4; /* append_bytes_as_words, wordbytes.h:22-28 */
    memset(out + pos, 0, nw * 4);
    memcpy(out + pos, rem, nb);
    pos += nw;
  }
  return pos;
}

int orc_decode_chunk(int codec, int delta, const uint32_t* payload,
                     size_t nwords, uint32_t n, uint32_t* out) {
  if (n == 0 || n > 65536) return IZG_E_CHUNK_LENGTH;
  const size_t core = (size_t)n / 128 * 128;
  size_t consumed = 0;
  int st = orc_decode_deltas(codec, payload, nwords, out, core, &consumed);
  if (st) return st;
  if (core < n) {
    size_t rb = 0;
    st = orc_vbyte_decode((const uint8_t*)(payload + consumed),
                          (nwords - consumed) * 4, out + core, n - core, &rb);
    if (st) return st;
    consumed += (rb + 3) / 4;
  }
  if (consumed != nwords) return IZG_E_PAYLOAD_SIZE;
  orc_delta_decode(delta, out, n);
  return IZG_OK;
}
