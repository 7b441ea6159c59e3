// encode.cuh — GPU encoder (secondary path).
//
// Restates, fused per chunk:
//   encode_array's chunk body       codec.cpp:21-35 (delta, core, VByte tail)
//   delta_encode_scalar / _stride4  delta.cpp:18-23, 53-58 (+ D2/DM extensions)
//   SimdBp128Codec::encode_deltas   codec_binpack.cpp:70-92
//   max_bitwidth / pack_vertical128 bitpack.cpp:287-291, 87-120
//   vbyte_encode                    codec_basic.cpp:16-25
// Output words are bit-identical to the reference encoder's
// (tests/test_gpu_encode.py compares them word for word).
//
// One warp encodes one chunk, four blocks per iteration in the same register
// layout as the decoder (lane 8q+s8 holds 16 consecutive integers of block
// q).  A block's width is an 8-lane OR reduction; its packed rows are built
// with shared-memory OR reductions in a per-warp tile and copied out
// coalesced.  A meta-block's 16-byte descriptor precedes its payloads but
// only earlier widths determine a block's offset, so the descriptor is
// written after the meta-block's last block.
#pragma once
#include <cstdint>

#include "../../include/intzip_b200.h"
#include "izg_ptx.cuh"

namespace izg {

constexpr int kEncWarps = 8;

__device__ __forceinline__ uint32_t bitw(uint32_t v) { return 32u - __clz(v); }

// Load one thread's 16 consecutive values of block `blk` (mapping C) and form
// their differences (delta.cpp:18-23, 53-58 + D2/DM extensions).  `carry` is
// the last slot of the previous warp iteration (zeros at the chunk start, so
// the first values are their own deltas); `bad` records a decrease.
template <int DELTA, bool WRAP>
__device__ __forceinline__ void load_deltas(const uint32_t* x, bool xal, uint32_t blk, bool live,
                                            int lane, uint4& carry, uint32_t (&d)[4][4],
                                            bool& bad) {
  const uint32_t s8 = lane & 7;
  constexpr bool kArray = DELTA != IZG_DELTA_NONE;
  const uint32_t* xb = x + (size_t)blk * 128 + 16 * s8;
  uint32_t v[4][4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (live) {
      if (xal) {
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(xb) + k);
        v[k][0] = t.x; v[k][1] = t.y; v[k][2] = t.z; v[k][3] = t.w;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) v[k][j] = __ldg(xb + 4 * k + j);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) v[k][j] = 0;
    }
  }
  uint4 prev;
  prev.x = __shfl_up_sync(0xFFFFFFFFu, v[3][0], 1);
  prev.y = __shfl_up_sync(0xFFFFFFFFu, v[3][1], 1);
  prev.z = __shfl_up_sync(0xFFFFFFFFu, v[3][2], 1);
  prev.w = __shfl_up_sync(0xFFFFFFFFu, v[3][3], 1);
  if (lane == 0) prev = carry;
  carry.x = __shfl_sync(0xFFFFFFFFu, v[3][0], 31);
  carry.y = __shfl_sync(0xFFFFFFFFu, v[3][1], 31);
  carry.z = __shfl_sync(0xFFFFFFFFu, v[3][2], 31);
  carry.w = __shfl_sync(0xFFFFFFFFu, v[3][3], 31);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t p0 = k ? v[k - 1][0] : prev.x, p1 = k ? v[k - 1][1] : prev.y;
    const uint32_t p2 = k ? v[k - 1][2] : prev.z, p3 = k ? v[k - 1][3] : prev.w;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t pr = 0;
      if (DELTA == IZG_DELTA_D4) pr = j == 0 ? p0 : j == 1 ? p1 : j == 2 ? p2 : p3;
      if (DELTA == IZG_DELTA_D1) pr = j ? v[k][j - 1] : p3;
      if (DELTA == IZG_DELTA_D2) pr = j >= 2 ? v[k][j - 2] : (j == 0 ? p2 : p3);
      if (DELTA == IZG_DELTA_DM) pr = p3;
      if (!WRAP && kArray && live && v[k][j] < pr) bad = true;
      d[k][j] = v[k][j] - pr;
    }
  }
}

// Variable Byte remainder of values [core, n) appended at o[pos..]
// (codec.cpp:29-33; codec_basic.cpp:16-25); one lane.  Returns an izg_status.
template <int DELTA, bool WRAP>
__device__ int32_t vbyte_append(const uint32_t* x, uint32_t core, uint32_t n, uint32_t* o,
                                uint32_t& pos) {
  uint32_t acc = 0, nbytes = 0;
  for (uint32_t i = core; i < n; ++i) {
    const uint32_t xi = x[i];
    uint32_t pr = 0;
    if (DELTA == IZG_DELTA_D4) pr = i >= 4 ? x[i - 4] : 0u;
    if (DELTA == IZG_DELTA_D1) pr = i >= 1 ? x[i - 1] : 0u;
    if (DELTA == IZG_DELTA_D2) pr = i >= 2 ? x[i - 2] : 0u;
    if (DELTA == IZG_DELTA_DM) pr = i >= 4 ? x[(i & ~3u) - 1] : 0u;
    if (!WRAP && xi < pr) return IZG_E_DECREASING;
    uint32_t dv = xi - pr;
    for (;;) {
      const uint32_t byte = dv >= 128 ? (dv & 0x7Fu) : (dv | 0x80u);
      acc |= byte << (8 * (nbytes & 3));
      if ((++nbytes & 3) == 0) {
        o[pos++] = acc;
        acc = 0;
      }
      if (dv < 128) break;
      dv >>= 7;
    }
  }
  if (nbytes & 3) o[pos++] = acc;
  return IZG_OK;
}

template <int DELTA, bool WRAP>
__global__ void __launch_bounds__(kEncWarps * 32)
    bp128_encode_kernel(const uint32_t* __restrict__ values, izg_chunk* __restrict__ chunks,
                        uint32_t n_chunks, uint32_t* __restrict__ words,
                        int32_t* __restrict__ status, uint32_t* __restrict__ next_chunk) {
  __shared__ uint32_t tiles[kEncWarps][512];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t q = lane >> 3, s8 = lane & 7;
  uint32_t* tile = tiles[warp];
  constexpr bool kArray = DELTA != IZG_DELTA_NONE;
  for (;;) {
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(next_chunk, 1u);
    c = __shfl_sync(0xFFFFFFFFu, c, 0);
    if (c >= n_chunks) break;
    const izg_chunk ch = chunks[c];
    const uint32_t n = ch.n;
    int32_t st = IZG_OK;
    if (kArray && (n == 0 || n > IZG_CHUNK_SIZE)) st = IZG_E_CHUNK_LENGTH;
    if (!kArray && n % 128 != 0) st = IZG_E_COUNT_MULTIPLE;
    uint32_t pos = 0;
    if (st == IZG_OK) {
      const uint32_t* x = values + ch.out_off;
      uint32_t* o = words + ch.word_off;
      const bool xal = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
      const uint32_t core = kArray ? n / 128 * 128 : n;
      const uint32_t nb = core / 128;
      bool bad = false;
      uint4 carry = make_uint4(0, 0, 0, 0);  // last slot of the previous iteration
      for (uint32_t mb0 = 0; mb0 < nb; mb0 += 16) {
        const uint32_t G = min(16u, nb - mb0);
        const uint32_t desc = pos;
        pos += 4;
        uint32_t wdesc = 0;  // lane g < 16: width of group g
        for (uint32_t g0 = 0; g0 < G; g0 += 4) {
          const bool live = g0 + q < G;
          uint32_t d[4][4];
          load_deltas<DELTA, WRAP>(x, xal, mb0 + g0 + q, live, lane, carry, d, bad);
          // block width: OR over the block's 8 lanes (bitpack.cpp:287-291)
          uint32_t acc = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) acc |= d[k][0] | d[k][1] | d[k][2] | d[k][3];
          acc |= __shfl_xor_sync(0xFFFFFFFFu, acc, 1);
          acc |= __shfl_xor_sync(0xFFFFFFFFu, acc, 2);
          acc |= __shfl_xor_sync(0xFFFFFFFFu, acc, 4);
          const uint32_t b = live ? bitw(acc) : 0u;
          // payload offsets of the four blocks (words), from the block widths
          const uint32_t b0 = __shfl_sync(0xFFFFFFFFu, b, 0), b1 = __shfl_sync(0xFFFFFFFFu, b, 8);
          const uint32_t b2 = __shfl_sync(0xFFFFFFFFu, b, 16), b3 = __shfl_sync(0xFFFFFFFFu, b, 24);
          const uint32_t off = 4u * (q == 0 ? 0 : q == 1 ? b0 : q == 2 ? b0 + b1 : b0 + b1 + b2);
          const uint32_t total = 4u * (b0 + b1 + b2 + b3);
          if (lane >= (int)g0 && lane < (int)g0 + 4) {
            const uint32_t k = lane - g0;
            wdesc = k == 0 ? b0 : k == 1 ? b1 : k == 2 ? b2 : b3;
          }
          // vertical pack into the tile (bitpack.h:18-23): value of slot s,
          // lane j -> bits [s*b, s*b+b) of lane j's stream
          for (uint32_t i = lane; i < total; i += 32) tile[i] = 0;
          __syncwarp();
          if (b) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t bit = (4u * s8 + k) * b;
              const uint32_t w0 = off + 4u * (bit >> 5), sh = bit & 31u;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                atomicOr(&tile[w0 + j], d[k][j] << sh);
                if (sh + b > 32) atomicOr(&tile[w0 + 4 + j], d[k][j] >> (32 - sh));
              }
            }
          }
          __syncwarp();
          for (uint32_t i = lane; i < total; i += 32) o[pos + i] = tile[i];
          pos += total;
          __syncwarp();
        }
        // descriptor: byte g = width of group g, absent groups 0 (codec_binpack.cpp:86-89)
        const uint32_t wv = lane < 16 ? wdesc : 0u;
        const uint32_t g4 = (lane & 3) * 4;
        const uint32_t w0 = __shfl_sync(0xFFFFFFFFu, wv, g4), w1 = __shfl_sync(0xFFFFFFFFu, wv, g4 + 1);
        const uint32_t w2 = __shfl_sync(0xFFFFFFFFu, wv, g4 + 2), w3 = __shfl_sync(0xFFFFFFFFu, wv, g4 + 3);
        if (lane < 4) o[desc + lane] = w0 | w1 << 8 | w2 << 16 | w3 << 24;
      }
      if (__any_sync(0xFFFFFFFFu, bad)) st = IZG_E_DECREASING;
      if (st == IZG_OK && kArray && core < n && lane == 0) {
        st = vbyte_append<DELTA, WRAP>(x, core, n, o, pos);
      }
      st = __shfl_sync(0xFFFFFFFFu, st, 0);
      pos = __shfl_sync(0xFFFFFFFFu, pos, 0);
    }
    if (lane == 0) {
      status[c] = st;
      chunks[c].n_words = st == IZG_OK ? pos : 0;
    }
  }
}


// ---- SIMD-FastPFOR encoder (codec_patched.cpp:219-290, vertical arrays) ----
//
// Two passes over the page per warp.  Pass 1: per block, the width
// histogram (shared-memory atomics) and the reference's cost argmin
// (codec_patched.cpp:15-48, ties toward the larger b) -> {b, maxbits, c} in a
// shared table; then A (byte-array offset), L (byte-array length), per-width
// counts and the exception-array layout are running sums.  Pass 2 recomputes
// the differences, packs the low b bits (masked) like SIMD-BP128, stores the
// byte-array entries (positions ranked by an 8-lane scan) and ORs every
// exception's high bits straight into its vertical array in global memory
// (zeroed first).
struct FpEncScratch {
  uint32_t tile[512];
  uint32_t tab[512];       // b | maxbits << 6 | c << 12
  uint32_t hist[4][36];
  uint32_t nw[33];         // per width w: exceptions of the page
  uint32_t base[33];       // per width w: page word of array w
};

template <int DELTA, bool WRAP>
__global__ void __launch_bounds__(kEncWarps * 32)
    fastpfor_encode_kernel(const uint32_t* __restrict__ values, izg_chunk* __restrict__ chunks,
                           uint32_t n_chunks, uint32_t* __restrict__ words,
                           int32_t* __restrict__ status, uint32_t* __restrict__ next_chunk) {
  extern __shared__ __align__(16) uint8_t esm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t q = lane >> 3, s8 = lane & 7;
  FpEncScratch& sc = reinterpret_cast<FpEncScratch*>(esm)[warp];
  constexpr bool kArray = DELTA != IZG_DELTA_NONE;
  for (;;) {
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(next_chunk, 1u);
    c = __shfl_sync(0xFFFFFFFFu, c, 0);
    if (c >= n_chunks) break;
    const izg_chunk ch = chunks[c];
    const uint32_t n = ch.n;
    int32_t st = IZG_OK;
    if (kArray && (n == 0 || n > IZG_CHUNK_SIZE)) st = IZG_E_CHUNK_LENGTH;
    if (!kArray && (n % 128 != 0)) st = IZG_E_COUNT_MULTIPLE;
    if (!kArray && n > IZG_CHUNK_SIZE) st = IZG_E_PAGE_TOO_LARGE;
    uint32_t pos = 0;
    if (st == IZG_OK) {
      const uint32_t* x = values + ch.out_off;
      uint32_t* o = words + ch.word_off;
      const bool xal = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
      const uint32_t core = kArray ? n / 128 * 128 : n;
      const uint32_t nb = core / 128;
      bool bad = false;
      if (nb) {
        // ---- pass 1: widths --------------------------------------------
        uint4 carry = make_uint4(0, 0, 0, 0);
        for (uint32_t g0 = 0; g0 < nb; g0 += 4) {
          const bool live = g0 + q < nb;
          uint32_t d[4][4];
          load_deltas<DELTA, WRAP>(x, xal, g0 + q, live, lane, carry, d, bad);
          for (uint32_t i = lane; i < 4 * 36; i += 32) (&sc.hist[0][0])[i] = 0;
          __syncwarp();
          if (live)
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
              for (int j = 0; j < 4; ++j) atomicAdd(&sc.hist[q][bitw(d[k][j])], 1u);
          __syncwarp();
          {
            // fastpfor_choose_width (codec_patched.cpp:33-48): argmin over b <= maxbits of
            // b*128 + (8+maxbits-b)*c(b), c(b) = values wider than b, ties toward the larger
            // b.  The block's eight lanes each take four candidates b = 4*s8 .. 4*s8+3 (lane
            // 7 also b = 32): c(b) is a suffix sum of the histogram (four bins per lane, an
            // 8-lane suffix scan), the winner an 8-lane min of cost << 14 | (63-b) << 8 | c.
            const uint32_t* h = sc.hist[q];
            const uint32_t h0 = h[4 * s8], h1 = h[4 * s8 + 1], h2 = h[4 * s8 + 2],
                           h3 = h[4 * s8 + 3], h32 = h[32];
            uint32_t orv = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) orv |= d[k][0] | d[k][1] | d[k][2] | d[k][3];
            orv |= __shfl_xor_sync(0xFFFFFFFFu, orv, 1);
            orv |= __shfl_xor_sync(0xFFFFFFFFu, orv, 2);
            orv |= __shfl_xor_sync(0xFFFFFFFFu, orv, 4);
            const uint32_t maxbits = bitw(orv);
            const uint32_t tot = h0 + h1 + h2 + h3;
            uint32_t incl = tot;
#pragma unroll
            for (int dd = 1; dd < 8; dd <<= 1) {
              const uint32_t y = __shfl_down_sync(0xFFFFFFFFu, incl, dd, 8);
              if (s8 + dd < 8) incl += y;
            }
            uint32_t above[4];
            above[3] = incl - tot + h32;  // values wider than 4*s8+3
            above[2] = above[3] + h3;
            above[1] = above[2] + h2;
            above[0] = above[1] + h1;
            uint32_t key = 0xFFFFFFFFu;
#pragma unroll
            for (uint32_t i = 0; i < 4; ++i) {
              const uint32_t b = 4 * s8 + i;
              const uint32_t cost = b * 128u + (8u + maxbits - b) * above[i];
              if (b <= maxbits) key = min(key, cost << 14 | (63u - b) << 8 | above[i]);
            }
            if (maxbits == 32) key = min(key, (32u * 128u) << 14 | (63u - 32u) << 8);
            key = min(key, __shfl_xor_sync(0xFFFFFFFFu, key, 1));
            key = min(key, __shfl_xor_sync(0xFFFFFFFFu, key, 2));
            key = min(key, __shfl_xor_sync(0xFFFFFFFFu, key, 4));
            if (s8 == 0 && live)
              sc.tab[g0 + q] = (63u - ((key >> 8) & 63u)) | maxbits << 6 | (key & 0xFFu) << 12;
          }
          __syncwarp();
        }
        if (__any_sync(0xFFFFFFFFu, bad)) st = IZG_E_DECREASING;
      }
      if (st == IZG_OK && nb) {
        // ---- layout: A, L, per-width counts, array bases ----------------
        sc.nw[lane] = 0;
        if (lane == 0) sc.nw[32] = 0;
        __syncwarp();
        uint32_t pk = 0, bl = 0;
        for (uint32_t k = lane; k < nb; k += 32) {
          const uint32_t e = sc.tab[k], b = e & 63u, mb = (e >> 6) & 63u, cc = e >> 12;
          pk += 4 * b;
          bl += mb > b ? 3 + cc : 2;
          if (mb > b) atomicAdd(&sc.nw[mb - b], cc);
        }
        pk = __reduce_add_sync(0xFFFFFFFFu, pk);
        bl = __reduce_add_sync(0xFFFFFFFFu, bl);
        __syncwarp();
        const uint32_t A = 1 + pk, L = bl, baw = (L + 3) / 4;
        uint32_t p = A + 1 + baw + 1;  // after the bitset word
        if (lane == 0) {
          uint32_t bits = 0;
          for (uint32_t w = 1; w <= 32; ++w) {
            if (!sc.nw[w]) continue;
            bits |= 1u << (w - 1);
            p += 1;
            p = (p + 3) & ~3u;
            sc.base[w] = p;
            p += (sc.nw[w] + 127) / 128 * 4 * w;
          }
          sc.base[0] = bits;
        }
        __syncwarp();
        p = __shfl_sync(0xFFFFFFFFu, p, 0);
        // zero [A+1, p): byte-array padding, count/pad words, exception arrays
        for (uint32_t i = A + 1 + lane; i < p; i += 32) o[i] = 0;
        __syncwarp();
        uint8_t* ba = reinterpret_cast<uint8_t*>(o + A + 1);
        // ---- pass 2: payloads, byte array, exception highs ---------------
        uint4 carry = make_uint4(0, 0, 0, 0);
        uint32_t packed = 1, bpos = 0;
        uint32_t used = 0;  // lane w-1: exceptions of width w placed so far
        bool dummy = false;
        for (uint32_t g0 = 0; g0 < nb; g0 += 4) {
          const uint32_t ng = min(4u, nb - g0);
          const bool live = q < ng;
          uint32_t d[4][4];
          load_deltas<DELTA, true>(x, xal, g0 + q, live, lane, carry, d, dummy);
          // lanes 0..3: block fields and running sums (as the decoder)
          uint32_t b = 0, mb = 0, cc = 0;
          if ((uint32_t)lane < ng) {
            const uint32_t e = sc.tab[g0 + lane];
            b = e & 63u;
            mb = (e >> 6) & 63u;
            cc = e >> 12;
          }
          const uint32_t w = mb - b;
          uint32_t acc = 0, add = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t wc = __shfl_sync(0xFFFFFFFFu, w | cc << 8, j);
            const uint32_t wj = wc & 0xFFu, cj = wc >> 8;
            if (j < lane && wj == w) acc += cj;
            if (cj && wj == (uint32_t)lane + 1) add += cj;
          }
          const uint32_t cur = __shfl_sync(0xFFFFFFFFu, used, (w - 1) & 31) + acc;
          used += add;
          uint32_t pkk = 4u * b, bll = (uint32_t)lane < ng ? (cc ? 3 + cc : 2) : 0u;
#pragma unroll
          for (int dd = 1; dd < 4; dd <<= 1) {
            const uint32_t y0 = __shfl_up_sync(0xFFFFFFFFu, pkk, dd, 4);
            const uint32_t y1 = __shfl_up_sync(0xFFFFFFFFu, bll, dd, 4);
            if ((lane & 3) >= dd) {
              pkk += y0;
              bll += y1;
            }
          }
          const uint32_t ent = bpos + bll - ((uint32_t)lane < ng ? (cc ? 3 + cc : 2) : 0u);
          if ((uint32_t)lane < ng) {  // entry header (codec_patched.cpp:233-240)
            ba[ent] = (uint8_t)b;
            ba[ent + 1] = (uint8_t)mb;
            if (cc) ba[ent + 2] = (uint8_t)cc;
          }
          // per-thread view of its block q
          const uint32_t myb = __shfl_sync(0xFFFFFFFFu, b, q);
          const uint32_t mymb = __shfl_sync(0xFFFFFFFFu, mb, q);
          const uint32_t myent = __shfl_sync(0xFFFFFFFFu, ent, q);
          const uint32_t mycur = __shfl_sync(0xFFFFFFFFu, cur, q);
          const uint32_t myoff = __shfl_sync(0xFFFFFFFFu, pkk, q) - 4u * myb;
          const uint32_t total = __shfl_sync(0xFFFFFFFFu, pkk, 3);
          // exceptions: rank within the block by an 8-lane exclusive scan
          uint32_t emask = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (live && myb < 32 && (d[k][j] >> myb)) emask |= 1u << (4 * k + j);
          uint32_t rank = __popc(emask);
#pragma unroll
          for (int dd = 1; dd < 8; dd <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, rank, dd, 8);
            if (s8 >= (uint32_t)dd) rank += y;
          }
          rank -= __popc(emask);
          const uint32_t ww = mymb - myb;
          const uint32_t bw_ = 4u * ww;
          for (uint32_t m = emask; m; m &= m - 1) {
            const uint32_t t = __ffs(m) - 1;
            const uint32_t kk = t >> 2, jj = t & 3;
            const uint32_t val = kk == 0 ? (jj == 0 ? d[0][0] : jj == 1 ? d[0][1] : jj == 2 ? d[0][2] : d[0][3])
                               : kk == 1 ? (jj == 0 ? d[1][0] : jj == 1 ? d[1][1] : jj == 2 ? d[1][2] : d[1][3])
                               : kk == 2 ? (jj == 0 ? d[2][0] : jj == 1 ? d[2][1] : jj == 2 ? d[2][2] : d[2][3])
                                         : (jj == 0 ? d[3][0] : jj == 1 ? d[3][1] : jj == 2 ? d[3][2] : d[3][3]);
            ba[myent + 3 + rank] = (uint8_t)(16 * s8 + t);
            const uint32_t r = mycur + rank;
            const uint32_t tt = r & 127u, bit = (tt >> 2) * ww, sh = bit & 31u;
            uint32_t* wp = o + sc.base[ww] + (r >> 7) * bw_ + 4u * (bit >> 5) + (tt & 3u);
            const uint32_t high = val >> myb;
            atomicOr(wp, high << sh);
            if (sh + ww > 32) atomicOr(wp + 4, high >> (32 - sh));
            ++rank;
          }
          // low bits, vertically packed (pack_vertical128_masked)
          const uint32_t mask = myb >= 32 ? 0xFFFFFFFFu : (1u << myb) - 1u;
          for (uint32_t i = lane; i < total; i += 32) sc.tile[i] = 0;
          __syncwarp();
          if (live && myb) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t bit = (4u * s8 + k) * myb;
              const uint32_t w0 = myoff + 4u * (bit >> 5), sh = bit & 31u;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint32_t lo = d[k][j] & mask;
                atomicOr(&sc.tile[w0 + j], lo << sh);
                if (sh + myb > 32) atomicOr(&sc.tile[w0 + 4 + j], lo >> (32 - sh));
              }
            }
          }
          __syncwarp();
          for (uint32_t i = lane; i < total; i += 32) o[packed + i] = sc.tile[i];
          packed += total;
          bpos += __shfl_sync(0xFFFFFFFFu, bll, 3);
          __syncwarp();
        }
        if (lane == 0) {
          o[0] = A;
          o[A] = L;
          o[A + 1 + baw] = sc.base[0];
          // count words: the word before each array's 16-byte-aligned start,
          // minus the zero padding (codec_patched.cpp:273-276)
          uint32_t q2 = A + 1 + baw + 1;
          for (uint32_t w2 = 1; w2 <= 32; ++w2) {
            if (!sc.nw[w2]) continue;
            o[q2] = sc.nw[w2];
            q2 = ((q2 + 1 + 3) & ~3u);
            q2 += (sc.nw[w2] + 127) / 128 * 4 * w2;
          }
        }
        pos = p;
      }
      if (st == IZG_OK && kArray && core < n && lane == 0) st = vbyte_append<DELTA, WRAP>(x, core, n, o, pos);
      st = __shfl_sync(0xFFFFFFFFu, st, 0);
      pos = __shfl_sync(0xFFFFFFFFu, pos, 0);
    }
    if (lane == 0) {
      status[c] = st;
      chunks[c].n_words = st == IZG_OK ? pos : 0;
    }
  }
}

inline uint64_t izg_encode_bound_impl(int codec, uint32_t n) {
  const uint64_t nb = n / 128;
  const uint64_t rem = 159;  // 127 VByte values of at most 5 bytes
  if (codec == IZG_SIMDBP128) return 4 * ((nb + 15) / 16) + 128 * nb + rem + 4;
  return 2 + 128 * nb + 1 + (131 * nb + 3) / 4 + 1 + 32 * 4 + 128 * nb + 32 * 128 + rem + 4;
}

}  // namespace izg
